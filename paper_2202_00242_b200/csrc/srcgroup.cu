// srcgroup.cu — K4s: source-grouped, warp-specialised fused lookup + accumulate.
//
// For batches whose source clouds are small (<= kSrcMax fp32 points, e.g. global mapping's
// 200-600-point submap sources, each shared by ~50 factors), every factor of one source is
// processed by one CTA while the source cloud sits in shared memory:
//   * the source points and fp64 covariances are loaded once per CTA pass (cp.async) instead
//     of once per factor and per hit — per correspondence the L2 traffic drops to the hash
//     probe (one 16 B bucket) plus, on a hit, the voxel record (80 B);
//   * 12 producer warps transform points straight out of shared memory, probe the target
//     map's hash (4 lookups in flight per lane: only the probe latency remains), compact the
//     hits and stream them as rounds of 32 into their own 3-slot ring: point indices plus the
//     voxel records gathered cooperatively by cp.async (5 lanes per 80 B record), completion
//     signalled through an mbarrier;
//   * 4 consumer warps (the fp64 math saturates with 4 warps/SM, tools/microbench) each
//     serve 3 producer rings, one whole factor at a time, and reduce each factor's 29-value
//     partial in a fixed order (deterministic).
// Reference: match_terms (registration.py:146-157) + linearize_from_terms (:207-248) for every
// MatchingCostFactor of a graph (factor_graph.py:209-308, 522-536).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace vg {

constexpr int kSrcMax = 1024;
constexpr int kProducers = 12;
constexpr int kConsumers = 4;
constexpr int kRingsPerConsumer = kProducers / kConsumers;
constexpr int kSlots = 3;
constexpr int kSgUnroll = 4;
constexpr int kStageCap = 32 + 32 * kSgUnroll;  // pending hits of a producer
constexpr int kRecU = 5;                         // 16 B units gathered per voxel record

enum : int { kSgLast = 1, kSgGroupEnd = 2 };

struct __align__(16) SgMeta {
  double T[12];
  int factor;
  int nvalid;
  int flags;
  int total;
  int item_begin;
  int item_count;
  int pad[2];
};

struct __align__(16) SgSlot {
  float4 rec[32][kRecU];       // gathered voxel records (mean, covariance)
  unsigned short idx[32];      // source point index of each hit
  SgMeta meta;
};

struct __align__(16) SgProducer {
  SgSlot slot[kSlots];
  unsigned long long full[kSlots];
  unsigned long long empty[kSlots];
  int2 stage[kStageCap];       // (point, slot) hits not yet emitted
};

struct __align__(16) SgSmem {
  float4 pt[kSrcMax];
  double2 c0[kSrcMax];
  double2 c1[kSrcMax];
  double2 c2[kSrcMax];
  SgProducer prod[kProducers];
  int group;
};

__device__ __forceinline__ unsigned sg_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void sg_cp16(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sg_u32(smem)), "l"(gmem));
}
__device__ __forceinline__ void sg_bar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sg_u32(bar)), "r"(count));
}
__device__ __forceinline__ void sg_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sg_u32(bar)) : "memory");
}
__device__ __forceinline__ void sg_arrive_cp(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sg_u32(bar))
               : "memory");
}
__device__ __forceinline__ bool sg_test(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(sg_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void sg_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "SGW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra SGW_%=;\n"
      "}\n" ::"r"(sg_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void sg_named_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"((kProducers + kConsumers) * 32) : "memory");
}

// group start (all threads): publish the claimed group id, stage its source cloud
__device__ __forceinline__ void sg_group_stage(SgSmem& sm, const SrcGroup* __restrict__ groups,
                                               int n_groups) {
  sg_named_bar();  // group id (written by thread 0 before the barrier) visible
  const int g = sm.group;
  if (g >= n_groups) return;
  const SrcGroup grp = groups[g];
  constexpr int kThreads = (kProducers + kConsumers) * 32;
  for (int u = threadIdx.x; u < 4 * grp.n; u += kThreads) {
    const int arr = u / grp.n, i = u - arr * grp.n;
    if (arr == 0) sg_cp16(&sm.pt[i], grp.a + i);
    else if (arr == 1) sg_cp16(&sm.c0[i], grp.c0 + i);
    else if (arr == 2) sg_cp16(&sm.c1[i], grp.c1 + i);
    else sg_cp16(&sm.c2[i], grp.c2 + i);
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  sg_named_bar();  // source visible to every warp
}

// per-hit fp64 math with the source Gaussian read from shared memory
template <int MODE>
__device__ __forceinline__ void sg_hit_math(const SgSmem& sm, const SgSlot& sl, int lane,
                                            const double (&R)[9], const double (&t)[3],
                                            double (&acc)[28]) {
  const int i = sl.idx[lane];
  const float4 a = sm.pt[i];
  const double px = a.x, py = a.y, pz = a.z;
  const double2 s0 = sm.c0[i], s1 = sm.c1[i], s2 = sm.c2[i];
  const double2 m01 = *reinterpret_cast<const double2*>(&sl.rec[lane][0]);
  const double2 m2c0 = *reinterpret_cast<const double2*>(&sl.rec[lane][1]);
  const double2 c12 = *reinterpret_cast<const double2*>(&sl.rec[lane][2]);
  const double2 c34 = *reinterpret_cast<const double2*>(&sl.rec[lane][3]);
  const double v5 = reinterpret_cast<const double*>(&sl.rec[lane][4])[0];
  // moved point (registration.py:148) and residual d = mu' - moved (:152)
  const double x = fma(R[0], px, fma(R[1], py, R[2] * pz)) + t[0];
  const double y = fma(R[3], px, fma(R[4], py, R[5] * pz)) + t[1];
  const double z = fma(R[6], px, fma(R[7], py, R[8] * pz)) + t[2];
  const double d0 = m01.x - x, d1 = m01.y - y, d2 = m2c0.x - z;
  // F = C' + R C R^T (:153)
  const double C00 = s0.x, C01 = s0.y, C02 = s1.x, C11 = s1.y, C12 = s2.x, C22 = s2.y;
  double A[9];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const double r0 = R[3 * q], r1 = R[3 * q + 1], r2 = R[3 * q + 2];
    A[3 * q + 0] = fma(r0, C00, fma(r1, C01, r2 * C02));
    A[3 * q + 1] = fma(r0, C01, fma(r1, C11, r2 * C12));
    A[3 * q + 2] = fma(r0, C02, fma(r1, C12, r2 * C22));
  }
  auto arT = [&](int a_, int c_) {
    return fma(A[3 * a_], R[3 * c_], fma(A[3 * a_ + 1], R[3 * c_ + 1], A[3 * a_ + 2] * R[3 * c_ + 2]));
  };
  const double fa = m2c0.y + arT(0, 0), fb = c12.x + arT(0, 1), fc = c12.y + arT(0, 2);
  const double fd = c34.x + arT(1, 1), fe = c34.y + arT(1, 2), ff = v5 + arT(2, 2);
  // W = F^-1 (:113-130)
  const double i00 = fma(fd, ff, -fe * fe), i01 = fma(fc, fe, -fb * ff),
               i02 = fma(fb, fe, -fc * fd), i11 = fma(fa, ff, -fc * fc),
               i12 = fma(fb, fc, -fa * fe), i22 = fma(fa, fd, -fb * fb);
  const double inv = rcp64(fma(fa, i00, fma(fb, i01, fc * i02)));
  const double W00 = i00 * inv, W01 = i01 * inv, W02 = i02 * inv, W11 = i11 * inv,
               W12 = i12 * inv, W22 = i22 * inv;
  const double wd0 = fma(W00, d0, fma(W01, d1, W02 * d2));
  const double wd1 = fma(W01, d0, fma(W11, d1, W12 * d2));
  const double wd2 = fma(W02, d0, fma(W12, d1, W22 * d2));
  acc[27] += fma(d0, wd0, fma(d1, wd1, d2 * wd2));  // cost (:156)
  if (MODE == 0) {
    const double vx = x - t[0], vy = y - t[1], vz = z - t[2];
    // N = hat(x') W, P = N hat(x')^T, b' = [x' x Wd ; Wd]  (J' = [-hat(x') | I])
    const double N00 = fma(-vz, W01, vy * W02), N01 = fma(-vz, W11, vy * W12),
                 N02 = fma(-vz, W12, vy * W22);
    const double N10 = fma(vz, W00, -vx * W02), N11 = fma(vz, W01, -vx * W12),
                 N12 = fma(vz, W02, -vx * W22);
    const double N20 = fma(-vy, W00, vx * W01), N21 = fma(-vy, W01, vx * W11),
                 N22 = fma(-vy, W02, vx * W12);
    acc[0] += fma(-vz, N01, vy * N02);
    acc[1] += fma(vz, N00, -vx * N02);
    acc[2] += fma(-vy, N00, vx * N01);
    acc[3] += fma(vz, N10, -vx * N12);
    acc[4] += fma(-vy, N10, vx * N11);
    acc[5] += fma(-vy, N20, vx * N21);
    acc[6] += N00; acc[7] += N01; acc[8] += N02;
    acc[9] += N10; acc[10] += N11; acc[11] += N12;
    acc[12] += N20; acc[13] += N21; acc[14] += N22;
    acc[15] += W00; acc[16] += W01; acc[17] += W02;
    acc[18] += W11; acc[19] += W12; acc[20] += W22;
    acc[21] += fma(vy, wd2, -vz * wd1);
    acc[22] += fma(vz, wd0, -vx * wd2);
    acc[23] += fma(vx, wd1, -vy * wd0);
    acc[24] += wd0; acc[25] += wd1; acc[26] += wd2;
  }
}

// producer: emit one round of n (<= 32) staged hits starting at stage[0] into the ring
__device__ __forceinline__ void sg_emit(SgProducer& pr, unsigned& cur, const MapView& mv,
                                       const double (&T)[12], int factor, int n, int flags,
                                       int total, int item_begin, int item_count, int lane) {
  const unsigned slot = cur % kSlots;
  sg_wait(&pr.empty[slot], ((cur / kSlots) & 1) ^ 1);
  SgSlot& sl = pr.slot[slot];
  if (lane < 12) sl.meta.T[lane] = T[lane];
  if (lane == 12) sl.meta.factor = factor;
  if (lane == 13) sl.meta.nvalid = n;
  if (lane == 14) sl.meta.flags = flags;
  if (lane == 15) sl.meta.total = total;
  if (lane == 16) sl.meta.item_begin = item_begin;
  if (lane == 17) sl.meta.item_count = item_count;
  const int2 e = pr.stage[lane < n ? lane : 0];
  if (lane < n) sl.idx[lane] = (unsigned short)e.x;
#pragma unroll
  for (int c = 0; c < kRecU; ++c) {
    const int u = c * 32 + lane;
    const int q = u / kRecU, j = u - q * kRecU;
    const int rec = __shfl_sync(0xffffffffu, e.y, q);
    if (q < n) sg_cp16(&sl.rec[q][j], reinterpret_cast<const char*>(mv.recs + rec) + 16 * j);
  }
  __syncwarp();
  sg_arrive_cp(&pr.full[slot]);
  if (lane == 0) sg_arrive(&pr.full[slot]);
  ++cur;
}

template <int MODE>
__global__ void __launch_bounds__((kProducers + kConsumers) * 32, 1)
    k_srcgroup(const SrcGroup* __restrict__ groups, int n_groups,
               const int* __restrict__ group_factors, const FactorDev* __restrict__ factors,
               const MapView* __restrict__ maps, int* __restrict__ counter,
               double* __restrict__ partials) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SgSmem& sm = *reinterpret_cast<SgSmem*>(smem_raw);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x < kProducers * kSlots) {
    SgProducer& pr = sm.prod[threadIdx.x / kSlots];
    sg_bar_init(&pr.full[threadIdx.x % kSlots], 33);  // 32 cp.async arrivals + 1 metadata
    sg_bar_init(&pr.empty[threadIdx.x % kSlots], 1);
  }
  __syncthreads();
  // Roles run separate loops (register budgets differ: setmaxnreg moves registers from the
  // 12 producer warps to the 4 consumer warps); groups are delimited by the named barrier 1.
  if (warp < kProducers) {
    // SMR_DEC
    SgProducer& pr = sm.prod[warp];
    const unsigned lt_mask = (1u << lane) - 1u;
    unsigned cur = 0;  // ring cursor (persists across groups)
    for (;;) {
      if (threadIdx.x == 0) sm.group = atomicAdd(counter, 1);
      sg_group_stage(sm, groups, n_groups);
      const int g = sm.group;
      if (g >= n_groups) break;
      const SrcGroup grp = groups[g];
      for (int fk = warp; fk < grp.fcount; fk += kProducers) {
        const int f = group_factors[grp.fbegin + fk];
        const FactorDev& fd = factors[f];
        double T[12];
#pragma unroll
        for (int q = 0; q < 12; ++q) T[q] = __ldg(fd.T + q);
        const MapView mv = maps[__ldg(&fd.map)];
        const int item_begin = __ldg(&fd.item_begin), item_count = __ldg(&fd.item_count);
        int staged = 0, total = 0;
        for (int base = 0; base < grp.n; base += 32 * kSgUnroll) {
          Query qy[kSgUnroll];
          ProbeGroup pg[kSgUnroll];
          bool live[kSgUnroll];
#pragma unroll
          for (int u = 0; u < kSgUnroll; ++u) {
            const int i = base + 32 * u + lane;
            const float4 a = sm.pt[min(i, grp.n - 1)];
            const double px = a.x, py = a.y, pz = a.z;
            // points @ R^T + t (registration.py:148), keys (preprocess.py:68-70)
            const double x = fma(T[0], px, fma(T[1], py, T[2] * pz)) + T[9];
            const double y = fma(T[3], px, fma(T[4], py, T[5] * pz)) + T[10];
            const double z = fma(T[6], px, fma(T[7], py, T[8] * pz)) + T[11];
            qy[u] = make_query(mv, floor_div(x, mv.res, mv.inv_res, mv.pow2),
                               floor_div(y, mv.res, mv.inv_res, mv.pow2),
                               floor_div(z, mv.res, mv.inv_res, mv.pow2), 1);
            live[u] = i < grp.n && mv.m && qy[u].inside;
            if (live[u]) pg[u] = probe_load(mv, qy[u].bucket, 1);
          }
#pragma unroll
          for (int u = 0; u < kSgUnroll; ++u) {
            int slot = -1;
            if (live[u]) {
              unsigned bk = qy[u].bucket;
              int r;
              while ((r = probe_scan(mv, pg[u], bk, qy[u], slot, 1)) < 0) {
                bk = next_bucket(bk, mv);
                pg[u] = probe_load(mv, bk, 1);
              }
              if (r != 1) slot = -1;
            }
            // misses contribute nothing (registration.py:150-156)
            const unsigned m = __ballot_sync(0xffffffffu, slot >= 0);
            if (slot >= 0)
              pr.stage[staged + __popc(m & lt_mask)] = make_int2(base + 32 * u + lane, slot);
            staged += __popc(m);
            total += __popc(m);
          }
          __syncwarp();
          // emit full rounds; the factor's last round is emitted after the final chunk
          const bool final_chunk = base + 32 * kSgUnroll >= grp.n;
          while (staged > 32 || (staged == 32 && !final_chunk)) {
            sg_emit(pr, cur, mv, T, f, 32, 0, total, item_begin, item_count, lane);
            const int rem = staged - 32;  // shift the remaining staged hits to the front
            int2 v[kSgUnroll];
#pragma unroll
            for (int q = 0; q < kSgUnroll; ++q)
              if (32 * q + lane < rem) v[q] = pr.stage[32 + 32 * q + lane];
            __syncwarp();
#pragma unroll
            for (int q = 0; q < kSgUnroll; ++q)
              if (32 * q + lane < rem) pr.stage[32 * q + lane] = v[q];
            __syncwarp();
            staged = rem;
          }
        }
        // last (possibly empty) round closes the factor
        sg_emit(pr, cur, mv, T, f, staged, kSgLast, total, item_begin, item_count, lane);
      }
      // group end marker for the consumer
      {
        const unsigned slot = cur % kSlots;
        sg_wait(&pr.empty[slot], ((cur / kSlots) & 1) ^ 1);
        if (lane == 0) pr.slot[slot].meta.flags = kSgGroupEnd;
        __syncwarp();
        sg_arrive_cp(&pr.full[slot]);
        if (lane == 0) sg_arrive(&pr.full[slot]);
        ++cur;
      }
      sg_named_bar();  // group done (consumers drained their rings)
    }
  } else {
    // SMR_INC
    const int c = warp - kProducers;
    static_assert(kRingsPerConsumer == 3, "ring selects below assume 3 rings per consumer");
    unsigned cur0 = 0, cur1 = 0, cur2 = 0;  // per-ring cursors (selects, no local memory)
    for (;;) {
      sg_group_stage(sm, groups, n_groups);
      if (sm.group >= n_groups) break;
      // Rounds are taken from whichever ring is ready (non-blocking polling), so all three
      // producers stay busy.  Each round is reduced across the warp (fixed butterfly) and
      // added, in ring order, to that ring's running factor sum: lane L holds component L.
      double run0 = 0.0, run1 = 0.0, run2 = 0.0;
      int done_mask = 0;
      while (done_mask != 7) {
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          if (done_mask & (1 << r)) continue;
          SgProducer& pr = sm.prod[c + kConsumers * r];
          const unsigned cr = r == 0 ? cur0 : (r == 1 ? cur1 : cur2);
          const unsigned slot = cr % kSlots;
          if (!sg_test(&pr.full[slot], (cr / kSlots) & 1)) continue;
          if (r == 0) ++cur0;
          else if (r == 1) ++cur1;
          else ++cur2;
          const SgSlot& sl = pr.slot[slot];
          const int flags = sl.meta.flags;
          if (flags & kSgGroupEnd) {
            __syncwarp();
            if (lane == 0) sg_arrive(&pr.empty[slot]);
            done_mask |= 1 << r;
            continue;
          }
          const int nvalid = sl.meta.nvalid;
          const int factor_item = sl.meta.item_begin, nitems = sl.meta.item_count;
          double R[9], t[3];
#pragma unroll
          for (int q = 0; q < 9; ++q) R[q] = sl.meta.T[q];
#pragma unroll
          for (int q = 0; q < 3; ++q) t[q] = sl.meta.T[9 + q];
          double acc[28];
#pragma unroll
          for (int q = 0; q < 28; ++q) acc[q] = 0.0;
          if (lane < nvalid) sg_hit_math<MODE>(sm, sl, lane, R, t, acc);
          __syncwarp();
          if (lane == 0) sg_arrive(&pr.empty[slot]);  // slot consumed
          double rv;
          if (MODE == 1) {
            double cc = acc[27];
#pragma unroll
            for (int q = 16; q >= 1; q >>= 1) cc += __shfl_xor_sync(0xffffffffu, cc, q);
            rv = lane == 0 ? cc : (lane == 1 ? (double)nvalid : 0.0);
          } else {
            double v[32];
#pragma unroll
            for (int q = 0; q < 28; ++q) v[q] = acc[q];
            v[28] = lane == 0 ? (double)nvalid : 0.0;
            v[29] = 0.0;
            v[30] = 0.0;
            v[31] = 0.0;
            rv = warp_transpose_reduce32(v, lane);
          }
          double run = (r == 0 ? run0 : (r == 1 ? run1 : run2)) + rv;
          if (flags & kSgLast) {
            if (MODE == 1) {
              if (lane < 2) partials[2 * (size_t)factor_item + lane] = run;
              if (lane < 2)
                for (int it = 1; it < nitems; ++it) partials[2 * (size_t)(factor_item + it) + lane] = 0.0;
            } else {
              partials[(size_t)factor_item * kPartialStride + lane] = run;
              for (int it = 1; it < nitems; ++it)
                partials[(size_t)(factor_item + it) * kPartialStride + lane] = 0.0;
            }
            run = 0.0;
          }
          if (r == 0) run0 = run;
          else if (r == 1) run1 = run;
          else run2 = run;
        }
      }
      sg_named_bar();  // group done
    }
  }
}

}  // namespace vg

using namespace vg;

size_t srcgroup_smem_bytes() { return sizeof(SgSmem); }
int srcgroup_max_points() { return kSrcMax; }

int launch_srcgroup(vg_ctx* ctx, vg_batch* b, int kmode) {
  static int sms = 0;
  if (!sms) VG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
  const size_t smem = sizeof(SgSmem);
  VG_CUDA(cudaMemsetAsync(b->work_counter, 0, sizeof(int), ctx->stream));
  const int grid = std::min(sms, b->num_groups);
  auto go = [&](auto kern) -> int {
    VG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, (kProducers + kConsumers) * 32, smem, ctx->stream>>>(
        b->groups, b->num_groups, b->group_factors, b->factors, b->maps, b->work_counter,
        b->partials);
    return 0;
  };
  const int rc = kmode == 1 ? go(k_srcgroup<1>) : go(k_srcgroup<0>);
  if (rc) return rc;
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  return 0;
}
