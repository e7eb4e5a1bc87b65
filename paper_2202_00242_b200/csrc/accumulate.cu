// accumulate.cu — K4a (correspondence lookup + per-item hit compaction) and K4b (fp64 fused
// covariance / inverse / Jacobian accumulation over compacted hits).
//
// Reference: match_terms (registration.py:146-157) + linearize_from_terms (:207-248) for
// every factor of a graph (factor_graph.py:522-536).
//
// K4a — one warp per (factor, <=512-point chunk) item, light on registers so many warps hide
//   the two dependent memory latencies of a lookup (source point, then the probed key
//   bucket).  x = R p + t (fp64) -> key (bit-exact floor) -> one 16 B bucket of 4 local keys.
//   Hits are written as (point, record) pairs into the item's region of a batch-wide hit
//   list with a warp ballot, preserving point order.  Misses contribute nothing (:150-156).
// K4b — one warp per item over its compacted hits, so every lane of the expensive fp64 path
//   does useful work.  Each round of 32 hits gathers the source point (16 B), source
//   covariance or its plane form (48 B) and voxel record (80 B) with cp.async into a 2-stage
//   shared-memory pipeline, so the gathers of round r+1 are in flight while round r computes
//   (hit entries are loaded two rounds ahead).
//   The per-item 29-value partial (target-frame 6x6 about the source origin)
//   is reduced across the warp in a fixed order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace vg {

// ---- K4a ------------------------------------------------------------------------------------
// One warp per CTA for K4a and K4b: an SM slot is released as soon as its item finishes
// (with 4-8 warp CTAs the slot waits for the CTA's slowest item; measured 12% slower for K4a,
// 7% for K4b).  Residency is set through the min-CTAs launch bound: 32 (K4a fast path,
// 64 registers), 24 (K4a generic), 12 (K4b, <= 170 registers).
// 1: K4a bucket probes with L1::no_allocate (measured 1.33x slower: consecutive points
// share bucket lines, so the probes' L1 allocation pays)
// K4b occupancy bound (one-warp CTAs): at 15 ptxas fits the per-hit math in 126 registers
// without spills, so 16 warps are resident per SM instead of 12 at 160 registers (config 5:
// K4 0.413 -> 0.394 ms; 13/14/16 measured 0.396/0.396/0.407, 18 spills)
#ifndef VG_K4B_MINB
#define VG_K4B_MINB 15
#endif
#ifndef VG_K4B_STAGES
#define VG_K4B_STAGES 2  // shared-memory ring depth of the fast-path linearize K4b
#endif
#ifndef VG_K4B_MINB_GEN
#define VG_K4B_MINB_GEN 15
#endif
#ifndef VG_K4B_MINB_COST
#define VG_K4B_MINB_COST 12
#endif
#ifndef VG_PROBE_NA
#define VG_PROBE_NA 0
#endif
#ifndef VG_K4A_WARPS
#define VG_K4A_WARPS 1
#endif
constexpr int kLookupWarps = VG_K4A_WARPS;

// KM: 1 = every map of the batch uses 32-bit local keys, 0 = all int64, 2 = mixed (runtime)
// P2: every map of the batch has a power-of-two resolution (x * (1/res) is exact)
template <int KM, int kMinBlocks, int P2 = 0>
__global__ void __launch_bounds__(kLookupWarps * 32, kMinBlocks)
    k_lookup_items(const ItemDev* __restrict__ items, int n_items,
                   const FactorDev* __restrict__ factors, const CloudView* __restrict__ clouds,
                   const MapView* __restrict__ maps, int2* __restrict__ hits,
                   int* __restrict__ counts, double* __restrict__ partials2,
                   AccDesc* __restrict__ descs) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * kLookupWarps + (threadIdx.x >> 5);
  if (w >= n_items) return;
  const ItemDev it = items[w];
  const FactorDev* f = factors + it.factor;
  double R[9], t[3];
#pragma unroll
  for (int k = 0; k < 9; ++k) R[k] = __ldg(f->T + k);
#pragma unroll
  for (int k = 0; k < 3; ++k) t[k] = __ldg(f->T + 9 + k);
  const CloudView cv = clouds[__ldg(&f->cloud)];
  const MapView mv = maps[__ldg(&f->map)];
  const int kmode = KM == 2 ? mv.kmode : KM;
  if (descs) {
    AccDesc& d = descs[w];
    double tv = 0.0;  // static register indexing (no local-memory copy of R)
#pragma unroll
    for (int k = 0; k < 9; ++k)
      if (lane == k) tv = R[k];
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (lane == 9 + k) tv = t[k];
    if (lane < 12) d.T[lane] = tv;
    else if (lane == 12) d.a = cv.a;
    else if (lane == 13) d.xyz64 = cv.xyz64;
    else if (lane == 14) d.c0 = cv.c0;
    else if (lane == 15) d.c1 = cv.c1;
    else if (lane == 16) d.c2 = cv.c2;
    else if (lane == 17) d.recs = mv.recs;
    else if (lane == 18) d.hoff = it.hoff;
  }
  const unsigned lt_mask = (1u << lane) - 1u;
  int2* out = hits + it.hoff;
  int cnt = 0;
  // the next iteration's source point is loaded before this iteration's probe is resolved,
  // so the two dependent latencies of consecutive iterations overlap
  const int last = it.end - 1;
  auto load_pt = [&](int i, double& px, double& py, double& pz) {
    const int ic = min(i, last);
    if (cv.xyz64) {
      px = __ldg(cv.xyz64 + 3 * (size_t)ic);
      py = __ldg(cv.xyz64 + 3 * (size_t)ic + 1);
      pz = __ldg(cv.xyz64 + 3 * (size_t)ic + 2);
    } else {
      const float4 a = __ldg(cv.a + ic);
      px = a.x;
      py = a.y;
      pz = a.z;
    }
  };
  // transform + key of point i (clamped into the item), probe of its home bucket
  auto make_q = [&](double px, double py, double pz) {
    // points @ R^T + t (registration.py:148), keys (preprocess.py:68-70)
    const double x = fma(R[0], px, fma(R[1], py, R[2] * pz)) + t[0];
    const double y = fma(R[3], px, fma(R[4], py, R[5] * pz)) + t[1];
    const double z = fma(R[6], px, fma(R[7], py, R[8] * pz)) + t[2];
    const double fx = P2 ? floor(x * mv.inv_res) : floor_div(x, mv.res, mv.inv_res, mv.pow2);
    const double fy = P2 ? floor(y * mv.inv_res) : floor_div(y, mv.res, mv.inv_res, mv.pow2);
    const double fz = P2 ? floor(z * mv.inv_res) : floor_div(z, mv.res, mv.inv_res, mv.pow2);
    return KM == 1 ? make_query_local(mv, fx, fy, fz) : make_query(mv, fx, fy, fz, kmode);
  };
  // Two-deep software pipeline per lane: the probe of iteration k+1 is in flight while
  // iteration k's probe is resolved, and the point of iteration k+2 is being loaded.
  double px, py, pz, nx, ny, nz;
  load_pt(it.begin + lane, px, py, pz);
  load_pt(it.begin + 32 + lane, nx, ny, nz);
  Query q0 = make_q(px, py, pz);
  bool live0 = it.begin + lane < it.end && mv.m && q0.inside;
  ProbeGroup g0;
  if (live0) g0 = probe_load(mv, q0.bucket, kmode);
  for (int base = it.begin; base < it.end; base += 32) {
    const int i = base + lane;
    // issue iteration k+1
    const Query q1 = make_q(nx, ny, nz);
    const bool live1 = i + 32 < it.end && mv.m && q1.inside;
    ProbeGroup g1;
    if (live1) g1 = probe_load(mv, q1.bucket, kmode);
    load_pt(i + 64, nx, ny, nz);
    // resolve iteration k
    int slot = -1;
    if (live0) {
      unsigned bk = q0.bucket;
      int r;
      while ((r = probe_scan(mv, g0, bk, q0, slot, kmode)) < 0) {
        bk = next_bucket(bk, mv);
        g0 = probe_load(mv, bk, kmode);
      }
      if (r == 1) slot = rec_index(mv, slot, kmode);
      else slot = -1;
    }
    // misses contribute nothing (registration.py:150-156)
    const unsigned m = __ballot_sync(0xffffffffu, slot >= 0);
    if (slot >= 0) out[cnt + __popc(m & lt_mask)] = make_int2(i, slot);
    cnt += __popc(m);
    q0 = q1;
    live0 = live1;
    g0 = g1;
  }
  if (lane == 0) {
    counts[w] = cnt;
    if (partials2) {  // inliers-only mode: the item's record is final
      partials2[2 * (size_t)w] = 0.0;
      partials2[2 * (size_t)w + 1] = (double)cnt;
    }
  }
  if (descs && lane == 0) descs[w].n = cnt;
}

#ifndef VG_HITS_NA
#define VG_HITS_NA 0
#endif
#ifndef VG_HITS_CS
#define VG_HITS_CS 0
#endif
#ifndef VG_PTS_NA
#define VG_PTS_NA 0
#endif
// cache-policy variants of the streaming accesses (read or written once), all measured on
// config 5 and left off: hit-entry loads with L1::no_allocate / hit stores with .cs change
// nothing (K4 0.4127 ms either way); K4a point loads with L1::no_allocate cost 1.2x (K4a)
__device__ __forceinline__ int2 ld_hit(const int2* p) {
#if VG_HITS_NA
  int2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}
__device__ __forceinline__ void st_hit(int2* p, int2 v) {
#if VG_HITS_CS
  asm volatile("st.global.cs.v2.s32 [%0], {%1, %2};" ::"l"(p), "r"(v.x), "r"(v.y));
#else
  *p = v;
#endif
}
__device__ __forceinline__ float4 ld_pt(const float4* p) {
#if VG_PTS_NA
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}

// K4a fast path: every map uses 32-bit local keys and a power-of-two resolution, every
// source point is fp32-exact.  The item header (T_ij + views, refreshed by K-compose) is read
// in one dependent step instead of item -> factor -> cloud/map views.
template <int kMinBlocks>
__global__ void __launch_bounds__(kLookupWarps * 32, kMinBlocks)
    k_lookup_fast(const ItemHdr* __restrict__ hdrs, int n_items, int2* __restrict__ hits,
                  int* __restrict__ counts, double* __restrict__ partials2,
                  AccDesc* __restrict__ descs) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * kLookupWarps + (threadIdx.x >> 5);
  pdl_release();
  pdl_wait();  // item headers carry T_ij written by K-compose
  if (w >= n_items) return;
  const ItemHdr* h = hdrs + w;
  double R[9], t[3];
#pragma unroll
  for (int k = 0; k < 9; ++k) R[k] = __ldg(h->T + k);
#pragma unroll
  for (int k = 0; k < 3; ++k) t[k] = __ldg(h->T + 9 + k);
  const float4* pa = (const float4*)__ldg((const unsigned long long*)&h->a);
  const unsigned* keys32 = (const unsigned*)__ldg((const unsigned long long*)&h->mv.keys32);
  const double inv_res = __ldg(&h->mv.inv_res);
  const int shift = __ldg(&h->mv.shift);
  const unsigned mask = __ldg(&h->mv.mask);
  const int m = __ldg(&h->mv.m);
  const int bx = __ldg(&h->mv.bx), by = __ldg(&h->mv.by), bz = __ldg(&h->mv.bz);
  const int ex = __ldg(&h->mv.ex), ey = __ldg(&h->mv.ey), ez = __ldg(&h->mv.ez);
  const int begin = __ldg(&h->begin), end = __ldg(&h->end), hoff = __ldg(&h->hoff);
  if (descs) {
    AccDesc& d = descs[w];
    if (lane < 12) d.T[lane] = __ldg(h->T + lane);
    else if (lane == 12) d.a = pa;
    else if (lane == 13) d.xyz64 = nullptr;
    else if (lane == 14) d.c0 = (const double2*)__ldg((const unsigned long long*)&h->c0);
    else if (lane == 15) d.c1 = (const double2*)__ldg((const unsigned long long*)&h->c1);
    else if (lane == 16) d.c2 = (const double2*)__ldg((const unsigned long long*)&h->c2);
    else if (lane == 17) d.recs = (const VoxelRec*)__ldg((const unsigned long long*)&h->mv.recs);
    else if (lane == 18) d.hoff = hoff;
  }
  const unsigned lt_mask = (1u << lane) - 1u;
  int2* out = hits + hoff;
  int cnt = 0;
  const int last = end - 1;
  struct Q {
    unsigned k32, bucket;
    bool live;
  };
  auto make_q = [&](float4 a, int i) {
    const double px = a.x, py = a.y, pz = a.z;
    // points @ R^T + t (registration.py:148); floor(p / res) exact for power-of-two res
    const double x = fma(R[0], px, fma(R[1], py, R[2] * pz)) + t[0];
    const double y = fma(R[3], px, fma(R[4], py, R[5] * pz)) + t[1];
    const double z = fma(R[6], px, fma(R[7], py, R[8] * pz)) + t[2];
    const double qx = x * inv_res, qy = y * inv_res, qz = z * inv_res;
    // floor in the convert (F2I.FLOOR, saturating), range-checked as integers
    const int ix = __double2int_rd(qx), iy = __double2int_rd(qy), iz = __double2int_rd(qz);
    Q q;
    q.live = false;
    q.k32 = 0;
    q.bucket = 0;
    if ((unsigned)(ix + 1048575) < 2097151u && (unsigned)(iy + 1048575) < 2097151u &&
        (unsigned)(iz + 1048575) < 2097151u) {
      // |floor| < 2^20: the reference's pack/unpack round trip is the identity
      const unsigned lx = (unsigned)(ix - bx);
      const unsigned ly = (unsigned)(iy - by);
      const unsigned lz = (unsigned)(iz - bz);
      q.live = lx < (unsigned)ex && ly < (unsigned)ey && lz < (unsigned)ez;
      q.k32 = lx | (ly << 11) | (lz << 22);
    } else {
      MapView mv;
      mv.bx = bx; mv.by = by; mv.bz = bz; mv.ex = ex; mv.ey = ey; mv.ez = ez; mv.shift = shift;
      const Query qq = make_query(mv, floor(qx), floor(qy), floor(qz), 1);
      q.live = qq.inside;
      q.k32 = qq.k32;
    }
    q.bucket = bucket32(q.k32, shift);
    q.live = q.live && i < end && m > 0;
    return q;
  };
  auto load_bucket = [&](unsigned bucket, unsigned (&g)[4]) {
#if VG_PROBE_NA
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(keys32 + (size_t)bucket * kBucket32));
#else
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(keys32 + (size_t)bucket * kBucket32));
#endif
    g[0] = v.x;
    g[1] = v.y;
    g[2] = v.z;
    g[3] = v.w;
  };
  // resolve the probe of one round (overflowing buckets continue into the next) and append
  // its hits in point order
  auto resolve = [&](const Q& q, unsigned (&g)[4], int i) {
    int slot = -1;
    if (q.live) {
      unsigned bk = q.bucket;
      for (unsigned probes = 0;; ++probes) {
        VG_DEVICE_CHECK(probes <= mask, "K4a: every bucket visited");
        int found = -1;
        bool empty = false;
#pragma unroll
        for (int j = kBucket32 - 1; j >= 0; --j) {
          if (g[j] == q.k32) found = j;
          empty |= (g[j] == kEmpty32);
        }
        if (found >= 0) {
          slot = (int)(bk * kBucket32 + found);
          break;
        }
        if (empty) break;
        bk = (bk + 1) & mask;
        load_bucket(bk, g);
      }
    }
    // misses contribute nothing (registration.py:150-156)
    const unsigned mb = __ballot_sync(0xffffffffu, slot >= 0);
    VG_DEVICE_CHECK(cnt + __popc(mb) <= end - begin, "K4a: hits overflow the item region");
    VG_DEVICE_CHECK(slot < 0 || (i >= begin && i < end), "K4a: hit outside the item");
    VG_DEVICE_CHECK(slot < (int)((mask + 1) * kBucket32), "K4a: slot out of the table");
    if (slot >= 0) st_hit(out + cnt + __popc(mb & lt_mask), make_int2(i, slot));
    cnt += __popc(mb);
  };
  // Two-deep pipeline, unrolled by two with ping-pong registers (A: even rounds, B: odd):
  // the probe of the next round and the point of the round after are in flight while a
  // round resolves, and no in-flight load result is ever copied (a copy would wait for it).
  float4 pA = ld_pt(pa + min(begin + lane, last));
  float4 pB = ld_pt(pa + min(begin + 32 + lane, last));
  Q qA = make_q(pA, begin + lane);
  unsigned gA[4] = {0, 0, 0, 0}, gB[4] = {0, 0, 0, 0};
  if (qA.live) load_bucket(qA.bucket, gA);
  pA = ld_pt(pa + min(begin + 64 + lane, last));
  for (int base = begin; base < end; base += 64) {
    const int i = base + lane;
    const Q qB = make_q(pB, i + 32);
    if (qB.live) load_bucket(qB.bucket, gB);
    pB = ld_pt(pa + min(i + 96, last));
    resolve(qA, gA, i);
    if (base + 32 >= end) break;
    qA = make_q(pA, i + 64);
    if (qA.live) load_bucket(qA.bucket, gA);
    pA = ld_pt(pa + min(i + 128, last));
    resolve(qB, gB, i + 32);
  }
  if (lane == 0) {
    counts[w] = cnt;
    if (partials2) {
      partials2[2 * (size_t)w] = 0.0;
      partials2[2 * (size_t)w + 1] = (double)cnt;
    }
    if (descs) descs[w].n = cnt;
  }
}

// ---- K4b ------------------------------------------------------------------------------------
constexpr int kAccWarps = 1;  // see kLookupWarps

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

// bit 0: voxel-record gathers bypass L1 (cp.async.cg; K4 0.417 -> 0.411 ms, cost mode -10%:
// records have no L1 reuse and their lines evicted the lane-own gathers' and hit entries');
// bit 1: the lane-own gathers too (either bit alone measures the same, both slower: 0.437)
#ifndef VG_CG_MASK
#define VG_CG_MASK 1
#endif
// L2-only variant (no L1 allocation) for gathers without L1 reuse
__device__ __forceinline__ void cp_async16_cg(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
template <int kBit>
__device__ __forceinline__ void cp_async16_sel(void* smem, const void* gmem) {
  if (VG_CG_MASK & kBit) cp_async16_cg(smem, gmem);
  else cp_async16(smem, gmem);
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// per-warp stage: own point (1-2 x 16 B, fp32 or fp64 xyz), own source covariance (3 x 16 B),
// and 32 voxel records gathered cooperatively (5 x 16 B each; the 80 B lane stride is 20
// banks, so 8 lanes of a 16 B shared-memory read hit 8 distinct 4-bank groups: conflict free)
#ifndef VG_K4A_MINB
#define VG_K4A_MINB 32
#endif
constexpr int kRecUnits = 5;
constexpr int kRecStride = 5;
// PT: 16 B point units per lane — 2 (fp64 xyz possible) or 1 (every point fp32-exact)
template <int PT>
struct AccStageT {
  float4 pt[PT][32];
  float4 cov[3][32];
  float4 rec[32][kRecStride];
};
using AccStage = AccStageT<2>;
template <int kStages, int PT = 2>
struct AccSmem {
  AccStageT<PT> stage[kStages];
};

// Gather one round (32 hits; the last round of an item pads with replays of its last hit) into
// stage `round % kStages`.  Point and covariance rows are
// lane-own (hits are in point order, so these are nearly coalesced); the random 80 B voxel
// records are gathered cooperatively: each cp.async instruction covers 32 consecutive 16 B
// units of 6-7 records instead of one unit of 32 records, cutting L1 wavefronts ~4x.
// Always commits one group so every lane has the same number of outstanding groups.
template <int kStages, int PT = 2>
__device__ __forceinline__ void issue_round(const CloudView& cv, const MapView& mv,
                                            AccSmem<kStages, PT>& sm, int round, int2 e,
                                            int nvalid, int lane, bool own = true) {
  AccStageT<PT>& st = sm.stage[round % kStages];
  if (lane < nvalid && own) {
    if (PT == 2 && cv.xyz64) {
      const double* p = cv.xyz64 + 3 * (size_t)e.x;
      double* d = reinterpret_cast<double*>(&st.pt[0][lane]);
      cp_async8(d, p);
      cp_async8(d + 1, p + 1);
      cp_async8(reinterpret_cast<double*>(&st.pt[PT - 1][lane]), p + 2);
    } else {
      cp_async16_sel<2>(&st.pt[0][lane], cv.a + e.x);
    }
    cp_async16_sel<2>(&st.cov[0][lane], cv.c0 + e.x);
    cp_async16_sel<2>(&st.cov[1][lane], cv.c1 + e.x);
    cp_async16_sel<2>(&st.cov[2][lane], cv.c2 + e.x);
  }
#pragma unroll
  for (int c = 0; c < kRecUnits; ++c) {
    const int u = c * 32 + lane;
    const int q = u / kRecUnits, j = u - q * kRecUnits;
    const int row = __shfl_sync(0xffffffffu, e.y, q);
    if (q < nvalid)
      cp_async16_sel<1>(&st.rec[q][j], reinterpret_cast<const char*>(mv.recs + row) + 16 * j);
  }
  cp_async_commit();
}

template <int MODE, int PLANE>
__device__ __forceinline__ void hit_core(double px, double py, double pz, double2 s0,
                                         double2 s1, double2 s2, const float4* rec,
                                         const double (&R)[9], const double (&t)[3],
                                         double scale, double (&acc)[28]);

// per-hit fp64 math of K4b on one staged hit: moved point, residual, fused covariance and its
// inverse, cost, and the target-frame Jacobian blocks about the source origin
template <int MODE, int PT = 2, int PLANE = 0>
__device__ __forceinline__ void hit_math(const AccStageT<PT>& st, int lane, bool f64pts,
                                         const double (&R)[9], const double (&t)[3],
                                         double scale, double (&acc)[28]) {
  double px, py, pz;
  if (PT == 2 && f64pts) {
    const double* d = reinterpret_cast<const double*>(&st.pt[0][lane]);
    px = d[0];
    py = d[1];
    pz = reinterpret_cast<const double*>(&st.pt[PT - 1][lane])[0];
  } else {
    const float4 a = st.pt[0][lane];
    px = a.x;
    py = a.y;
    pz = a.z;
  }
  const double2 s0 = *reinterpret_cast<const double2*>(&st.cov[0][lane]);
  const double2 s1 = *reinterpret_cast<const double2*>(&st.cov[1][lane]);
  const double2 s2 = *reinterpret_cast<const double2*>(&st.cov[2][lane]);
  hit_core<MODE, PLANE>(px, py, pz, s0, s1, s2, st.rec[lane], R, t, scale, acc);
}

// the math of one hit from its source point, source covariance rows (PLANE: the plane form
// (n0, n1), (n2, kappa), (alpha, 0), map_build.cu) and staged voxel record
template <int MODE, int PLANE>
__device__ __forceinline__ void hit_core(double px, double py, double pz, double2 s0,
                                         double2 s1, double2 s2, const float4* rec,
                                         const double (&R)[9], const double (&t)[3],
                                         double scale, double (&acc)[28]) {
  const double2 m01 = *reinterpret_cast<const double2*>(&rec[0]);
  const double2 m2c0 = *reinterpret_cast<const double2*>(&rec[1]);
  const double2 c12 = *reinterpret_cast<const double2*>(&rec[2]);
  const double2 c34 = *reinterpret_cast<const double2*>(&rec[3]);
  const double v5 = reinterpret_cast<const double*>(&rec[4])[0];
  // moved point (registration.py:148) and residual d = mu' - moved (:152); the lever arm
  // about the source origin is x' = R p
  const double vx = fma(R[0], px, fma(R[1], py, R[2] * pz));
  const double vy = fma(R[3], px, fma(R[4], py, R[5] * pz));
  const double vz = fma(R[6], px, fma(R[7], py, R[8] * pz));
  const double d0 = m01.x - (vx + t[0]), d1 = m01.y - (vy + t[1]), d2 = m2c0.x - (vz + t[2]);
  // F = C' + R C R^T (:153)
  double fa, fb, fc, fd, fe, ff;
  if (PLANE) {
    // R C R^T = alpha I - kappa m m^T, m = R n
    const double n0 = s0.x, n1 = s0.y, n2 = s1.x, kappa = s1.y, alpha = s2.x;
    const double m0 = fma(R[0], n0, fma(R[1], n1, R[2] * n2));
    const double m1 = fma(R[3], n0, fma(R[4], n1, R[5] * n2));
    const double m2 = fma(R[6], n0, fma(R[7], n1, R[8] * n2));
    const double km0 = kappa * m0, km1 = kappa * m1, km2 = kappa * m2;
    fa = fma(-km0, m0, m2c0.y + alpha);
    fb = fma(-km0, m1, c12.x);
    fc = fma(-km0, m2, c12.y);
    fd = fma(-km1, m1, c34.x + alpha);
    fe = fma(-km1, m2, c34.y);
    ff = fma(-km2, m2, v5 + alpha);
  } else {
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
  fa = m2c0.y + arT(0, 0);
  fb = c12.x + arT(0, 1);
  fc = c12.y + arT(0, 2);
  fd = c34.x + arT(1, 1);
  fe = c34.y + arT(1, 2);
  ff = v5 + arT(2, 2);
  }
  // W = F^-1 = adj(F) / det(F) (:113-130).  W itself is never formed: every accumulated
  // term is linear in W, so the terms use the adjugate I and are scaled by s = scale / det
  // in their accumulating FMA.  `scale` is 0 for padding lanes (which replay a valid hit),
  // so padding contributes exact zeros without a branch.
  const double i00 = fma(fd, ff, -fe * fe), i01 = fma(fc, fe, -fb * ff),
               i02 = fma(fb, fe, -fc * fd), i11 = fma(fa, ff, -fc * fc),
               i12 = fma(fb, fc, -fa * fe), i22 = fma(fa, fd, -fb * fb);
  const double sw = rcp64(fma(fa, i00, fma(fb, i01, fc * i02))) * scale;
  // I d  (W d = s I d)
  const double wd0 = fma(i00, d0, fma(i01, d1, i02 * d2));
  const double wd1 = fma(i01, d0, fma(i11, d1, i12 * d2));
  const double wd2 = fma(i02, d0, fma(i12, d1, i22 * d2));
  acc[27] = fma(fma(d0, wd0, fma(d1, wd1, d2 * wd2)), sw, acc[27]);  // cost (:156)
  if (MODE == 0) {
    // N = hat(x') W, P = N hat(x')^T, b' = [x' x Wd ; Wd]  (J' = [-hat(x') | I]), all / s
    const double N00 = fma(-vz, i01, vy * i02), N01 = fma(-vz, i11, vy * i12),
                 N02 = fma(-vz, i12, vy * i22);
    const double N10 = fma(vz, i00, -vx * i02), N11 = fma(vz, i01, -vx * i12),
                 N12 = fma(vz, i02, -vx * i22);
    const double N20 = fma(-vy, i00, vx * i01), N21 = fma(-vy, i01, vx * i11),
                 N22 = fma(-vy, i02, vx * i12);
    acc[0] = fma(fma(-vz, N01, vy * N02), sw, acc[0]);
    acc[1] = fma(fma(vz, N00, -vx * N02), sw, acc[1]);
    acc[2] = fma(fma(-vy, N00, vx * N01), sw, acc[2]);
    acc[3] = fma(fma(vz, N10, -vx * N12), sw, acc[3]);
    acc[4] = fma(fma(-vy, N10, vx * N11), sw, acc[4]);
    acc[5] = fma(fma(-vy, N20, vx * N21), sw, acc[5]);
    acc[6] = fma(N00, sw, acc[6]);
    acc[7] = fma(N01, sw, acc[7]);
    acc[8] = fma(N02, sw, acc[8]);
    acc[9] = fma(N10, sw, acc[9]);
    acc[10] = fma(N11, sw, acc[10]);
    acc[11] = fma(N12, sw, acc[11]);
    acc[12] = fma(N20, sw, acc[12]);
    acc[13] = fma(N21, sw, acc[13]);
    acc[14] = fma(N22, sw, acc[14]);
    acc[15] = fma(i00, sw, acc[15]);
    acc[16] = fma(i01, sw, acc[16]);
    acc[17] = fma(i02, sw, acc[17]);
    acc[18] = fma(i11, sw, acc[18]);
    acc[19] = fma(i12, sw, acc[19]);
    acc[20] = fma(i22, sw, acc[20]);
    acc[21] = fma(fma(vy, wd2, -vz * wd1), sw, acc[21]);
    acc[22] = fma(fma(vz, wd0, -vx * wd2), sw, acc[22]);
    acc[23] = fma(fma(vx, wd1, -vy * wd0), sw, acc[23]);
    acc[24] = fma(wd0, sw, acc[24]);
    acc[25] = fma(wd1, sw, acc[25]);
    acc[26] = fma(wd2, sw, acc[26]);
  }
}

// K4b: one warp per item.  kStages staged rounds: the gathers of the next kStages - 1 rounds
// are in flight while a round computes; hit entries are loaded two rounds ahead of their
// gather (clamped index, so the loads are unconditional).
template <int MODE, int kStages, int kMinBlocks, int PT = 2, int PLANE = 0>
__global__ void __launch_bounds__(kAccWarps * 32, kMinBlocks)
    k_accumulate(const AccDesc* __restrict__ descs, const ItemDev* __restrict__ items,
                 int n_items, const int2* __restrict__ hits, double* __restrict__ partials,
                 int dbg) {
  static_assert(kStages >= 2, "stage reuse hazard");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int w = blockIdx.x * kAccWarps + wib;
  pdl_release();
  // the item's hit-list region and size are static (batch setup): the first hit entries are
  // loaded alongside the descriptor instead of after it (one dependent round trip less per
  // item); entries past the hit count are never used (clamped to the region, validity by n)
  const int w_ = min(w, n_items - 1);
  const int hoff = __ldg(&items[w_].hoff);
  const int isz = __ldg(&items[w_].end) - __ldg(&items[w_].begin);
  pdl_wait();  // descriptors and hit lists written by K4a
  if (w >= n_items) return;
  AccSmem<kStages, PT>& sm = reinterpret_cast<AccSmem<kStages, PT>*>(smem_raw)[wib];
  const AccDesc* dsc = descs + w;
  const int n = __ldg(&dsc->n);
  VG_DEVICE_CHECK(n >= 0 && n <= isz, "K4b: hit count exceeds the item");
  VG_DEVICE_CHECK(__ldg(&dsc->hoff) == hoff, "K4b: descriptor / item hit-list offsets differ");
  const int2* hl = hits + hoff;
  // the item's hit list (contiguous) was written by K4a and may have left L2: one prefetch
  // per 128 B line for its first 512 entries, all issued up front, instead of a DRAM round
  // trip every few rounds (covering longer lists too measured slower)
  if (16 * lane < isz) asm volatile("prefetch.global.L2 [%0];" ::"l"(hl + 16 * lane));
  double R[9], t[3];
#pragma unroll
  for (int k = 0; k < 9; ++k) R[k] = __ldg(dsc->T + k);
#pragma unroll
  for (int k = 0; k < 3; ++k) t[k] = __ldg(dsc->T + 9 + k);
  CloudView cv;
  cv.a = (const float4*)__ldg((const unsigned long long*)&dsc->a);
  cv.xyz64 = (const double*)__ldg((const unsigned long long*)&dsc->xyz64);
  cv.c0 = (const double2*)__ldg((const unsigned long long*)&dsc->c0);
  cv.c1 = (const double2*)__ldg((const unsigned long long*)&dsc->c1);
  cv.c2 = (const double2*)__ldg((const unsigned long long*)&dsc->c2);
  cv.n = 0;
  MapView mv;
  mv.recs = (const VoxelRec*)__ldg((const unsigned long long*)&dsc->recs);
  const bool f64pts = PT == 2 && cv.xyz64 != nullptr;
  // profiling knobs (VGICP_K4B_DEBUG): 1 no gathers, 2 no math, 4 no lane-own gathers
  const bool gather = !(dbg & 1), math = !(dbg & 2), own = !(dbg & 4);

  double acc[28];
#pragma unroll
  for (int k = 0; k < 28; ++k) acc[k] = 0.0;
  const int rounds = (n + 31) / 32;
  constexpr int kAhead = kStages - 1;
  const int klast = isz > 0 ? isz - 1 : 0;  // static bound of the item's hit region
  if (n > 0) {
#pragma unroll
    for (int r = 0; r < kAhead; ++r)
      issue_round<kStages, PT>(cv, mv, sm, r, ld_hit(hl + min(r * 32 + lane, klast)),
                               gather ? n - r * 32 : 0, lane, own);
    int2 nxt = ld_hit(hl + min(kAhead * 32 + lane, klast));
    int2 nxt2 = ld_hit(hl + min((kAhead + 1) * 32 + lane, klast));
    for (int r = 0; r < rounds; ++r) {
      const int ri = r + kAhead;
      issue_round<kStages, PT>(cv, mv, sm, ri, nxt, gather ? n - ri * 32 : 0, lane, own);
      nxt = nxt2;
      nxt2 = ld_hit(hl + min((ri + 2) * 32 + lane, klast));
      cp_async_wait<kAhead>();
      __syncwarp();
      if (math && r * 32 + lane < n)
        hit_math<MODE, PT, PLANE>(sm.stage[r % kStages], lane, f64pts, R, t, 1.0, acc);
      __syncwarp();  // stage r % kStages is refilled by round r + kStages
    }
    cp_async_wait<0>();
  }

  if (MODE == 1) {
    double c = acc[27];
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) c += __shfl_xor_sync(0xffffffffu, c, s);
    if (lane == 0) {
      partials[2 * (size_t)w] = c;
      partials[2 * (size_t)w + 1] = (double)n;
    }
    return;
  }
  double v[32];
#pragma unroll
  for (int k = 0; k < 28; ++k) v[k] = acc[k];
  v[28] = lane == 0 ? (double)n : 0.0;
  v[29] = 0.0;
  v[30] = 0.0;
  v[31] = 0.0;
  partials[(size_t)w * kPartialStride + lane] = warp_transpose_reduce32(v, lane);
}



// ---- K4b with TMA record gathers (VG_TMA_REC) ---------------------------------------------
// The fast-path K4b (fp32-exact points, plane-form covariances) with the 80 B voxel records
// fetched by the tensor-memory accelerator instead of cooperative cp.async: per round, lanes
// 0..7 each issue one cp.async.bulk.tensor.2d...tile::gather4 (4 record rows of the map's
// record tensor -> 320 B of shared memory), completing on the stage's mbarrier; no LSU / L1
// wavefronts for the record gathers.  Lane-own point / covariance gathers stay cp.async.
// Record rows of a group land 80 B apart in a 128 B-aligned 384 B slot.
struct alignas(128) AccStageTma {
  float4 pt[32];
  float4 cov[3][32];
  float4 rec[8][24];  // group g = records 4g..4g+3 at rec[g][5 * (q % 4) + unit]
};
struct alignas(128) AccSmemTma {
  AccStageTma stage[2];
  unsigned long long bar[2];
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_gather4(void* dst, const void* tmap, int r0, int r1, int r2,
                                            int r3, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void issue_round_tma(const CloudView& cv, const void* tmap,
                                                AccSmemTma& sm, int round, int2 e, int nvalid,
                                                int lane) {
  AccStageTma& st = sm.stage[round & 1];
  if (lane < nvalid) {
    cp_async16_sel<2>(&st.pt[lane], cv.a + e.x);
    cp_async16_sel<2>(&st.cov[0][lane], cv.c0 + e.x);
    cp_async16_sel<2>(&st.cov[1][lane], cv.c1 + e.x);
    cp_async16_sel<2>(&st.cov[2][lane], cv.c2 + e.x);
  }
  cp_async_commit();
  // record rows of group (lane & 7); rows past the round's hits replay a valid one
  const int g = lane & 7;
  int rr[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) rr[k] = __shfl_sync(0xffffffffu, e.y, 4 * g + k);
  const int ngroups = nvalid <= 0 ? 0 : min(8, (nvalid + 3) >> 2);
#pragma unroll
  for (int k = 1; k < 4; ++k)
    if (4 * g + k >= nvalid) rr[k] = rr[0];
  if (lane == 0) mbar_expect_tx(&sm.bar[round & 1], 320u * (unsigned)ngroups);
  if (lane < ngroups) tma_gather4(&st.rec[g][0], tmap, rr[0], rr[1], rr[2], rr[3], &sm.bar[round & 1]);
}

template <int MODE, int kMinBlocks>
__global__ void __launch_bounds__(32, kMinBlocks)
    k_accumulate_tma(const AccDesc* __restrict__ descs, const ItemDev* __restrict__ items,
                     const void* const* __restrict__ item_tmap, int n_items,
                     const int2* __restrict__ hits, double* __restrict__ partials) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  AccSmemTma& sm = *reinterpret_cast<AccSmemTma*>(smem_raw);
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x;
  pdl_release();
  const int w_ = min(w, n_items - 1);
  const int hoff = __ldg(&items[w_].hoff);
  const int isz = __ldg(&items[w_].end) - __ldg(&items[w_].begin);
  const void* tmap = item_tmap[w_];
  if (lane == 0) {
    mbar_init(&sm.bar[0], 1);
    mbar_init(&sm.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  pdl_wait();  // descriptors and hit lists written by K4a
  if (w >= n_items) return;
  const AccDesc* dsc = descs + w;
  const int n = __ldg(&dsc->n);
  VG_DEVICE_CHECK(n >= 0 && n <= isz, "K4b-tma: hit count exceeds the item");
  const int2* hl = hits + hoff;
  if (16 * lane < isz) asm volatile("prefetch.global.L2 [%0];" ::"l"(hl + 16 * lane));
  double R[9], t[3];
#pragma unroll
  for (int k = 0; k < 9; ++k) R[k] = __ldg(dsc->T + k);
#pragma unroll
  for (int k = 0; k < 3; ++k) t[k] = __ldg(dsc->T + 9 + k);
  CloudView cv;
  cv.a = (const float4*)__ldg((const unsigned long long*)&dsc->a);
  cv.xyz64 = nullptr;
  cv.c0 = (const double2*)__ldg((const unsigned long long*)&dsc->c0);
  cv.c1 = (const double2*)__ldg((const unsigned long long*)&dsc->c1);
  cv.c2 = (const double2*)__ldg((const unsigned long long*)&dsc->c2);
  cv.n = 0;
  double acc[28];
#pragma unroll
  for (int k = 0; k < 28; ++k) acc[k] = 0.0;
  const int rounds = (n + 31) / 32;
  const int klast = isz > 0 ? isz - 1 : 0;
  if (n > 0) {
    issue_round_tma(cv, tmap, sm, 0, ld_hit(hl + min(lane, klast)), n, lane);
    int2 nxt = ld_hit(hl + min(32 + lane, klast));
    int2 nxt2 = ld_hit(hl + min(64 + lane, klast));
    for (int r = 0; r < rounds; ++r) {
      const int ri = r + 1;
      issue_round_tma(cv, tmap, sm, ri, nxt, n - ri * 32, lane);
      nxt = nxt2;
      nxt2 = ld_hit(hl + min((ri + 2) * 32 + lane, klast));
      cp_async_wait<1>();
      mbar_wait(&sm.bar[r & 1], (unsigned)((r >> 1) & 1));
      __syncwarp();
      if (r * 32 + lane < n) {
        const AccStageTma& st = sm.stage[r & 1];
        const float4 a = st.pt[lane];
        const double2 s0 = *reinterpret_cast<const double2*>(&st.cov[0][lane]);
        const double2 s1 = *reinterpret_cast<const double2*>(&st.cov[1][lane]);
        const double2 s2 = *reinterpret_cast<const double2*>(&st.cov[2][lane]);
        hit_core<MODE, 1>(a.x, a.y, a.z, s0, s1, s2, &st.rec[lane >> 2][5 * (lane & 3)], R, t,
                          1.0, acc);
      }
      __syncwarp();  // stage r & 1 is refilled by round r + 2
    }
    cp_async_wait<0>();
    // the last issued round (rounds) may still be in flight on its mbarrier: drain it so no
    // async-proxy write lands in shared memory after the CTA exits
    mbar_wait(&sm.bar[rounds & 1], (unsigned)((rounds >> 1) & 1));
  }
  if (MODE == 1) {
    double c = acc[27];
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) c += __shfl_xor_sync(0xffffffffu, c, s);
    if (lane == 0) {
      partials[2 * (size_t)w] = c;
      partials[2 * (size_t)w + 1] = (double)n;
    }
    return;
  }
  double v[32];
#pragma unroll
  for (int k = 0; k < 28; ++k) v[k] = acc[k];
  v[28] = lane == 0 ? (double)n : 0.0;
  v[29] = 0.0;
  v[30] = 0.0;
  v[31] = 0.0;
  partials[(size_t)w * kPartialStride + lane] = warp_transpose_reduce32(v, lane);
}

// ---- K4c: cost mode, lookup and cost fused ----------------------------------------------------
// The LM's candidate evaluations need only each factor's cost and inlier count
// (factor_graph.py:589-591 -> MatchingCostFactor.cost -> matching_cost, registration.py:160-165).
// Without the 28 accumulators the per-hit math is ~70 fp64 ops, so the K4a -> K4b split (hit
// list written and re-read, a second launch with its own per-item prologue) costs more than
// compaction saves: here one warp per item probes a round of 32 points exactly as K4a does,
// gathers that round's hit records (cooperatively, 5 lanes per 80 B record) and plane-form
// covariances into a 2-stage shared-memory ring, and computes the previous round's costs while
// those gathers fly; lanes whose point missed sit out the math.  Fast path only (32-bit local
// keys, power-of-two resolutions, fp32-exact points, plane-form covariances).  Per-hit cost:
// hit_core's, term for term; summed per lane in round order, then a fixed butterfly.
// OWN_REG: the point and plane covariance of a hit ride in registers to the next round (lane-own,
// nearly coalesced loads) and only the records are staged: 5 KB of shared memory per warp
// instead of 9 KB, which leaves the L1 to the point / bucket loads.
struct CostSmem {
  float4 rec[2][32][kRecStride];
};
// MODE 0 (linearize, the 28 accumulators and K4b's transpose reduction): the fused variant
// kept for measurement only (VGICP_LIN_FUSED=1).
template <int kMinBlocks, int OWN_REG, int MODE = 1>
__global__ void __launch_bounds__(32, kMinBlocks)
    k_cost_fused(const ItemHdr* __restrict__ hdrs, int n_items, double* __restrict__ partials) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  AccSmem<2, 1>& sm = *reinterpret_cast<AccSmem<2, 1>*>(smem_raw);
  CostSmem& smr = *reinterpret_cast<CostSmem*>(smem_raw);
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x;
  pdl_release();
  pdl_wait();  // item headers carry T_ij written by K-compose
  if (w >= n_items) return;
  const ItemHdr* h = hdrs + w;
  double R[9], t[3];
#pragma unroll
  for (int k = 0; k < 9; ++k) R[k] = __ldg(h->T + k);
#pragma unroll
  for (int k = 0; k < 3; ++k) t[k] = __ldg(h->T + 9 + k);
  const float4* pa = (const float4*)__ldg((const unsigned long long*)&h->a);
  const double2* c0 = (const double2*)__ldg((const unsigned long long*)&h->c0);
  const double2* c1 = (const double2*)__ldg((const unsigned long long*)&h->c1);
  const double2* c2 = (const double2*)__ldg((const unsigned long long*)&h->c2);
  const VoxelRec* recs = (const VoxelRec*)__ldg((const unsigned long long*)&h->mv.recs);
  const unsigned* keys32 = (const unsigned*)__ldg((const unsigned long long*)&h->mv.keys32);
  const double inv_res = __ldg(&h->mv.inv_res);
  const int shift = __ldg(&h->mv.shift);
  const unsigned mask = __ldg(&h->mv.mask);
  const int m = __ldg(&h->mv.m);
  const int bx = __ldg(&h->mv.bx), by = __ldg(&h->mv.by), bz = __ldg(&h->mv.bz);
  const int ex = __ldg(&h->mv.ex), ey = __ldg(&h->mv.ey), ez = __ldg(&h->mv.ez);
  const int begin = __ldg(&h->begin), end = __ldg(&h->end);
  const int last = end - 1;
  struct Q {
    unsigned k32, bucket;
    bool live;
  };
  auto make_q = [&](float4 a, int i) {  // k_lookup_fast's query, step for step
    const double px = a.x, py = a.y, pz = a.z;
    const double x = fma(R[0], px, fma(R[1], py, R[2] * pz)) + t[0];
    const double y = fma(R[3], px, fma(R[4], py, R[5] * pz)) + t[1];
    const double z = fma(R[6], px, fma(R[7], py, R[8] * pz)) + t[2];
    const double qx = x * inv_res, qy = y * inv_res, qz = z * inv_res;
    const int ix = __double2int_rd(qx), iy = __double2int_rd(qy), iz = __double2int_rd(qz);
    Q q;
    q.live = false;
    q.k32 = 0;
    if ((unsigned)(ix + 1048575) < 2097151u && (unsigned)(iy + 1048575) < 2097151u &&
        (unsigned)(iz + 1048575) < 2097151u) {
      const unsigned lx = (unsigned)(ix - bx), ly = (unsigned)(iy - by), lz = (unsigned)(iz - bz);
      q.live = lx < (unsigned)ex && ly < (unsigned)ey && lz < (unsigned)ez;
      q.k32 = lx | (ly << 11) | (lz << 22);
    } else {
      MapView mv;
      mv.bx = bx; mv.by = by; mv.bz = bz; mv.ex = ex; mv.ey = ey; mv.ez = ez; mv.shift = shift;
      const Query qq = make_query(mv, floor(qx), floor(qy), floor(qz), 1);
      q.live = qq.inside;
      q.k32 = qq.k32;
    }
    q.bucket = bucket32(q.k32, shift);
    q.live = q.live && i < end && m > 0;
    return q;
  };
  auto load_bucket = [&](unsigned bucket, unsigned (&g)[4]) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(keys32 + (size_t)bucket * kBucket32));
    g[0] = v.x;
    g[1] = v.y;
    g[2] = v.z;
    g[3] = v.w;
  };
  auto resolve = [&](const Q& q, unsigned (&g)[4]) {
    int slot = -1;
    if (q.live) {
      unsigned bk = q.bucket;
      for (unsigned probes = 0;; ++probes) {
        VG_DEVICE_CHECK(probes <= mask, "K4c: every bucket visited");
        int found = -1;
        bool empty = false;
#pragma unroll
        for (int j = kBucket32 - 1; j >= 0; --j) {
          if (g[j] == q.k32) found = j;
          empty |= (g[j] == kEmpty32);
        }
        if (found >= 0) {
          slot = (int)(bk * kBucket32 + found);
          break;
        }
        if (empty) break;
        bk = (bk + 1) & mask;
        load_bucket(bk, g);
      }
    }
    return slot;
  };
  double acc[28];
#pragma unroll
  for (int k = 0; k < 28; ++k) acc[k] = 0.0;
  int cnt = 0;
  bool prev_hit = false;
  float4 pp = make_float4(0.f, 0.f, 0.f, 0.f);  // OWN_REG: previous round's point, covariance
  double2 s0p = make_double2(0.0, 0.0), s1p = s0p, s2p = s0p;
  float4 p0 = ld_pt(pa + min(begin + lane, last));
  float4 p1 = ld_pt(pa + min(begin + 32 + lane, last));
  unsigned g0[4] = {0, 0, 0, 0}, g1[4] = {0, 0, 0, 0};
  Q q0 = make_q(p0, begin + lane);
  if (q0.live) load_bucket(q0.bucket, g0);
  int r = 0;
  for (int base = begin; base < end; base += 32, ++r) {
    const int i = base + lane;
    // the next round's probe and the point after it are in flight while this round resolves
    const Q q1 = make_q(p1, i + 32);
    if (q1.live) load_bucket(q1.bucket, g1);
    const float4 p2 = ld_pt(pa + min(i + 64, last));
    const int slot = resolve(q0, g0);
    cnt += __popc(__ballot_sync(0xffffffffu, slot >= 0));
    // this round's gathers into stage r & 1 (misses contribute nothing, registration.py:150-156)
    AccStageT<1>& st = sm.stage[r & 1];
    double2 s0n = make_double2(0.0, 0.0), s1n = s0n, s2n = s0n;
    if (slot >= 0) {
      if (OWN_REG) {
        s0n = __ldg(c0 + i);
        s1n = __ldg(c1 + i);
        s2n = __ldg(c2 + i);
      } else {
        st.pt[0][lane] = p0;
        cp_async16_sel<2>(&st.cov[0][lane], c0 + i);
        cp_async16_sel<2>(&st.cov[1][lane], c1 + i);
        cp_async16_sel<2>(&st.cov[2][lane], c2 + i);
      }
    }
#pragma unroll
    for (int c = 0; c < kRecUnits; ++c) {
      const int u = c * 32 + lane;
      const int q = u / kRecUnits, j = u - q * kRecUnits;
      const int row = __shfl_sync(0xffffffffu, slot, q);
      if (row >= 0)
        cp_async16_sel<1>(OWN_REG ? &smr.rec[r & 1][q][j] : &st.rec[q][j],
                          reinterpret_cast<const char*>(recs + row) + 16 * j);
    }
    cp_async_commit();
    // the previous round's costs
    if (r > 0) {
      cp_async_wait<1>();
      __syncwarp();
      if (prev_hit) {
        if (OWN_REG)
          hit_core<MODE, 1>(pp.x, pp.y, pp.z, s0p, s1p, s2p, smr.rec[(r - 1) & 1][lane], R, t,
                            1.0, acc);
        else
          hit_math<MODE, 1, 1>(sm.stage[(r - 1) & 1], lane, false, R, t, 1.0, acc);
      }
      __syncwarp();  // stage (r - 1) & 1 is refilled by round r + 1
    }
    prev_hit = slot >= 0;
    if (OWN_REG) {
      pp = p0;
      s0p = s0n;
      s1p = s1n;
      s2p = s2n;
    }
    p0 = p1;
    p1 = p2;
    q0 = q1;
#pragma unroll
    for (int k = 0; k < 4; ++k) g0[k] = g1[k];
  }
  cp_async_wait<0>();
  __syncwarp();
  if (r > 0 && prev_hit) {
    if (OWN_REG)
      hit_core<MODE, 1>(pp.x, pp.y, pp.z, s0p, s1p, s2p, smr.rec[(r - 1) & 1][lane], R, t, 1.0,
                        acc);
    else
      hit_math<MODE, 1, 1>(sm.stage[(r - 1) & 1], lane, false, R, t, 1.0, acc);
  }
  if (MODE == 1) {
    double c = acc[27];
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) c += __shfl_xor_sync(0xffffffffu, c, s);
    if (lane == 0) {
      partials[2 * (size_t)w] = c;
      partials[2 * (size_t)w + 1] = (double)cnt;
    }
    return;
  }
  double v[32];
#pragma unroll
  for (int k = 0; k < 28; ++k) v[k] = acc[k];
  v[28] = lane == 0 ? (double)cnt : 0.0;
  v[29] = 0.0;
  v[30] = 0.0;
  v[31] = 0.0;
  partials[(size_t)w * kPartialStride + lane] = warp_transpose_reduce32(v, lane);
}

}  // namespace vg

using namespace vg;

static int launch_lookup_range(vg_ctx* ctx, vg_batch* b, int kmode, int off, int cnt,
                               cudaStream_t st) {
  const int lb = (cnt + kLookupWarps - 1) / kLookupWarps;
  double* p2 = kmode == 2 ? b->partials + 2 * (size_t)off : nullptr;
  const ItemDev* it = b->items + off;
  int* hc = b->hit_counts + off;
  AccDesc* dd = b->descs + off;
  if (b->key_mode == 1 && b->all_pow2 && b->all_f32)  // fast path
    VG_CUDA(launch_pdl(k_lookup_fast<VG_K4A_MINB>, dim3(lb), dim3(kLookupWarps * 32), 0, st,
                       (const ItemHdr*)(b->hdrs + off), cnt, b->hits, hc, p2, dd));
  else if (b->key_mode == 1 && b->all_pow2)
    k_lookup_items<1, 24, 1><<<lb, kLookupWarps * 32, 0, st>>>(it, cnt, b->factors, b->clouds,
                                                              b->maps, b->hits, hc, p2, dd);
  else if (b->key_mode == 1)
    k_lookup_items<1, 24><<<lb, kLookupWarps * 32, 0, st>>>(it, cnt, b->factors, b->clouds,
                                                           b->maps, b->hits, hc, p2, dd);
  else if (b->key_mode == 0)
    k_lookup_items<0, 24><<<lb, kLookupWarps * 32, 0, st>>>(it, cnt, b->factors, b->clouds,
                                                           b->maps, b->hits, hc, p2, dd);
  else
    k_lookup_items<2, 24><<<lb, kLookupWarps * 32, 0, st>>>(it, cnt, b->factors, b->clouds,
                                                           b->maps, b->hits, hc, p2, dd);
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  return 0;
}

template <class K>
static int launch_acc_kernel(vg_ctx* ctx, K kern, size_t smem, const AccDesc* d,
                             const ItemDev* items, int cnt, const int2* hits, double* partials,
                             cudaStream_t st) {
  static const int dbg = [] {
    // profiling only: 1 no gathers, 2 no math, 4 no lane-own point/covariance gathers
    const char* e = getenv("VGICP_K4B_DEBUG");
    return e ? atoi(e) : 0;
  }();
  VG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  VG_CUDA(launch_pdl(kern, dim3((cnt + kAccWarps - 1) / kAccWarps), dim3(kAccWarps * 32), smem,
                     st, d, items, cnt, hits, partials, dbg));
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  return 0;
}

#ifndef VG_TMA_REC
#define VG_TMA_REC 0
#endif
#ifndef VG_K4B_MINB_TMA
#define VG_K4B_MINB_TMA 15
#endif

static int launch_acc_range(vg_ctx* ctx, vg_batch* b, int kmode, int off, int cnt,
                            cudaStream_t st) {
  const AccDesc* d = b->descs + off;
  static const int tma_env = [] {
    const char* e = getenv("VGICP_TMA_REC");  // 0/1 overrides the build default
    return e ? atoi(e) : VG_TMA_REC;
  }();
  if (tma_env && b->item_tmap && b->all_f32 && b->all_plane && kmode != 2) {
    const size_t smem = sizeof(AccSmemTma);
    const void* const* tm = b->item_tmap + off;
    if (kmode == 1) {
      VG_CUDA(cudaFuncSetAttribute(k_accumulate_tma<1, VG_K4B_MINB_COST>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      VG_CUDA(launch_pdl(k_accumulate_tma<1, VG_K4B_MINB_COST>, dim3(cnt), dim3(32), smem, st, d,
                         (const ItemDev*)(b->items + off), tm, cnt, (const int2*)b->hits,
                         b->partials + 2 * (size_t)off));
    } else {
      VG_CUDA(cudaFuncSetAttribute(k_accumulate_tma<0, VG_K4B_MINB_TMA>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      VG_CUDA(launch_pdl(k_accumulate_tma<0, VG_K4B_MINB_TMA>, dim3(cnt), dim3(32), smem, st, d,
                         (const ItemDev*)(b->items + off), tm, cnt, (const int2*)b->hits,
                         b->partials + (size_t)off * kPartialStride));
    }
    ctx->launches++;
    VG_CUDA(cudaGetLastError());
    return 0;
  }
  const size_t s2 = sizeof(AccSmem<2>) * kAccWarps, s1 = sizeof(AccSmem<2, 1>) * kAccWarps;
  if (kmode == 1) {  // cost only (LM candidate steps, factor_graph.py:591)
    double* p = b->partials + 2 * (size_t)off;
    if (b->all_f32)
      return b->all_plane
                 ? launch_acc_kernel(ctx, k_accumulate<1, 2, VG_K4B_MINB_COST, 1, 1>, s1, d, b->items + off, cnt, b->hits, p, st)
                 : launch_acc_kernel(ctx, k_accumulate<1, 2, VG_K4B_MINB_COST, 1, 0>, s1, d, b->items + off, cnt, b->hits, p, st);
    return b->all_plane
               ? launch_acc_kernel(ctx, k_accumulate<1, 2, VG_K4B_MINB_COST, 2, 1>, s2, d, b->items + off, cnt, b->hits, p, st)
               : launch_acc_kernel(ctx, k_accumulate<1, 2, VG_K4B_MINB_COST, 2, 0>, s2, d, b->items + off, cnt, b->hits, p, st);
  }
  double* p = b->partials + (size_t)off * kPartialStride;
  // PT = 1: every point fp32-exact, one 16 B point unit per lane (more L1 left)
  if (b->all_f32)
    return b->all_plane
               ? launch_acc_kernel(ctx, k_accumulate<0, VG_K4B_STAGES, VG_K4B_MINB, 1, 1>,
                                   sizeof(AccSmem<VG_K4B_STAGES, 1>) * kAccWarps, d, b->items + off, cnt, b->hits, p, st)
               : launch_acc_kernel(ctx, k_accumulate<0, 2, VG_K4B_MINB_GEN, 1, 0>, s1, d, b->items + off, cnt, b->hits, p, st);
  return b->all_plane
             ? launch_acc_kernel(ctx, k_accumulate<0, 2, VG_K4B_MINB_GEN, 2, 1>, s2, d, b->items + off, cnt, b->hits, p, st)
             : launch_acc_kernel(ctx, k_accumulate<0, 2, VG_K4B_MINB_GEN, 2, 0>, s2, d, b->items + off, cnt, b->hits, p, st);
}

#ifndef VG_COST_MINB
#define VG_COST_MINB 24
#endif
#ifndef VG_COST_OWN_REG
#define VG_COST_OWN_REG 1
#endif

// cost mode on the fast path: K4c (lookup + cost fused) instead of K4a + K4b
static bool cost_fused(const vg_batch* b, int kmode) {
  static const int env = [] {
    const char* e = getenv("VGICP_COST_FUSED");  // 0: K4a + K4b (ablation)
    return e ? atoi(e) : 1;
  }();
  return env && kmode == 1 && b->key_mode == 1 && b->all_pow2 && b->all_f32 && b->all_plane;
}

static int launch_cost_fused(vg_ctx* ctx, vg_batch* b, int off, int cnt, cudaStream_t st) {
  const size_t smem = VG_COST_OWN_REG ? sizeof(CostSmem) : sizeof(AccSmem<2, 1>);
  auto kern = k_cost_fused<VG_COST_MINB, VG_COST_OWN_REG>;
  VG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  VG_CUDA(launch_pdl(kern, dim3(cnt), dim3(32), smem, st,
                     (const ItemHdr*)(b->hdrs + off), cnt, b->partials + 2 * (size_t)off));
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  return 0;
}

#ifndef VG_LIN_FUSED_MINB
#define VG_LIN_FUSED_MINB 14
#endif
// linearize mode through the fused kernel (VGICP_LIN_FUSED=1; measurement only): large batches
// run 16% slower fused, config 1's single factor 5% faster (0.037 vs 0.039 ms) — not enabled
// by size, so a factor's record does not change with the path its batch takes
static bool lin_fused(const vg_batch* b, int kmode) {
  static const int env = [] {
    const char* e = getenv("VGICP_LIN_FUSED");
    return e ? atoi(e) : 0;
  }();
  return env == 1 && kmode == 0 && b->key_mode == 1 && b->all_pow2 && b->all_f32 &&
         b->all_plane;
}

static int launch_lin_fused(vg_ctx* ctx, vg_batch* b, int off, int cnt, cudaStream_t st) {
  const size_t smem = sizeof(CostSmem);
  auto kern = k_cost_fused<VG_LIN_FUSED_MINB, 1, 0>;
  VG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  VG_CUDA(launch_pdl(kern, dim3(cnt), dim3(32), smem, st, (const ItemHdr*)(b->hdrs + off), cnt,
                     b->partials + (size_t)off * kPartialStride));
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  return 0;
}

int launch_accumulate_range(vg_ctx* ctx, vg_batch* b, int kmode, int lo, int hi) {
  if (hi <= lo) return 0;
  if (cost_fused(b, kmode)) return launch_cost_fused(ctx, b, lo, hi - lo, ctx->stream);
  if (lin_fused(b, kmode)) return launch_lin_fused(ctx, b, lo, hi - lo, ctx->stream);
  VG_CHECK(launch_lookup_range(ctx, b, kmode, lo, hi - lo, ctx->stream));
  if (kmode != 2) VG_CHECK(launch_acc_range(ctx, b, kmode, lo, hi - lo, ctx->stream));
  return 0;
}

int launch_accumulate_range_ev(vg_ctx* ctx, vg_batch* b, int kmode, int lo, int hi,
                               cudaEvent_t after_lookup) {
  if (cost_fused(b, kmode) || lin_fused(b, kmode)) {  // one kernel: the event marks its end
    if (hi > lo)
      VG_CHECK(cost_fused(b, kmode) ? launch_cost_fused(ctx, b, lo, hi - lo, ctx->stream)
                                    : launch_lin_fused(ctx, b, lo, hi - lo, ctx->stream));
    VG_CUDA(cudaEventRecord(after_lookup, ctx->stream));
    return 0;
  }
  if (hi > lo) VG_CHECK(launch_lookup_range(ctx, b, kmode, lo, hi - lo, ctx->stream));
  VG_CUDA(cudaEventRecord(after_lookup, ctx->stream));
  if (hi > lo && kmode != 2) VG_CHECK(launch_acc_range(ctx, b, kmode, lo, hi - lo, ctx->stream));
  return 0;
}

// K4a + K4b over the whole batch (DESIGN.md §9 lists the alternatives that measured slower)
int launch_accumulate(vg_ctx* ctx, vg_batch* b, int kmode) {
  return launch_accumulate_range(ctx, b, kmode, 0, (int)b->num_items);
}

namespace vg {
// Correspondence export (vg_batch_lookup_rows): the (point, record) hit lists the last K4a
// pass compacted — exactly what K4b consumes — scattered as the reference row of every hit
// point (GaussianVoxelMap.lookup's result, registration.py:47-55,149) into the factor's slice
// of `rows` (pre-filled with -1 = miss).  One warp per item.
__global__ void k_export_rows(const ItemDev* __restrict__ items, int n_items,
                              const AccDesc* __restrict__ descs, const int2* __restrict__ hits,
                              const long long* __restrict__ pt_off,
                              long long* __restrict__ rows) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= n_items) return;
  const int n = descs[w].n;
  const int hoff = items[w].hoff;
  const VoxelRec* recs = descs[w].recs;
  long long* dst = rows + pt_off[items[w].factor];
  for (int k = lane; k < n; k += 32) {
    const int2 h = hits[hoff + k];
    VG_DEVICE_CHECK(h.x >= items[w].begin && h.x < items[w].end, "export: point outside item");
    dst[h.x] = recs[h.y].row;
  }
}
}  // namespace vg

int launch_export_rows(vg_ctx* ctx, vg_batch* b, const long long* pt_off_dev, long long* rows_dev) {
  if (b->num_items == 0) return 0;
  const int warps = 4;
  k_export_rows<<<(int)((b->num_items + warps - 1) / warps), warps * 32, 0, ctx->stream>>>(
      b->items, (int)b->num_items, b->descs, b->hits, pt_off_dev, rows_dev);
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  return 0;
}
