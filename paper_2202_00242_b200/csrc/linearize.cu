// linearize.cu — K3 lookup, K3t per-point terms (the per-factor API), K5 finalize, and the
// on-device pose composition T_ij = T_j^-1 T_i (K4a/K4b, the batched path, are in
// accumulate.cu).
//
// Reference: registration.py:146-157 (match_terms), :207-248 (linearize_from_terms),
// :251-269 (linearize_matching_cost), factor_graph.py:253-308 (MatchingCostFactor).
//
// Per correspondence the kernels read the source Gaussian (fp32 xyz + fp64 covariance, SoA)
// and one voxel record (fp64 mean + covariance) found through the hash, and do all math in
// fp64:
//   x = R p + t -> key (bit-exact floor) -> probe -> d = mu' - x -> W = (C' + R C R^T)^-1
//   (adjugate) -> accumulate the 6x6 target-frame block about the source origin (29 values,
//   H_ii, H_ij, H_jj, b_i, b_j are exact fp64 adjoint transforms of it, so
//   nothing else is accumulated per point).
// The warp reduction and the per-factor sum are fixed-order, so results are deterministic.
#include <cuda_runtime.h>

#include "common.cuh"
#include "internal.h"

namespace vg {

struct PointTerms {
  double d[3];
  double W[6];   // 00 01 02 11 12 22
  double wd[3];
  double xp[3];  // x - t == R p : lever arm about the source origin
  double cost;
};

__device__ __forceinline__ void load_T(const double* __restrict__ T, double (&R)[9],
                                       double (&t)[3]) {
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = __ldg(T + i);
#pragma unroll
  for (int i = 0; i < 3; ++i) t[i] = __ldg(T + 9 + i);
}

__device__ __forceinline__ void transform(const double (&R)[9], const double (&t)[3],
                                          double px, double py, double pz, double& x,
                                          double& y, double& z) {
  // points @ R^T + t (registration.py:148)
  x = fma(R[0], px, fma(R[1], py, R[2] * pz)) + t[0];
  y = fma(R[3], px, fma(R[4], py, R[5] * pz)) + t[1];
  z = fma(R[6], px, fma(R[7], py, R[8] * pz)) + t[2];
}

__device__ __forceinline__ void load_point(const CloudView& cv, long long i, double& px,
                                           double& py, double& pz, float4& pa) {
  pa = __ldg(cv.a + i);
  if (cv.xyz64) {
    px = __ldg(cv.xyz64 + 3 * i);
    py = __ldg(cv.xyz64 + 3 * i + 1);
    pz = __ldg(cv.xyz64 + 3 * i + 2);
  } else {
    px = pa.x;
    py = pa.y;
    pz = pa.z;
  }
}

// fused covariance, inverse, residual and Mahalanobis cost of one correspondence
// (registration.py:150-156), all fp64.
__device__ __forceinline__ void point_terms(const double (&R)[9], const CloudView& cv,
                                            long long i, const VoxelRec* __restrict__ sl,
                                            double x, double y, double z, const double (&t)[3],
                                            PointTerms& o) {
  const double2 m01 = __ldg(reinterpret_cast<const double2*>(&sl->mean[0]));
  const double2 m2c0 = __ldg(reinterpret_cast<const double2*>(&sl->mean[2]));
  const double2 c12 = __ldg(reinterpret_cast<const double2*>(&sl->cov[1]));
  const double2 c34 = __ldg(reinterpret_cast<const double2*>(&sl->cov[3]));
  const double v5 = __ldg(&sl->cov[5]);
  const double2 s0 = __ldg(cv.c0 + i), s1 = __ldg(cv.c1 + i), s2 = __ldg(cv.c2 + i);
  // d = mu' - moved (registration.py:152)
  o.d[0] = m01.x - x;
  o.d[1] = m01.y - y;
  o.d[2] = m2c0.x - z;
  o.xp[0] = x - t[0];
  o.xp[1] = y - t[1];
  o.xp[2] = z - t[2];
  // source covariance C: c00 c01 c02 c11 c12 c22
  const double C00 = s0.x, C01 = s0.y, C02 = s1.x, C11 = s1.y, C12 = s2.x, C22 = s2.y;
  double A[9];  // A = R C
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const double r0 = R[3 * r], r1 = R[3 * r + 1], r2 = R[3 * r + 2];
    A[3 * r + 0] = fma(r0, C00, fma(r1, C01, r2 * C02));
    A[3 * r + 1] = fma(r0, C01, fma(r1, C11, r2 * C12));
    A[3 * r + 2] = fma(r0, C02, fma(r1, C12, r2 * C22));
  }
  // F = C' + A R^T  (registration.py:153)
  auto arT = [&](int r, int c) {
    return fma(A[3 * r], R[3 * c], fma(A[3 * r + 1], R[3 * c + 1], A[3 * r + 2] * R[3 * c + 2]));
  };
  const double a = m2c0.y + arT(0, 0);
  const double b = c12.x + arT(0, 1);
  const double c = c12.y + arT(0, 2);
  const double dd = c34.x + arT(1, 1);
  const double e = c34.y + arT(1, 2);
  const double f = v5 + arT(2, 2);
  // W = F^-1 by the adjugate (registration.py:113-130)
  const double i00 = fma(dd, f, -e * e);
  const double i01 = fma(c, e, -b * f);
  const double i02 = fma(b, e, -c * dd);
  const double i11 = fma(a, f, -c * c);
  const double i12 = fma(b, c, -a * e);
  const double i22 = fma(a, dd, -b * b);
  const double det = fma(a, i00, fma(b, i01, c * i02));
  const double inv = rcp64(det);
  o.W[0] = i00 * inv;
  o.W[1] = i01 * inv;
  o.W[2] = i02 * inv;
  o.W[3] = i11 * inv;
  o.W[4] = i12 * inv;
  o.W[5] = i22 * inv;
  o.wd[0] = fma(o.W[0], o.d[0], fma(o.W[1], o.d[1], o.W[2] * o.d[2]));
  o.wd[1] = fma(o.W[1], o.d[0], fma(o.W[3], o.d[1], o.W[4] * o.d[2]));
  o.wd[2] = fma(o.W[2], o.d[0], fma(o.W[4], o.d[1], o.W[5] * o.d[2]));
  o.cost = fma(o.d[0], o.wd[0], fma(o.d[1], o.wd[1], o.d[2] * o.wd[2]));
}

// ---- warp reductions ---------------------------------------------------------------------

// ---- K5: per-factor fixed-order sum of item partials + fp64 adjoint expansion ------------
__device__ __forceinline__ void mat3_mul(const double* A, const double* B, double* C) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      C[3 * r + c] = A[3 * r] * B[c] + A[3 * r + 1] * B[3 + c] + A[3 * r + 2] * B[6 + c];
}
__device__ __forceinline__ void mat3_tmul(const double* A, const double* B, double* C) {
  // C = A^T B
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      C[3 * r + c] = A[r] * B[c] + A[3 + r] * B[3 + c] + A[6 + r] * B[6 + c];
}

// write the upper triangle of a 6x6 assembled from 3x3 blocks [[A, B], [B^T, D]]
__device__ __forceinline__ void store_sym6(double* out, const double* A, const double* B,
                                           const double* D, double scale) {
  int k = 0;
  for (int r = 0; r < 6; ++r)
    for (int c = r; c < 6; ++c) {
      double v;
      if (r < 3 && c < 3) v = A[3 * r + c];
      else if (r < 3) v = B[3 * r + (c - 3)];
      else v = D[3 * (r - 3) + (c - 3)];
      out[k++] = scale * v;
    }
}

__device__ __forceinline__ void expand_record(const FactorDev& f, const double* s, double* o);

// one factor; LINEARIZE records go to `o92` (shared memory staging), others straight to out
__device__ __forceinline__ void finalize_one(const FactorDev& f, int fi,
                                             const double* __restrict__ partials, int mode,
                                             double* __restrict__ out, double* o92) {
  if (mode == 1 || mode == 3) {
    double c = 0.0, n = 0.0;
    for (int it = 0; it < f.item_count; ++it) {
      c += partials[2 * (size_t)(f.item_begin + it)];
      n += partials[2 * (size_t)(f.item_begin + it) + 1];
    }
    out[2 * (size_t)fi] = c;
    out[2 * (size_t)fi + 1] = n;
    return;
  }
  double s[29];
#pragma unroll
  for (int k = 0; k < 29; ++k) s[k] = 0.0;
  for (int it = 0; it < f.item_count; ++it) {
    const double* p = partials + (size_t)(f.item_begin + it) * kPartialStride;
#pragma unroll
    for (int k = 0; k < 29; ++k) s[k] += p[k];
  }
  if (mode == 2) {
    double* o = out + (size_t)fi * 29;
#pragma unroll
    for (int k = 0; k < 29; ++k) o[k] = s[k];
    return;
  }
  expand_record(f, s, o92);
}

// fp64 adjoint expansion of one factor's 29 sums (H' 21, b' 6, cost, inliers) into the
// 92-double record, with min_inliers gating (factor_graph.py:282-291)
__device__ __forceinline__ void expand_record(const FactorDev& f, const double* s, double* o) {
  const double cost = s[27], inliers = s[28];
  if (inliers < (double)f.min_inliers) {  // DegenerateConstraint -> zero blocks
    for (int k = 0; k < 90; ++k) o[k] = 0.0;
    o[90] = cost;
    o[91] = inliers;
    return;
  }
  // H' = [[P, N], [N^T, S]], b' = [br; bt]
  const double P[9] = {s[0], s[1], s[2], s[1], s[3], s[4], s[2], s[4], s[5]};
  const double N[9] = {s[6], s[7], s[8], s[9], s[10], s[11], s[12], s[13], s[14]};
  const double S[9] = {s[15], s[16], s[17], s[16], s[18], s[19], s[17], s[19], s[20]};
  const double br[3] = {s[21], s[22], s[23]};
  const double bt[3] = {s[24], s[25], s[26]};
  const double* R = f.T;
  const double t0 = f.T[9], t1 = f.T[10], t2 = f.T[11];
  const double Ch[9] = {0.0, -t2, t1, t2, 0.0, -t0, -t1, t0, 0.0};  // hat(t)
  double Nt[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) Nt[3 * r + c] = N[3 * c + r];
  double tmp[9], tmp2[9];
  // ---- source block: H_ii = Rd^T H' Rd, b_i = -Rd^T b'  (Rd = diag(R, R))
  double RtP[9], RtN[9], RtS[9], Hii_a[9], Hii_b[9], Hii_d[9];
  mat3_tmul(R, P, RtP);
  mat3_tmul(R, N, RtN);
  mat3_tmul(R, S, RtS);
  mat3_mul(RtP, R, Hii_a);
  mat3_mul(RtN, R, Hii_b);
  mat3_mul(RtS, R, Hii_d);
  store_sym6(o, Hii_a, Hii_b, Hii_d, 2.0);
  double* bi = o + 78;
  for (int r = 0; r < 3; ++r) {
    bi[r] = -2.0 * (R[r] * br[0] + R[3 + r] * br[1] + R[6 + r] * br[2]);
    bi[3 + r] = -2.0 * (R[r] * bt[0] + R[3 + r] * bt[1] + R[6 + r] * bt[2]);
  }
  o[90] = cost;
  o[91] = inliers;
  if (f.flags & 1) {  // unary: target fixed (registration.py:233-235)
    for (int k = 21; k < 78; ++k) o[k] = 0.0;
    for (int k = 84; k < 90; ++k) o[k] = 0.0;
    return;
  }
  // ---- target block: H_jj = E^T H' E, E = [[I, 0], [-C, I]], C = hat(t)
  double NC[9], CNt[9], CS[9], SC[9], CSC[9];
  mat3_mul(N, Ch, NC);
  mat3_mul(Ch, Nt, CNt);
  mat3_mul(Ch, S, CS);
  mat3_mul(S, Ch, SC);
  mat3_mul(CS, Ch, CSC);
  double Ja[9], Jb[9];
  for (int k = 0; k < 9; ++k) {
    Ja[k] = P[k] + CNt[k] - NC[k] - CSC[k];
    Jb[k] = N[k] + CS[k];
  }
  store_sym6(o + 57, Ja, Jb, S, 2.0);
  double* bj = o + 84;
  bj[0] = 2.0 * (br[0] + Ch[0] * bt[0] + Ch[1] * bt[1] + Ch[2] * bt[2]);
  bj[1] = 2.0 * (br[1] + Ch[3] * bt[0] + Ch[4] * bt[1] + Ch[5] * bt[2]);
  bj[2] = 2.0 * (br[2] + Ch[6] * bt[0] + Ch[7] * bt[1] + Ch[8] * bt[2]);
  bj[3] = 2.0 * bt[0];
  bj[4] = 2.0 * bt[1];
  bj[5] = 2.0 * bt[2];
  // ---- cross block: H_ij = -Rd^T H' E = -[[R^T(P - N C), R^T N], [R^T(N^T - S C), R^T S]]
  double* hij = o + 21;
  for (int k = 0; k < 9; ++k) tmp[k] = P[k] - NC[k];
  mat3_tmul(R, tmp, tmp2);  // R^T (P - N C)
  double lowL[9];
  for (int k = 0; k < 9; ++k) tmp[k] = Nt[k] - SC[k];
  mat3_tmul(R, tmp, lowL);  // R^T (N^T - S C)
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) {
      double v;
      if (r < 3 && c < 3) v = tmp2[3 * r + c];
      else if (r < 3) v = RtN[3 * r + (c - 3)];
      else if (c < 3) v = lowL[3 * (r - 3) + c];
      else v = RtS[3 * (r - 3) + (c - 3)];
      hij[6 * r + c] = -2.0 * v;
    }
}

constexpr int kFinBlock = 64;
constexpr int kFinStride = 93;  // odd stride: conflict-free staging rows

// Word e (0..93) of the compact host record (VG_REC_LINEARIZE_F32, include/vgicp.h): the 90
// block values rounded to fp32 (north_star: fp32 H/b within 1e-4 of the fp64 oracle), the cost
// kept fp64 in words 90-91 (low word first) so LM accept/reject decisions see the same cost as
// the fp64 path, the inlier count as int32 in word 92, word 93 padding (8 B-aligned records).
__device__ __forceinline__ unsigned rec32_word(const double* o, int e) {
  if (e < 90) return __float_as_uint(__double2float_rn(o[e]));
  if (e < 92) {
    const unsigned long long c = (unsigned long long)__double_as_longlong(o[90]);
    return e == 90 ? (unsigned)c : (unsigned)(c >> 32);
  }
  return e == 92 ? (unsigned)(int)o[91] : 0u;
}

// K5: per-factor fixed-order sum of item partials + fp64 adjoint expansion.  LINEARIZE
// records (92 doubles, or 94 words when F32) are staged in shared memory and written out
// contiguously.
template <int F32>
__global__ void __launch_bounds__(kFinBlock)
    k_finalize(const FactorDev* __restrict__ factors, int fbase, int F,
               const double* __restrict__ partials, int mode, double* __restrict__ out,
               double2* __restrict__ gcost) {
  __shared__ double sh[kFinBlock * kFinStride];
  const int f0 = fbase + blockIdx.x * kFinBlock;
  const int fi = f0 + threadIdx.x;
  pdl_release();
  pdl_wait();  // item partials written by K4b
  if (mode != 0) {
    if (fi < F) finalize_one(factors[fi], fi, partials, mode, out, nullptr);
    return;
  }
  double gc = 0.0, gn = 0.0;
  if (fi < F) {
    const double* o = sh + threadIdx.x * kFinStride;
    finalize_one(factors[fi], fi, partials, mode, out, sh + threadIdx.x * kFinStride);
    const bool in = o[91] >= (double)factors[fi].min_inliers;
    gc = in ? o[90] : 0.0;
    gn = in ? 1.0 : 0.0;
  }
  if (gcost) {
    // gated cost + count of this CTA's 64 factors for the normal-equation assembly
    // (factor_graph.py:271-275): a fixed butterfly per warp, warp 0 then warp 1; one partial
    // per 64-factor window (stage boundaries are multiples of 64), summed by K6's cost unit
#pragma unroll
    for (int sft = 16; sft >= 1; sft >>= 1) {
      gc += __shfl_xor_sync(0xffffffffu, gc, sft);
      gn += __shfl_xor_sync(0xffffffffu, gn, sft);
    }
    __shared__ double2 wsum[kFinBlock / 32];
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = make_double2(gc, gn);
    __syncthreads();
    if (threadIdx.x == 0)
      gcost[f0 / kFinBlock] = make_double2(wsum[0].x + wsum[1].x, wsum[0].y + wsum[1].y);
  }
  __syncthreads();
  const int nf = min(kFinBlock, F - f0);
  if (F32) {
    unsigned* dst = reinterpret_cast<unsigned*>(out) + (size_t)f0 * 94;
    for (int k = threadIdx.x; k < nf * 94; k += kFinBlock) {
      const int r = k / 94;
      dst[k] = rec32_word(sh + r * kFinStride, k - r * 94);
    }
    return;
  }
  double* dst = out + (size_t)f0 * 92;
  for (int k = threadIdx.x; k < nf * 92; k += kFinBlock) {
    const int r = k / 92;
    dst[k] = sh[r * kFinStride + (k - r * 92)];
  }
}

// K5, warp per factor (batches with few factors or many items per factor): lane k sums value
// k over the factor's items in item order — the same additions as k_finalize's per-thread
// loop, so the records are bit-identical — then lane 0 expands and the warp writes out.
constexpr int kFinWarps = 4;
template <int F32>
__global__ void __launch_bounds__(kFinWarps * 32)
    k_finalize_warp(const FactorDev* __restrict__ factors, int fbase, int F,
                    const double* __restrict__ partials, int mode, double* __restrict__ out,
                    double2* __restrict__ gcost) {
  __shared__ double sh[kFinWarps][32 + 92];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int fi = fbase + blockIdx.x * kFinWarps + w;
  if (fi >= F) return;
  const FactorDev& f = factors[fi];
  const int ib = f.item_begin, ic = f.item_count;
  if (mode == 1 || mode == 3) {
    if (lane < 2) {
      double v = 0.0;
      for (int it = 0; it < ic; ++it) v += partials[2 * (size_t)(ib + it) + lane];
      out[2 * (size_t)fi + lane] = v;
    }
    return;
  }
  double v = 0.0;
  if (lane < 29)
    for (int it = 0; it < ic; ++it) v += partials[(size_t)(ib + it) * kPartialStride + lane];
  if (mode == 2) {
    if (lane < 29) out[(size_t)fi * 29 + lane] = v;
    return;
  }
  double* sw = sh[w];
  sw[lane] = v;
  __syncwarp();
  if (lane == 0) {
    expand_record(f, sw, sw + 32);
    if (gcost) {
      const bool in = sw[32 + 91] >= (double)f.min_inliers;
      gcost[fi] = make_double2(in ? sw[32 + 90] : 0.0, in ? 1.0 : 0.0);
    }
  }
  __syncwarp();
  if (F32) {
    unsigned* dst = reinterpret_cast<unsigned*>(out) + (size_t)fi * 94;
    for (int k = lane; k < 94; k += 32) dst[k] = rec32_word(sw + 32, k);
    return;
  }
  for (int k = lane; k < 92; k += 32) out[(size_t)fi * 92 + k] = sw[32 + k];
}


// ---- K3f: Gauss-Newton blocks from explicit per-point terms (linearize_from_terms with a
// MatchTerms that carries no voxel map, e.g. one made by the reference's own match_terms,
// registration.py:207-248).  The weights W and W d come from the caller; per point the kernel
// forms the target-frame terms about the source origin (lever arm x' = R mu, as K4b) and
// one block reduces them in a fixed order; thread 0 then expands the 29 sums like K5.
constexpr int kTermThreads = 256;
__global__ void __launch_bounds__(kTermThreads)
    k_terms_linearize(const double* __restrict__ mu, const double* __restrict__ W,
                      const double* __restrict__ wd, long long n, FactorDev f, double cost,
                      double inliers, double* __restrict__ out) {
  __shared__ double red[kTermThreads / 32][29];
  __shared__ double sums[32];
  __shared__ double rec[92];
  double acc[27];
#pragma unroll
  for (int k = 0; k < 27; ++k) acc[k] = 0.0;
  const double* R = f.T;
  for (long long i = threadIdx.x; i < n; i += kTermThreads) {
    const double px = mu[3 * i], py = mu[3 * i + 1], pz = mu[3 * i + 2];
    const double vx = fma(R[0], px, fma(R[1], py, R[2] * pz));
    const double vy = fma(R[3], px, fma(R[4], py, R[5] * pz));
    const double vz = fma(R[6], px, fma(R[7], py, R[8] * pz));
    const double* w = W + 9 * i;
    const double i00 = w[0], i01 = w[1], i02 = w[2], i11 = w[4], i12 = w[5], i22 = w[8];
    const double wd0 = wd[3 * i], wd1 = wd[3 * i + 1], wd2 = wd[3 * i + 2];
    // N = hat(x') W, P = N hat(x')^T, b' = [x' x Wd ; Wd] (J' = [-hat(x') | I]), as K4b
    const double N00 = fma(-vz, i01, vy * i02), N01 = fma(-vz, i11, vy * i12),
                 N02 = fma(-vz, i12, vy * i22);
    const double N10 = fma(vz, i00, -vx * i02), N11 = fma(vz, i01, -vx * i12),
                 N12 = fma(vz, i02, -vx * i22);
    const double N20 = fma(-vy, i00, vx * i01), N21 = fma(-vy, i01, vx * i11),
                 N22 = fma(-vy, i02, vx * i12);
    acc[0] += fma(-vz, N01, vy * N02);
    acc[1] += fma(vz, N00, -vx * N02);
    acc[2] += fma(-vy, N00, vx * N01);
    acc[3] += fma(vz, N10, -vx * N12);
    acc[4] += fma(-vy, N10, vx * N11);
    acc[5] += fma(-vy, N20, vx * N21);
    acc[6] += N00;
    acc[7] += N01;
    acc[8] += N02;
    acc[9] += N10;
    acc[10] += N11;
    acc[11] += N12;
    acc[12] += N20;
    acc[13] += N21;
    acc[14] += N22;
    acc[15] += i00;
    acc[16] += i01;
    acc[17] += i02;
    acc[18] += i11;
    acc[19] += i12;
    acc[20] += i22;
    acc[21] += fma(vy, wd2, -vz * wd1);
    acc[22] += fma(vz, wd0, -vx * wd2);
    acc[23] += fma(vx, wd1, -vy * wd0);
    acc[24] += wd0;
    acc[25] += wd1;
    acc[26] += wd2;
  }
  // fixed-order reduction: butterfly inside each warp, warps in index order
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 27; ++k) {
    double v = acc[k];
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
    if (lane == 0) red[wid][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < 27) {
    double v = 0.0;
    for (int q = 0; q < kTermThreads / 32; ++q) v += red[q][threadIdx.x];
    sums[threadIdx.x] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    sums[27] = cost;
    sums[28] = inliers;
    expand_record(f, sums, rec);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 92; k += kTermThreads) out[k] = rec[k];
}

// ---- K6: block-sparse normal equations (FactorGraph._assemble_dense, factor_graph.py:522-536)
// One warp per output unit: unit u < V is variable u's diagonal block (21, upper) + gradient
// (6); V <= u < V + P is the H block of variable pair u - V (36); unit -1 (the first block)
// sums the gated cost and count.
// A unit's contributions are listed in factor order (CSR, code = factor * 8 + role), and each
// lane sums its element in that order from 0.0, so the result is the reference's sequential
// per-block sum.  Roles: 0 source block (H_ii, b_i), 1 target block (H_jj, b_j), 2 H_ij as is,
// 3 H_ij transposed, 4 H_ij + H_ij^T (a factor whose two keys are the same variable).
// Records of factors below min_inliers have zero blocks (K5), so they add exact zeros.
__constant__ unsigned char kUpperRow[21] = {0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1,
                                            2, 2, 2, 2, 3, 3, 3, 4, 4, 5};
__constant__ unsigned char kUpperCol[21] = {0, 1, 2, 3, 4, 5, 1, 2, 3, 4, 5,
                                            2, 3, 4, 5, 3, 4, 5, 4, 5, 5};

__device__ __forceinline__ double asm_value(const double* __restrict__ r, int role, int k) {
  // k: element index of the unit (diag: 0..20 H upper, 21..26 g; pair: 0..35)
  switch (role) {
    case 0: return k < 21 ? __ldg(r + k) : __ldg(r + 78 + (k - 21));
    case 1: return k < 21 ? __ldg(r + 57 + k) : __ldg(r + 84 + (k - 21));
    case 2: return __ldg(r + 21 + k);
    case 3: return __ldg(r + 21 + 6 * (k % 6) + k / 6);
    default: {
      if (k >= 21) return 0.0;
      const int a = kUpperRow[k], c = kUpperCol[k];
      return __ldg(r + 21 + 6 * a + c) + __ldg(r + 21 + 6 * c + a);
    }
  }
}

constexpr int kAsmWarps = 1;  // one-warp CTAs: the long diagonal units do not hold CTA slots
#ifndef VG_K6_MLP
#define VG_K6_MLP 8
#endif
__global__ void __launch_bounds__(kAsmWarps * 32)
    k_assemble(const double* __restrict__ rec, const FactorDev* __restrict__ factors, int F,
               const int* __restrict__ begin, const int* __restrict__ codes, int V, int P,
               const int* __restrict__ pidx, const double2* __restrict__ gcost, int n_parts,
               double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int u = blockIdx.x * kAsmWarps + (threadIdx.x >> 5) - 1;  // unit -1: the cost
  pdl_release();
  pdl_wait();  // records and gated costs written by K5
  if (u >= V + P) return;
  if (u < 0) {
    // cost and count of the factors that pass their inlier gate (factor_graph.py:271-275),
    // from K5's per-window partials (64 factors, or 1 for the warp-per-factor K5): lane L sums
    // partials L, L + 32, ... in four interleaved chains, chains and lanes combined in a fixed
    // order (deterministic); this is the first block, so it starts first
    double c[4] = {0.0, 0.0, 0.0, 0.0}, n[4] = {0.0, 0.0, 0.0, 0.0};
    for (int f = lane; f < n_parts; f += 128) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
        if (f + 32 * a < n_parts) {
          const double2 v = __ldg(gcost + f + 32 * a);
          c[a] += v.x;
          n[a] += v.y;
        }
    }
    double cs = (c[0] + c[1]) + (c[2] + c[3]), ns = (n[0] + n[1]) + (n[2] + n[3]);
#pragma unroll
    for (int sft = 16; sft >= 1; sft >>= 1) {
      cs += __shfl_xor_sync(0xffffffffu, cs, sft);
      ns += __shfl_xor_sync(0xffffffffu, ns, sft);
    }
    if (lane == 0) {
      out[0] = cs;
      out[1] = ns;
    }
    return;
  }
  const int k0 = __ldg(begin + u), k1 = __ldg(begin + u + 1);
  const bool diag = u < V;
  const int nel = diag ? 27 : 36;
  double acc0 = 0.0, acc1 = 0.0;  // elements lane and lane + 32
  const bool has0 = lane < nel, has1 = lane + 32 < nel;
  // 32 codes per coalesced load and VG_K6_MLP contributions' values in flight per step (the
  // long diagonal units — ~100 contributions at config 5 — are chains of L2 round trips); the
  // additions stay in contribution order
  for (int kb = k0; kb < k1; kb += 32) {
    const int my_code = kb + lane < k1 ? __ldg(codes + kb + lane) : 0;
    const int nk = min(32, k1 - kb);
    for (int j = 0; j < nk; j += VG_K6_MLP) {
      double v0[VG_K6_MLP], v1[VG_K6_MLP];
#pragma unroll
      for (int q = 0; q < VG_K6_MLP; ++q) {
        const int code = __shfl_sync(0xffffffffu, my_code, (j + q) & 31);
        VG_DEVICE_CHECK(j + q >= nk || (code >> 3) < F, "K6: contribution of no factor");
        v0[q] = 0.0;
        v1[q] = 0.0;
        if (j + q < nk) {
          const double* r = rec + (size_t)(code >> 3) * 92;
          if (has0) v0[q] = asm_value(r, code & 7, lane);
          if (has1) v1[q] = asm_value(r, code & 7, lane + 32);
        }
      }
#pragma unroll
      for (int q = 0; q < VG_K6_MLP; ++q)
        if (j + q < nk) {
          acc0 += v0[q];
          acc1 += v1[q];
        }
    }
  }
  if (diag) {
    if (lane < 21) out[2 + (size_t)u * 21 + lane] = acc0;
    else if (lane < 27) out[2 + (size_t)V * 21 + (size_t)u * 6 + (lane - 21)] = acc0;
  } else {
    // pair block slot: the unit's own index, or its slot in a larger (e.g. global) layout
    const int slot = pidx ? __ldg(pidx + (u - V)) : u - V;
    double* o = out + 2 + (size_t)V * 27 + (size_t)slot * 36;
    o[lane] = acc0;
    if (has1) o[lane + 32] = acc1;
  }
}

// ---- pose composition on the device (geometry.py:47-144,231-237) ------------------------
// Mirrors Rotation's quaternion arithmetic operation for operation without FMA contraction,
// so T_ij matches pose_compose(pose_inverse(t_j), t_i) to the last bit except for numpy's
// 4-term dot order in the renormalisation.
struct Quat {
  double x, y, z, w;
};
__device__ __forceinline__ Quat q_normalize(Quat q) {
  const double n = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(q.x, q.x), __dmul_rn(q.y, q.y)),
                                                  __dmul_rn(q.z, q.z)),
                                         __dmul_rn(q.w, q.w)));
  return Quat{__ddiv_rn(q.x, n), __ddiv_rn(q.y, n), __ddiv_rn(q.z, n), __ddiv_rn(q.w, n)};
}
#define M_(a, b) __dmul_rn(a, b)
#define A_(a, b) __dadd_rn(a, b)
#define S_(a, b) __dsub_rn(a, b)
__device__ __forceinline__ Quat q_mul(Quat a, Quat b) {
  Quat r;
  r.x = S_(A_(A_(M_(a.w, b.x), M_(b.w, a.x)), M_(a.y, b.z)), M_(a.z, b.y));
  r.y = S_(A_(A_(M_(a.w, b.y), M_(b.w, a.y)), M_(a.z, b.x)), M_(a.x, b.z));
  r.z = S_(A_(A_(M_(a.w, b.z), M_(b.w, a.z)), M_(a.x, b.y)), M_(a.y, b.x));
  r.w = S_(S_(S_(M_(a.w, b.w), M_(a.x, b.x)), M_(a.y, b.y)), M_(a.z, b.z));
  return r;
}
__device__ __forceinline__ void q_apply(Quat q, const double v[3], double out[3]) {
  const double ux = q.x, uy = q.y, uz = q.z, w = q.w;
  const double tx = M_(2.0, S_(M_(uy, v[2]), M_(uz, v[1])));
  const double ty = M_(2.0, S_(M_(uz, v[0]), M_(ux, v[2])));
  const double tz = M_(2.0, S_(M_(ux, v[1]), M_(uy, v[0])));
  out[0] = S_(A_(A_(v[0], M_(w, tx)), M_(uy, tz)), M_(uz, ty));
  out[1] = S_(A_(A_(v[1], M_(w, ty)), M_(uz, tx)), M_(ux, tz));
  out[2] = S_(A_(A_(v[2], M_(w, tz)), M_(ux, ty)), M_(uy, tx));
}
__device__ __forceinline__ void q_matrix(Quat q, double* R) {
  const double xx = M_(q.x, q.x), yy = M_(q.y, q.y), zz = M_(q.z, q.z);
  const double xy = M_(q.x, q.y), xz = M_(q.x, q.z), yz = M_(q.y, q.z);
  const double wx = M_(q.w, q.x), wy = M_(q.w, q.y), wz = M_(q.w, q.z);
  R[0] = S_(1.0, M_(2.0, A_(yy, zz)));
  R[1] = M_(2.0, S_(xy, wz));
  R[2] = M_(2.0, A_(xz, wy));
  R[3] = M_(2.0, A_(xy, wz));
  R[4] = S_(1.0, M_(2.0, A_(xx, zz)));
  R[5] = M_(2.0, S_(yz, wx));
  R[6] = M_(2.0, S_(xz, wy));
  R[7] = M_(2.0, A_(yz, wx));
  R[8] = S_(1.0, M_(2.0, A_(xx, yy)));
}
#undef M_
#undef A_
#undef S_

// One thread composes one factor's T_ij; the 12 doubles are then stored warp-cooperatively
// (staged in shared memory, 32 lanes writing contiguous 8 B words of ~3 records per store) so
// the factor table and item headers take ~3x fewer L2 sectors per store than per-thread
// 96 B writes (r02 ncu of the per-thread version: lg_throttle 24% + drain 30% of stalls).
__device__ __forceinline__ void compose_T(const double* __restrict__ pi,
                                          const double* __restrict__ pj, double* T);
constexpr int kComposeThreads = 128;
__global__ void __launch_bounds__(kComposeThreads)
    k_compose(FactorDev* __restrict__ factors, int F, const double* __restrict__ poses,
              ItemHdr* __restrict__ hdrs) {
  __shared__ double sT[kComposeThreads][13];
  const int fi = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, wbase = fi - lane;
  double* T = sT[threadIdx.x];
  pdl_release();
  pdl_wait();  // the previous step's K5 still reads T_ij
  // (item_begin, item_count, var_source, var_target): one 16 B load
  const int4 meta =
      fi < F ? *reinterpret_cast<const int4*>(&factors[fi].item_begin) : make_int4(0, 0, 0, 0);
  if (fi < F) compose_T(poses + 8 * (size_t)meta.z, poses + 8 * (size_t)meta.w, T);
  __syncwarp();
  const int nw = min(32, F - wbase);  // factors in this warp
  for (int e = lane; e < 12 * 32; e += 32) {
    const int j = e / 12, q = e - 12 * j;
    const int ib = __shfl_sync(0xffffffffu, meta.x, j);
    const int ic = __shfl_sync(0xffffffffu, meta.y, j);
    if (j < nw) {
      const double v = sT[threadIdx.x - lane + j][q];
      factors[wbase + j].T[q] = v;
      if (ic > 0) hdrs[ib].T[q] = v;  // empty sources have no item
    }
  }
  if (fi < F)  // factors split into several items (> 1,024 source points): rare
    for (int it = 1; it < meta.y; ++it)
      for (int q = 0; q < 12; ++q) hdrs[meta.x + it].T[q] = T[q];
}

__device__ __forceinline__ void compose_T(const double* __restrict__ pi,
                                          const double* __restrict__ pj, double* T) {
  // pose_inverse(t_j): rotation inverse (renormalised by the constructor), t = -R^-1 t_j
  Quat qj = q_normalize(Quat{-pj[0], -pj[1], -pj[2], pj[3]});
  double tj[3] = {pj[4], pj[5], pj[6]}, tinv[3];
  q_apply(qj, tj, tinv);
  tinv[0] = -tinv[0];
  tinv[1] = -tinv[1];
  tinv[2] = -tinv[2];
  // pose_compose(inv_j, t_i)
  Quat qi{pi[0], pi[1], pi[2], pi[3]};
  Quat q = q_normalize(q_mul(qj, qi));
  double ti[3] = {pi[4], pi[5], pi[6]}, tt[3];
  q_apply(qj, ti, tt);
  q_matrix(q, T);
  T[9] = __dadd_rn(tt[0], tinv[0]);
  T[10] = __dadd_rn(tt[1], tinv[1]);
  T[11] = __dadd_rn(tt[2], tinv[2]);
}

__global__ void k_spread_T(const FactorDev* __restrict__ factors, int F, ItemHdr* __restrict__ hdrs) {
  const int fi = blockIdx.x * blockDim.x + threadIdx.x;
  if (fi >= F) return;
  const FactorDev& f = factors[fi];
  for (int it = 0; it < f.item_count; ++it)
    for (int q = 0; q < 12; ++q) hdrs[f.item_begin + it].T[q] = f.T[q];
}

// ---- K3: transform + lookup (GaussianVoxelMap.lookup / overlap_rate) ----------------------
__global__ void k_lookup(CloudView cv, MapView mv, const double* __restrict__ Tp,
                         long long* __restrict__ rows, unsigned long long* __restrict__ hits) {
  double R[9], t[3];
  load_T(Tp, R, t);
  unsigned long long local = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cv.n;
       i += (long long)gridDim.x * blockDim.x) {
    double px, py, pz;
    float4 pa;
    load_point(cv, i, px, py, pz, pa);
    double x, y, z;
    transform(R, t, px, py, pz, x, y, z);
    const Query q = make_query(mv, floor_div(x, mv.res, mv.inv_res, mv.pow2),
                               floor_div(y, mv.res, mv.inv_res, mv.pow2),
                               floor_div(z, mv.res, mv.inv_res, mv.pow2), mv.kmode);
    const int slot = probe_query(mv, q);
    const long long row = slot < 0 ? -1 : slot_row(mv, slot, mv.kmode);
    if (rows) rows[i] = row;
    local += (row >= 0);
  }
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) local += __shfl_xor_sync(0xffffffffu, local, s);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(hits, local);  // integer: deterministic
}

// ---- K3t: per-point match terms (match_terms materialised for API parity) -----------------
__global__ void k_terms(CloudView cv, MapView mv, const double* __restrict__ Tp,
                        long long* __restrict__ rows, double* __restrict__ moved,
                        double* __restrict__ dout, double* __restrict__ wout,
                        double* __restrict__ wdout, double* __restrict__ pcost,
                        long long* __restrict__ pinl) {
  double R[9], t[3];
  load_T(Tp, R, t);
  double csum = 0.0;
  long long isum = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cv.n;
       i += (long long)gridDim.x * blockDim.x) {
    double px, py, pz;
    float4 pa;
    load_point(cv, i, px, py, pz, pa);
    double x, y, z;
    transform(R, t, px, py, pz, x, y, z);
    moved[3 * i] = x;
    moved[3 * i + 1] = y;
    moved[3 * i + 2] = z;
    const Query q = make_query(mv, floor_div(x, mv.res, mv.inv_res, mv.pow2),
                               floor_div(y, mv.res, mv.inv_res, mv.pow2),
                               floor_div(z, mv.res, mv.inv_res, mv.pow2), mv.kmode);
    const int slot = probe_query(mv, q);
    if (slot < 0) {
      rows[i] = -1;
      for (int k = 0; k < 3; ++k) dout[3 * i + k] = 0.0, wdout[3 * i + k] = 0.0;
      for (int k = 0; k < 9; ++k) wout[9 * i + k] = 0.0;
      continue;
    }
    rows[i] = slot_row(mv, slot, mv.kmode);
    PointTerms o;
    point_terms(R, cv, i, mv.recs + rec_index(mv, slot, mv.kmode), x, y, z, t, o);
    const int sym[9] = {0, 1, 2, 1, 3, 4, 2, 4, 5};
    for (int k = 0; k < 3; ++k) dout[3 * i + k] = o.d[k], wdout[3 * i + k] = o.wd[k];
    for (int k = 0; k < 9; ++k) wout[9 * i + k] = o.W[sym[k]];
    csum += o.cost;
    ++isum;
  }
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    csum += __shfl_xor_sync(0xffffffffu, csum, s);
    isum += __shfl_xor_sync(0xffffffffu, isum, s);
  }
  __shared__ double sc[32];
  __shared__ long long si[32];
  const int wid = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) sc[wid] = csum, si[wid] = isum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double c = 0.0;
    long long n = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) c += sc[k], n += si[k];
    pcost[blockIdx.x] = c;
    pinl[blockIdx.x] = n;
  }
}

}  // namespace vg

using namespace vg;

static int grid_for(long long n, int threads, int cap) {
  long long g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

int launch_lookup(vg_ctx* ctx, const CloudView& cv, const MapView& mv, const double* T_dev,
                  long long* rows_dev, unsigned long long* hits_dev) {
  if (cv.n == 0) return 0;
  k_lookup<<<grid_for(cv.n, 256, 148 * 16), 256, 0, ctx->stream>>>(cv, mv, T_dev, rows_dev,
                                                                   hits_dev);
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  return 0;
}

int launch_terms(vg_ctx* ctx, const CloudView& cv, const MapView& mv, const double* T_dev,
                 long long* rows, double* moved, double* d, double* w, double* wd,
                 double* partial_cost, long long* partial_inl, int nblocks) {
  if (cv.n == 0) return 0;
  k_terms<<<nblocks, 256, 0, ctx->stream>>>(cv, mv, T_dev, rows, moved, d, w, wd, partial_cost,
                                            partial_inl);
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  return 0;
}

int launch_terms_linearize(vg_ctx* ctx, const double* mu_dev, const double* W_dev,
                           const double* wd_dev, long long n, const FactorDev& f, double cost,
                           double inliers, double* out_dev) {
  k_terms_linearize<<<1, kTermThreads, 0, ctx->stream>>>(mu_dev, W_dev, wd_dev, n, f, cost,
                                                         inliers, out_dev);
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  return 0;
}

int launch_compose(vg_ctx* ctx, vg_batch* b, const double* poses_dev) {
  if (b->F == 0) return 0;
  VG_CUDA(launch_pdl(k_compose, dim3(grid_for(b->F, kComposeThreads, 1 << 30)), dim3(kComposeThreads), 0, ctx->stream,
                     b->factors, (int)b->F, poses_dev, b->hdrs));
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  return 0;
}

int launch_spread_T(vg_ctx* ctx, vg_batch* b) {
  if (b->F == 0) return 0;
  k_spread_T<<<grid_for(b->F, 128, 1 << 30), 128, 0, ctx->stream>>>(b->factors, (int)b->F,
                                                                    b->hdrs);
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  return 0;
}

int launch_finalize_range(vg_ctx* ctx, vg_batch* b, int mode, void* out_dev, int f0, int f1,
                          int f32) {
  if (f1 <= f0) return 0;
  double* out = static_cast<double*>(out_dev);
  double2* gc = mode == 0 ? b->asm_gcost : nullptr;
  const FactorDev* fac = b->factors;
  const double* part = b->partials;
  // few factors or long item lists: a warp per factor sums the items in parallel lanes
  if (b->F < 4096 || b->num_items > 4 * b->F) {
    const dim3 grid((f1 - f0 + kFinWarps - 1) / kFinWarps), block(kFinWarps * 32);
    if (f32 && mode == 0)
      k_finalize_warp<1><<<grid, block, 0, ctx->stream>>>(fac, f0, f1, part, mode, out, gc);
    else
      k_finalize_warp<0><<<grid, block, 0, ctx->stream>>>(fac, f0, f1, part, mode, out, gc);
    ctx->launches++;
    VG_CUDA(cudaGetLastError());
    return 0;
  }
  const dim3 grid((f1 - f0 + kFinBlock - 1) / kFinBlock), block(kFinBlock);
  if (gc && f0 % kFinBlock) return vg_cuda_fail(cudaErrorInvalidValue, "K5 window alignment");
  if (f32 && mode == 0)
    VG_CUDA(launch_pdl(k_finalize<1>, grid, block, 0, ctx->stream, fac, f0, f1, part, mode, out, gc));
  else
    VG_CUDA(launch_pdl(k_finalize<0>, grid, block, 0, ctx->stream, fac, f0, f1, part, mode, out, gc));
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  return 0;
}

int launch_finalize(vg_ctx* ctx, vg_batch* b, int mode, void* out_dev, int f32) {
  return launch_finalize_range(ctx, b, mode, out_dev, 0, (int)b->F, f32);
}

int launch_assemble(vg_ctx* ctx, vg_batch* b, const double* rec, double* out_dev) {
  const int units = (int)(b->asm_vars + b->asm_pairs_n) + 1;  // + the cost unit
  VG_CUDA(launch_pdl(k_assemble, dim3((units + kAsmWarps - 1) / kAsmWarps), dim3(kAsmWarps * 32),
                     0, ctx->stream, rec, (const FactorDev*)b->factors, (int)b->F,
                     (const int*)b->asm_begin, (const int*)b->asm_codes, (int)b->asm_vars,
                     (int)b->asm_pairs_n, (const int*)b->asm_pidx,
                     (const double2*)b->asm_gcost, (int)b->asm_gparts, out_dev));
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  return 0;
}
