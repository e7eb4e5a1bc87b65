// map_build.cu — K1 voxel keys, cloud packing, K2 Gaussian voxel-map build + hash insert.
//
// build_voxelmap (registration.py:74-98) on the device, bit-identical to the reference:
//   keys (preprocess.py:68-70) -> stable radix sort of (key, index) (== np.unique order and
//   np.add.at's index order inside every cell) -> run-length encode -> one thread per cell
//   sums its members sequentially in index order with correctly rounded fp64 adds (no FMA),
//   exactly the rounding sequence of np.add.at + true division.
// The fp64 arrays are kept on the device for export; the hot path reads the 64 B slots.
#include <algorithm>
#include <climits>
#include <vector>

#include <cstdio>
#include <cstdlib>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>

#include <cuda.h>

#include "common.cuh"
#include "internal.h"

namespace vg {

__global__ void k_pack_keys(const double* __restrict__ xyz, long long n, double res,
                            long long* __restrict__ keys, int* __restrict__ idx) {
  const double inv = 1.0 / res;
  int e2 = 0;
  const int pow2 = (frexp(res, &e2) == 0.5) ? 1 : 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    keys[i] = pack_key(floor_div(xyz[3 * i], res, inv, pow2),
                       floor_div(xyz[3 * i + 1], res, inv, pow2),
                       floor_div(xyz[3 * i + 2], res, inv, pow2));
    if (idx) idx[i] = (int)i;
  }
}

// Bounds of the packed keys (K2's first pass, with k_pack_keys' output): per block a
// shared-memory min / max of the key and of its three fields as the reference's round trip
// decodes them (hi = key >> 42 arithmetic, mid = bits 21..41, lo = bits 0..20; the signed int64
// order of keys is the lexicographic order of (hi, mid, lo)), then 64-bit atomics.
// b[0..7] = min hi, max hi, min mid, max mid, min lo, max lo, min key, max key.
__global__ void k_key_bounds(const long long* __restrict__ keys, long long n,
                             long long* __restrict__ b) {
  long long v[8] = {LLONG_MAX, LLONG_MIN, LLONG_MAX, LLONG_MIN,
                    LLONG_MAX, LLONG_MIN, LLONG_MAX, LLONG_MIN};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long k = keys[i];
    const long long f[4] = {k >> 42, (k >> 21) & ((1LL << 21) - 1), k & ((1LL << 21) - 1), k};
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      v[2 * a] = min(v[2 * a], f[a]);
      v[2 * a + 1] = max(v[2 * a + 1], f[a]);
    }
  }
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      const long long o = __shfl_xor_sync(0xffffffffu, v[a], s);
      v[a] = (a & 1) ? max(v[a], o) : min(v[a], o);
    }
  // one atomic per value and block (a grid of a few hundred blocks): per-warp atomics on the
  // eight shared addresses serialise into milliseconds
  __shared__ long long sw[32][8];
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int a = 0; a < 8; ++a) sw[w][a] = v[a];
  __syncthreads();
  if (threadIdx.x < 8) {
    const int a = threadIdx.x;
    long long r = sw[0][a];
    for (int q = 1; q < nw; ++q) r = (a & 1) ? max(r, sw[q][a]) : min(r, sw[q][a]);
    if (a & 1) atomicMax(b + a, r);
    else atomicMin(b + a, r);
  }
}

__global__ void k_bounds_init(long long* __restrict__ b) {
  if (threadIdx.x < 8) b[threadIdx.x] = (threadIdx.x & 1) ? LLONG_MIN : LLONG_MAX;
}

// order-preserving 32-bit local key: fields relative to the bounds, (hi, mid, lo) packed
// most-significant first in sh / sm / 0 bit positions
__global__ void k_local_keys(const long long* __restrict__ keys, long long n,
                             const long long* __restrict__ b, int sh, int sm,
                             unsigned* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long k = keys[i];
    out[i] = (sh < 32 ? (unsigned)((k >> 42) - b[0]) << sh : 0u) |
             ((unsigned)(((k >> 21) & ((1LL << 21) - 1)) - b[2]) << sm) |
             (unsigned)((k & ((1LL << 21) - 1)) - b[4]);
  }
}

// the packed key of each unique local key (k_local_keys inverted)
__global__ void k_unlocal_keys(const unsigned* __restrict__ local, const int* __restrict__ m,
                               const long long* __restrict__ b, int sh, int sm,
                               long long* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < *m; i += gridDim.x * blockDim.x) {
    const unsigned u = local[i];
    const long long hi = (long long)(sh < 32 ? u >> sh : 0u) + b[0];
    const long long mid = (long long)((u >> sm) & ((1u << (sh - sm)) - 1u)) + b[2];
    const long long lo = (long long)(sm ? u & ((1u << sm) - 1u) : 0u) + b[4];
    out[i] = (long long)((unsigned long long)hi << 42) | (mid << 21) | lo;
  }
}

// fp64 AoS (n x 3 points, n x 9 covariances) -> fp32 xyz + fp64 covariance SoA
__global__ void k_cloud_pack(const double* __restrict__ xyz, const double* __restrict__ cov,
                             long long n, float4* __restrict__ a, double2* __restrict__ c0,
                             double2* __restrict__ c1, double2* __restrict__ c2) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    a[i] = make_float4((float)xyz[3 * i], (float)xyz[3 * i + 1], (float)xyz[3 * i + 2], 0.f);
    if (cov) {
      const double* C = cov + 9 * i;
      c0[i] = make_double2(C[0], C[1]);
      c1[i] = make_double2(C[2], C[4]);
      c2[i] = make_double2(C[5], C[8]);
    }
  }
}

// Plane form of a source covariance: C = alpha I - kappa n n^T (|n| = 1), which every
// covariance estimate_covariances makes (V diag(eps, 1, 1) V^T = I - (1 - eps) n n^T;
// degenerate: eps I), so R C R^T = alpha I - kappa (R n)(R n)^T costs 21 fp64 ops per
// correspondence in K4b instead of 45.  alpha and kappa follow from the trace and the
// Frobenius norm (alpha is the double eigenvalue), n from the largest column of
// alpha I - C; a point is accepted when the reconstruction matches C to 1e-13 of its largest
// entry (the fit itself is accurate to ~1e-16), otherwise the cloud keeps the general form.  Layout: p0 = (n0, n1), p1 = (n2, kappa), p2 = (alpha, 0).
__global__ void k_plane_fit(const double* __restrict__ cov, long long n, double2* __restrict__ p0,
                            double2* __restrict__ p1, double2* __restrict__ p2,
                            unsigned* __restrict__ fails) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double* C = cov + 9 * i;
    // fit the symmetric part (V diag V^T is symmetric only to the last bit); the acceptance
    // test below checks all nine entries
    const double a00 = C[0], a11 = C[4], a22 = C[8];
    const double a01 = 0.5 * (C[1] + C[3]), a02 = 0.5 * (C[2] + C[6]), a12 = 0.5 * (C[5] + C[7]);
    bool ok = true;
    double alpha = 0.0, kappa = 0.0, n0 = 1.0, n1 = 0.0, n2 = 0.0;
    if (a01 == 0.0 && a02 == 0.0 && a12 == 0.0 && a00 == a11 && a11 == a22 && C[1] == 0.0 &&
        C[2] == 0.0 && C[5] == 0.0) {
      alpha = a00;  // isotropic (degenerate neighbourhoods: eps I)
    } else {
      const double t = a00 + a11 + a22;
      const double q = a00 * a00 + a11 * a11 + a22 * a22 + 2.0 * (a01 * a01 + a02 * a02 + a12 * a12);
      alpha = (4.0 * t + sqrt(fmax(24.0 * q - 8.0 * t * t, 0.0))) / 12.0;
      kappa = 3.0 * alpha - t;
      const double m[3][3] = {{alpha - a00, -a01, -a02}, {-a01, alpha - a11, -a12},
                              {-a02, -a12, alpha - a22}};
      int k = 0;
      if (m[1][1] > m[k][k]) k = 1;
      if (m[2][2] > m[k][k]) k = 2;
      if (!(kappa > 0.0) || !(m[k][k] > 0.0)) {
        ok = false;
      } else {
        const double sc = 1.0 / sqrt(kappa * m[k][k]);
        n0 = m[0][k] * sc;
        n1 = m[1][k] * sc;
        n2 = m[2][k] * sc;
        const double nv[3] = {n0, n1, n2};
        double r = 0.0;
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b)
            r = fmax(r, fabs((a == b ? alpha : 0.0) - kappa * nv[a] * nv[b] - C[3 * a + b]));
        // relative to the matrix scale, so scaled covariances are held to the same accuracy
        double cmax = 0.0;
        for (int a = 0; a < 9; ++a) cmax = fmax(cmax, fabs(C[a]));
        ok = r <= 1e-13 * cmax;
      }
    }
    if (!ok) atomicAdd(fails, 1u);
    p0[i] = make_double2(n0, n1);
    p1[i] = make_double2(n2, kappa);
    p2[i] = make_double2(alpha, 0.0);
  }
}

// one thread per cell: mean then scatter, both sequential in index order (np.add.at).  The
// member loads are issued kCellBatch at a time ahead of the in-order additions, so a cell of
// thousands of points (coarse maps near the sensor) pays the dependent fp64 adds, not one
// L2 round trip per member.
constexpr int kCellBatch = 8;
#ifndef VG_BIG_CELL
#define VG_BIG_CELL 16
#endif
constexpr int kBigCell = VG_BIG_CELL;  // cells with at least this many points: one warp per cell
__global__ void k_cell_stats(const int* __restrict__ offsets, const int* __restrict__ counts,
                             const int* __restrict__ perm, const double* __restrict__ xyz,
                             const double* __restrict__ cov, int m, double* __restrict__ means,
                             double* __restrict__ covs, long long* __restrict__ cnt_out) {
  const int cidx = blockIdx.x * blockDim.x + threadIdx.x;
  if (cidx >= m) return;
  const int off = offsets[cidx], cnt = counts[cidx];
  if (cnt >= kBigCell) return;  // k_cell_stats_big
  double sx = 0.0, sy = 0.0, sz = 0.0;
  for (int j0 = off; j0 < off + cnt; j0 += kCellBatch) {
    const int nb = min(kCellBatch, off + cnt - j0);
    double px[kCellBatch], py[kCellBatch], pz[kCellBatch];
#pragma unroll
    for (int u = 0; u < kCellBatch; ++u) {
      if (u < nb) {
        const int i = perm[j0 + u];
        px[u] = xyz[3 * (size_t)i];
        py[u] = xyz[3 * (size_t)i + 1];
        pz[u] = xyz[3 * (size_t)i + 2];
      }
    }
#pragma unroll
    for (int u = 0; u < kCellBatch; ++u) {
      if (u < nb) {
        sx = add_rn(sx, px[u]);
        sy = add_rn(sy, py[u]);
        sz = add_rn(sz, pz[u]);
      }
    }
  }
  const double dc = (double)cnt;
  const double mx = __ddiv_rn(sx, dc), my = __ddiv_rn(sy, dc), mz = __ddiv_rn(sz, dc);
  double acc[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) acc[k] = 0.0;
  constexpr int kB = kCellBatch / 2;
  for (int j0 = off; j0 < off + cnt; j0 += kB) {
    const int nb = min(kB, off + cnt - j0);
    double c3[kB][3], cv[kB][9];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      if (u < nb) {
        const int i = perm[j0 + u];
        c3[u][0] = sub_rn(xyz[3 * (size_t)i], mx);
        c3[u][1] = sub_rn(xyz[3 * (size_t)i + 1], my);
        c3[u][2] = sub_rn(xyz[3 * (size_t)i + 2], mz);
#pragma unroll
        for (int k = 0; k < 9; ++k) cv[u][k] = cov[9 * (size_t)i + k];
      }
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      if (u < nb) {
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int c = 0; c < 3; ++c)
            acc[3 * r + c] = add_rn(acc[3 * r + c],
                                    add_rn(cv[u][3 * r + c], mul_rn(c3[u][r], c3[u][c])));
      }
    }
  }
  means[3 * cidx] = mx;
  means[3 * cidx + 1] = my;
  means[3 * cidx + 2] = mz;
#pragma unroll
  for (int k = 0; k < 9; ++k) covs[9 * (size_t)cidx + k] = __ddiv_rn(acc[k], dc);
  cnt_out[cidx] = cnt;
}

// one warp per big cell (>= kBigCell = 16 points; coarse maps near the sensor hold thousands;
// thresholds 32/48/96 measured 5-17% slower for config 2's three maps).
// The additions stay sequential in index order — lanes 0-2 carry the three position sums,
// lanes 0-8 the nine covariance sums — while all 32 lanes load the next 32 members and form
// their terms (C_k + (p_k - mu)(p_k - mu)^T, the same correctly rounded operations as the
// per-thread kernel) into shared memory, so the result is bit-identical and a cell costs one
// dependent fp64 add per member instead of a single thread's whole instruction stream.
constexpr int kBigWarps = 4;
__global__ void __launch_bounds__(kBigWarps * 32)
    k_cell_stats_big(const int* __restrict__ offsets, const int* __restrict__ counts,
                     const int* __restrict__ perm, const double* __restrict__ xyz,
                     const double* __restrict__ cov, int m, double* __restrict__ means,
                     double* __restrict__ covs, long long* __restrict__ cnt_out) {
  __shared__ double term[kBigWarps][9][33];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int cidx = blockIdx.x * kBigWarps + wib;
  if (cidx >= m) return;
  const int off = offsets[cidx], cnt = counts[cidx];
  if (cnt < kBigCell) return;
  double (*t)[33] = term[wib];
  double acc = 0.0;  // lane c < 3: position sum c; later lane k < 9: covariance sum k
  for (int j0 = off; j0 < off + cnt; j0 += 32) {
    const int nb = min(32, off + cnt - j0);
    if (lane < nb) {
      const int i = perm[j0 + lane];
      t[0][lane] = xyz[3 * (size_t)i];
      t[1][lane] = xyz[3 * (size_t)i + 1];
      t[2][lane] = xyz[3 * (size_t)i + 2];
    }
    __syncwarp();
    if (lane < 3)
      for (int u = 0; u < nb; ++u) acc = add_rn(acc, t[lane][u]);
    __syncwarp();
  }
  const double dc = (double)cnt;
  const double mean_l = __ddiv_rn(acc, dc);
  const double mx = __shfl_sync(0xffffffffu, mean_l, 0), my = __shfl_sync(0xffffffffu, mean_l, 1),
               mz = __shfl_sync(0xffffffffu, mean_l, 2);
  acc = 0.0;
  for (int j0 = off; j0 < off + cnt; j0 += 32) {
    const int nb = min(32, off + cnt - j0);
    if (lane < nb) {
      const int i = perm[j0 + lane];
      const double c3[3] = {sub_rn(xyz[3 * (size_t)i], mx), sub_rn(xyz[3 * (size_t)i + 1], my),
                            sub_rn(xyz[3 * (size_t)i + 2], mz)};
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          t[3 * r + c][lane] = add_rn(cov[9 * (size_t)i + 3 * r + c], mul_rn(c3[r], c3[c]));
    }
    __syncwarp();
    if (lane < 9)
      for (int u = 0; u < nb; ++u) acc = add_rn(acc, t[lane][u]);
    __syncwarp();
  }
  if (lane < 3) means[3 * cidx + lane] = lane == 0 ? mx : (lane == 1 ? my : mz);
  if (lane < 9) covs[9 * (size_t)cidx + lane] = __ddiv_rn(acc, dc);
  if (lane == 0) cnt_out[cidx] = cnt;
}

// ---- voxel downsampling (preprocess.py:73-119) -------------------------------------------
// Grouping is the map build's: stable radix sort of (key, index) + run-length encode, so each
// group lists its members in scan order (np.argsort(kind="stable") + np.split).  One thread
// per group then reproduces the reference's arithmetic in its order: exact stamp min/max,
// the running-mean split rule in scan order (:100-111), sequential fp64 position sums from
// 0.0 (`points[cell].mean(axis=0)`) and NumPy's pairwise stamp sum (`stamps[cell].mean()`).

// NumPy's float64 pairwise add.reduce over a contiguous array: < 8 elements sequentially,
// <= 128 with 8 interleaved accumulators, above that split at a multiple of 8 and recurse
// (evaluated here with explicit stacks: left subtree, right subtree, then their sum).
__device__ double pairwise_leaf(const double* a, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = add_rn(res, a[i]);
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = add_rn(r[j], a[i + j]);
  double res = add_rn(add_rn(add_rn(r[0], r[1]), add_rn(r[2], r[3])),
                      add_rn(add_rn(r[4], r[5]), add_rn(r[6], r[7])));
  for (; i < n; ++i) res = add_rn(res, a[i]);
  return res;
}

__device__ double pairwise_sum(const double* a, int n) {
  if (n <= 128) return pairwise_leaf(a, n);
  int2 ops[96];  // (offset, n); n < 0 marks "add the top two values"
  double vals[48];
  int no = 0, nv = 0;
  ops[no++] = make_int2(0, n);
  while (no > 0) {
    const int2 op = ops[--no];
    if (op.y < 0) {
      const double r = vals[--nv];
      vals[nv - 1] = add_rn(vals[nv - 1], r);
    } else if (op.y <= 128) {
      vals[nv++] = pairwise_leaf(a + op.x, op.y);
    } else {
      int n2 = op.y / 2;
      n2 -= n2 % 8;
      ops[no++] = make_int2(0, -1);
      ops[no++] = make_int2(op.x + n2, op.y - n2);
      ops[no++] = make_int2(op.x, n2);
    }
  }
  return vals[0];
}

// per group: cell of every member (0 primary, 1 overflow) and the number of output cells
__global__ void k_ds_assign(const int* __restrict__ offsets, const int* __restrict__ counts,
                            const int* __restrict__ perm, const double* __restrict__ stamps,
                            int m, double tol, unsigned char* __restrict__ cell,
                            int* __restrict__ ncell) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= m) return;
  const int off = offsets[g], cnt = counts[g];
  double tmin = stamps[perm[off]], tmax = tmin;
  for (int j = off + 1; j < off + cnt; ++j) {
    const double t = stamps[perm[j]];
    tmin = t < tmin ? t : tmin;
    tmax = t > tmax ? t : tmax;
  }
  if (sub_rn(tmax, tmin) <= tol) {
    for (int j = off; j < off + cnt; ++j) cell[j] = 0;
    ncell[g] = 1;
    return;
  }
  long long n0 = 0, n1 = 0;
  double s0 = 0.0;
  for (int j = off; j < off + cnt; ++j) {
    const double t = stamps[perm[j]];
    const bool primary = n0 == 0 || fabs(sub_rn(t, __ddiv_rn(s0, (double)n0))) <= tol;
    cell[j] = primary ? 0 : 1;
    if (primary) {
      ++n0;
      s0 = add_rn(s0, t);
    } else {
      ++n1;
    }
  }
  ncell[g] = n1 > 0 ? 2 : 1;
}

// per group: the mean position and stamp of each of its cells, written at its output slot;
// `scratch` (one double per point) holds each cell's stamps contiguously for the pairwise sum
__global__ void k_ds_emit(const int* __restrict__ offsets, const int* __restrict__ counts,
                          const int* __restrict__ perm, const double* __restrict__ xyz,
                          const double* __restrict__ stamps, const unsigned char* __restrict__ cell,
                          const int* __restrict__ ncell, const int* __restrict__ out_off, int m,
                          double* __restrict__ scratch, double* __restrict__ xyz_out,
                          double* __restrict__ stamps_out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= m) return;
  const int off = offsets[g], cnt = counts[g];
  int o = out_off[g];
  int base = off;
  for (int c = 0; c < ncell[g]; ++c) {
    double sx = 0.0, sy = 0.0, sz = 0.0;
    int k = 0;
    for (int j = off; j < off + cnt; ++j) {
      if (cell[j] != c) continue;
      const int i = perm[j];
      sx = add_rn(sx, xyz[3 * (size_t)i]);
      sy = add_rn(sy, xyz[3 * (size_t)i + 1]);
      sz = add_rn(sz, xyz[3 * (size_t)i + 2]);
      scratch[base + k++] = stamps[i];
    }
    const double dk = (double)k;
    xyz_out[3 * (size_t)o] = __ddiv_rn(sx, dk);
    xyz_out[3 * (size_t)o + 1] = __ddiv_rn(sy, dk);
    xyz_out[3 * (size_t)o + 2] = __ddiv_rn(sz, dk);
    stamps_out[o] = __ddiv_rn(add_rn(0.0, pairwise_sum(scratch + base, k)), dk);
    base += k;
    ++o;
  }
}

// one thread per cell: insert key into the bucketized hash (home bucket first, then the next
// bucket; CAS on the key), then write the 128 B record (fp64 Gaussian + reference row) at the
// slot (kmode 1) or at the row with a slot -> row entry (kmode 0).
__global__ void k_hash_insert(const long long* __restrict__ keys, const double* __restrict__ means,
                              const double* __restrict__ covs, int m, MapView mv,
                              long long* __restrict__ pkeys, int* __restrict__ prows,
                              unsigned* __restrict__ pkeys32, VoxelRec* __restrict__ recs) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  const long long key = keys[r];
  size_t h = 0;
  if (mv.kmode) {
    const long long dx = (key >> 42) - kKeyOffset;
    const long long dy = ((key >> 21) & ((1LL << 21) - 1)) - kKeyOffset;
    const long long dz = (key & ((1LL << 21) - 1)) - kKeyOffset;
    const unsigned k32 =
        (unsigned)(dx - mv.bx) | ((unsigned)(dy - mv.by) << 11) | ((unsigned)(dz - mv.bz) << 22);
    bool placed = false;
    unsigned probes = 0;
    for (unsigned b = bucket32(k32, mv.shift); !placed; b = (b + 1) & mv.mask, ++probes) {
      VG_DEVICE_CHECK(probes <= mv.mask, "k_hash_insert: table full (32-bit keys)");
      for (int j = 0; j < kBucket32 && !placed; ++j) {
        h = (size_t)b * kBucket32 + j;
        placed = atomicCAS(pkeys32 + h, kEmpty32, k32) == kEmpty32;
      }
    }
  } else {
    bool placed = false;
    unsigned probes = 0;
    for (unsigned b = slot_of(key, mv.shift); !placed; b = (b + 1) & mv.mask, ++probes) {
      VG_DEVICE_CHECK(probes <= mv.mask, "k_hash_insert: table full (int64 keys)");
      for (int j = 0; j < kBucket && !placed; ++j) {
        h = (size_t)b * kBucket + j;
        const unsigned long long prev =
            atomicCAS(reinterpret_cast<unsigned long long*>(pkeys + h),
                      (unsigned long long)mv.empty_key, (unsigned long long)key);
        placed = prev == (unsigned long long)mv.empty_key;
      }
    }
    prows[h] = r;
  }
  VoxelRec v;
  v.mean[0] = means[3 * r];
  v.mean[1] = means[3 * r + 1];
  v.mean[2] = means[3 * r + 2];
  const double* C = covs + 9 * (size_t)r;
  v.cov[0] = C[0];
  v.cov[1] = C[1];
  v.cov[2] = C[2];
  v.cov[3] = C[4];
  v.cov[4] = C[5];
  v.cov[5] = C[8];
  v.row = r;
#pragma unroll
  for (int k = 0; k < 6; ++k) v.pad[k] = 0.0;
  VG_DEVICE_CHECK(h < (size_t)(mv.mask + 1) * (mv.kmode ? kBucket32 : kBucket),
                  "k_hash_insert: slot out of the table");
  recs[mv.kmode ? h : (size_t)r] = v;
}

__global__ void k_fill(long long* __restrict__ p, long long v, unsigned n) {
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[i] = v;
}

}  // namespace vg

using namespace vg;

static int grid1(long long n, int threads) {
  long long g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 64) g = 148 * 64;
  return (int)g;
}

int launch_pack_keys(vg_ctx* ctx, const double* xyz_dev, long long n, double res,
                     long long* keys_dev) {
  if (n == 0) return 0;
  k_pack_keys<<<grid1(n, 256), 256, 0, ctx->stream>>>(xyz_dev, n, res, keys_dev, nullptr);
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  return 0;
}

int launch_cloud_pack(vg_ctx* ctx, vg_cloud* cl) {
  cl->plane = false;
  if (cl->n == 0) return 0;
  k_cloud_pack<<<grid1(cl->n, 256), 256, 0, ctx->stream>>>(cl->xyz64, cl->cov64, cl->n, cl->a,
                                                           cl->c0, cl->c1, cl->c2);
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  if (!cl->cov64) return 0;
  if (!cl->p0) {
    VG_CUDA(cudaMallocAsync((void**)&cl->p0, sizeof(double2) * cl->n, ctx->stream));
    VG_CUDA(cudaMallocAsync((void**)&cl->p1, sizeof(double2) * cl->n, ctx->stream));
    VG_CUDA(cudaMallocAsync((void**)&cl->p2, sizeof(double2) * cl->n, ctx->stream));
  }
  unsigned* dfail = nullptr;
  unsigned hfail = 1;
  VG_CUDA(cudaMallocAsync((void**)&dfail, sizeof(unsigned), ctx->stream));
  VG_CUDA(cudaMemsetAsync(dfail, 0, sizeof(unsigned), ctx->stream));
  k_plane_fit<<<grid1(cl->n, 256), 256, 0, ctx->stream>>>(cl->cov64, cl->n, cl->p0, cl->p1,
                                                          cl->p2, dfail);
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  VG_CUDA(cudaMemcpyAsync(&hfail, dfail, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  VG_CUDA(cudaFreeAsync(dfail, ctx->stream));
  cl->plane = hfail == 0;
  if (getenv("VGICP_DEBUG_PLANE"))
    fprintf(stderr, "plane fit: %lld points, %u not in plane form\n", cl->n, hfail);
  return 0;
}

// Record tensor map of a voxel map for K4b's TMA gathers: a 2D fp64 tensor of `rows` records x
// 16 doubles (128 B rows), box 10 x 1 (the 80 B of mean, covariance and row that K4b reads),
// no swizzle.  Encoded on the host (driver entry point resolved through the runtime) and kept
// in device memory; null when the driver refuses (K4b then gathers with cp.async).
static void make_record_tmap(vg_map* map, unsigned long long rows) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
      return (EncodeFn) nullptr;
    return (EncodeFn)p;
  }();
  if (!encode || !map->recs || rows == 0 || rows >= (1ull << 31)) return;
  CUtensorMap tm;
  const cuuint64_t dims[2] = {16, rows};
  const cuuint64_t strides[1] = {sizeof(VoxelRec)};
  const cuuint32_t box[2] = {10, 1};
  const cuuint32_t estr[2] = {1, 1};
  if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, map->recs, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return;
  void* d = nullptr;
  if (cudaMalloc(&d, sizeof(tm)) != cudaSuccess) return;
  if (cudaMemcpy(d, &tm, sizeof(tm), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    return;
  }
  map->tmap = d;
}

// bounds (k_key_bounds layout) of the map's keys when the build computed them on the device:
// the local frame and the empty marker then come without copying the keys to the host
int launch_map_finish(vg_ctx* ctx, vg_map* map, const long long* bounds) {
  long long empty = (long long)0x8000000000000000ull;
  map->kmode = 0;
  if (map->m && bounds && bounds[6] != LLONG_MIN) {
    const long long lo[3] = {bounds[0] - kKeyOffset, bounds[2] - kKeyOffset, bounds[4] - kKeyOffset};
    const long long hi[3] = {bounds[1] - kKeyOffset, bounds[3] - kKeyOffset, bounds[5] - kKeyOffset};
    const bool fits = hi[0] - lo[0] < 2048 && hi[1] - lo[1] < 2048 && hi[2] - lo[2] < 1023 &&
                      lo[0] > INT_MIN && lo[1] > INT_MIN && lo[2] > INT_MIN &&
                      hi[0] < INT_MAX && hi[1] < INT_MAX && hi[2] < INT_MAX &&
                      map->m < (1LL << 31);
    if (fits) {
      map->kmode = 1;
      map->bx = (int)lo[0];
      map->by = (int)lo[1];
      map->bz = (int)lo[2];
      map->ex = (int)(hi[0] - lo[0] + 1);
      map->ey = (int)(hi[1] - lo[1] + 1);
      map->ez = (int)(hi[2] - lo[2] + 1);
    }
    // the smallest key is above INT64_MIN, so INT64_MIN itself is absent (kmode 0 marker)
  } else if (map->m) {
    // local key frame from the decoded keys (all keys scanned on the host)
    std::vector<long long> hk((size_t)map->m);
    VG_CUDA(cudaMemcpyAsync(hk.data(), map->keys, sizeof(long long) * map->m,
                            cudaMemcpyDeviceToHost, ctx->stream));
    VG_CUDA(cudaStreamSynchronize(ctx->stream));
    long long lo[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX}, hi[3] = {LLONG_MIN, LLONG_MIN, LLONG_MIN};
    for (long long k : hk) {
      const long long d[3] = {(k >> 42) - kKeyOffset, ((k >> 21) & ((1LL << 21) - 1)) - kKeyOffset,
                              (k & ((1LL << 21) - 1)) - kKeyOffset};
      for (int a = 0; a < 3; ++a) {
        lo[a] = std::min(lo[a], d[a]);
        hi[a] = std::max(hi[a], d[a]);
      }
    }
    const bool fits = hi[0] - lo[0] < 2048 && hi[1] - lo[1] < 2048 && hi[2] - lo[2] < 1023 &&
                      lo[0] > INT_MIN && lo[1] > INT_MIN && lo[2] > INT_MIN &&
                      hi[0] < INT_MAX && hi[1] < INT_MAX && hi[2] < INT_MAX &&
                      map->m < (1LL << 31);
    if (fits) {
      map->kmode = 1;
      map->bx = (int)lo[0];
      map->by = (int)lo[1];
      map->bz = (int)lo[2];
      map->ex = (int)(hi[0] - lo[0] + 1);
      map->ey = (int)(hi[1] - lo[1] + 1);
      map->ez = (int)(hi[2] - lo[2] + 1);
    }
    // kmode 0 empty marker: the smallest value absent from the (strictly increasing) keys
    for (size_t i = 0; i < hk.size() && hk[i] == empty; ++i) ++empty;
  }
  map->empty_key = empty;
  // capacity: pow2 >= 4m slots (load <= 0.25) in 8-slot (kmode 0) / 4-slot (kmode 1) buckets
  int l2 = VG_BLOCK_HASH ? 6 : 3;  // the block hash needs >= 16 buckets of 4
  while ((1LL << l2) < 4 * map->m) ++l2;
  map->capacity = 1u << l2;
  map->log2cap = l2;
  const int gfill = (int)std::min<unsigned>((map->capacity + 255) / 256, 148 * 16);
  if (map->kmode) {
    VG_CUDA(cudaMallocAsync((void**)&map->pkeys32, sizeof(unsigned) * (size_t)map->capacity, ctx->stream));
    VG_CUDA(cudaMemsetAsync(map->pkeys32, 0xff, sizeof(unsigned) * (size_t)map->capacity, ctx->stream));
  } else {
    VG_CUDA(cudaMallocAsync((void**)&map->pkeys, sizeof(long long) * (size_t)map->capacity, ctx->stream));
    VG_CUDA(cudaMallocAsync((void**)&map->prows, sizeof(int) * (size_t)map->capacity, ctx->stream));
    k_fill<<<gfill, 256, 0, ctx->stream>>>(map->pkeys, empty, map->capacity);
    ctx->launches++;
    VG_CUDA(cudaGetLastError());
  }
  if (map->m == 0) return 0;
  VG_CUDA(cudaMallocAsync((void**)&map->recs,
                          sizeof(VoxelRec) * (size_t)(map->kmode ? map->capacity : map->m),
                          ctx->stream));
  k_hash_insert<<<(int)((map->m + 127) / 128), 128, 0, ctx->stream>>>(
      map->keys, map->means, map->covs, (int)map->m, map->view(), map->pkeys, map->prows,
      map->pkeys32, map->recs);
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  make_record_tmap(map, map->kmode ? map->capacity : (unsigned long long)map->m);
  return 0;
}

int launch_voxel_downsample(vg_ctx* ctx, const double* xyz, const double* stamps, long long n,
                            double res, double tol, double* xyz_out, double* stamps_out,
                            long long* m_out) {
  *m_out = 0;
  if (n == 0) return 0;
  cudaStream_t st = ctx->stream;
  long long *keys = nullptr, *keys_sorted = nullptr, *ukeys = nullptr;
  int *idx = nullptr, *perm = nullptr, *counts = nullptr, *offsets = nullptr, *num_runs = nullptr;
  int *ncell = nullptr, *out_off = nullptr;
  unsigned char* cell = nullptr;
  double *dx = nullptr, *dt = nullptr, *scratch = nullptr, *ox = nullptr, *ot = nullptr;
  void* tmp = nullptr;
  size_t t1 = 0, t2 = 0, t3 = 0, t4 = 0;
  DeviceTemps temps(st);
  VG_CUDA(temps.alloc(&dx, 3 * (size_t)n));
  VG_CUDA(temps.alloc(&dt, (size_t)n));
  VG_CUDA(temps.alloc(&keys, (size_t)n));
  VG_CUDA(temps.alloc(&keys_sorted, (size_t)n));
  VG_CUDA(temps.alloc(&ukeys, (size_t)n));
  VG_CUDA(temps.alloc(&idx, (size_t)n));
  VG_CUDA(temps.alloc(&perm, (size_t)n));
  VG_CUDA(temps.alloc(&counts, (size_t)n));
  VG_CUDA(temps.alloc(&offsets, (size_t)n));
  VG_CUDA(temps.alloc(&ncell, (size_t)n));
  VG_CUDA(temps.alloc(&out_off, (size_t)n));
  VG_CUDA(temps.alloc(&cell, (size_t)n));
  VG_CUDA(temps.alloc(&scratch, (size_t)n));
  VG_CUDA(temps.alloc(&ox, 3 * (size_t)n));
  VG_CUDA(temps.alloc(&ot, (size_t)n));
  VG_CUDA(temps.alloc(&num_runs, 1));
  VG_CUDA(cudaMemcpyAsync(dx, xyz, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
  VG_CUDA(cudaMemcpyAsync(dt, stamps, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  k_pack_keys<<<grid1(n, 256), 256, 0, st>>>(dx, n, res, keys, idx);
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  cub::DeviceRadixSort::SortPairs(nullptr, t1, keys, keys_sorted, idx, perm, (int)n, 0, 64, st);
  cub::DeviceRunLengthEncode::Encode(nullptr, t2, keys_sorted, ukeys, counts, num_runs, (int)n, st);
  cub::DeviceScan::ExclusiveSum(nullptr, t3, counts, offsets, (int)n, st);
  cub::DeviceScan::ExclusiveSum(nullptr, t4, ncell, out_off, (int)n, st);
  VG_CUDA(temps.alloc((unsigned char**)&tmp, std::max(std::max(t1, t2), std::max(t3, t4))));
  VG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t1, keys, keys_sorted, idx, perm, (int)n, 0, 64, st));
  VG_CUDA(cub::DeviceRunLengthEncode::Encode(tmp, t2, keys_sorted, ukeys, counts, num_runs, (int)n, st));
  int m = 0;
  VG_CUDA(cudaMemcpyAsync(&m, num_runs, sizeof(int), cudaMemcpyDeviceToHost, st));
  VG_CUDA(cudaStreamSynchronize(st));
  VG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, t3, counts, offsets, m, st));
  k_ds_assign<<<(m + 127) / 128, 128, 0, st>>>(offsets, counts, perm, dt, m, tol, cell, ncell);
  VG_CUDA(cudaGetLastError());
  VG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, t4, ncell, out_off, m, st));
  k_ds_emit<<<(m + 127) / 128, 128, 0, st>>>(offsets, counts, perm, dx, dt, cell, ncell, out_off,
                                             m, scratch, ox, ot);
  VG_CUDA(cudaGetLastError());
  ctx->launches += 9;  // pack, sort (>=2), rle, 2 scans, assign, emit (cub counted conservatively)
  int total = 0, last = 0;
  VG_CUDA(cudaMemcpyAsync(&total, out_off + m - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  VG_CUDA(cudaMemcpyAsync(&last, ncell + m - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  VG_CUDA(cudaStreamSynchronize(st));
  total += last;
  VG_CUDA(cudaMemcpyAsync(xyz_out, ox, sizeof(double) * 3 * total, cudaMemcpyDeviceToHost, st));
  VG_CUDA(cudaMemcpyAsync(stamps_out, ot, sizeof(double) * total, cudaMemcpyDeviceToHost, st));
  VG_CUDA(cudaStreamSynchronize(st));
  *m_out = total;
  return 0;
}

int launch_map_build(vg_ctx* ctx, const vg_cloud* cl, double res, vg_map* map) {
  const long long n = cl->n;
  map->res = res;
  map->m = 0;
  if (n == 0) return launch_map_finish(ctx, map);
  cudaStream_t st = ctx->stream;
  long long *keys = nullptr, *keys_sorted = nullptr, *ukeys = nullptr;
  int *idx = nullptr, *perm = nullptr, *counts = nullptr, *offsets = nullptr, *num_runs = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0, t1 = 0, t2 = 0, t3 = 0;
  DeviceTemps temps(st);  // released on every exit path
  VG_CUDA(temps.alloc(&keys, (size_t)n));
  VG_CUDA(temps.alloc(&keys_sorted, (size_t)n));
  VG_CUDA(temps.alloc(&ukeys, (size_t)n));
  VG_CUDA(temps.alloc(&idx, (size_t)n));
  VG_CUDA(temps.alloc(&perm, (size_t)n));
  VG_CUDA(temps.alloc(&counts, (size_t)n));
  VG_CUDA(temps.alloc(&offsets, (size_t)n));
  VG_CUDA(temps.alloc(&num_runs, 1));
  long long* bnd = nullptr;
  VG_CUDA(temps.alloc(&bnd, 8));
  k_pack_keys<<<grid1(n, 256), 256, 0, st>>>(cl->xyz64, n, res, keys, idx);
  k_bounds_init<<<1, 32, 0, st>>>(bnd);
  k_key_bounds<<<(unsigned)std::min<long long>((n + 255) / 256, 2 * 148), 256, 0, st>>>(keys, n, bnd);
  ctx->launches += 3;
  VG_CUDA(cudaGetLastError());
  long long hb[8];
  VG_CUDA(cudaMemcpyAsync(hb, bnd, sizeof(hb), cudaMemcpyDeviceToHost, st));
  VG_CUDA(cudaStreamSynchronize(st));
  // the (hi, mid, lo) fields' spans: when they fit 32 bits together, sort order-preserving 32-bit
  // local keys over just those bits (3-4 radix passes of 4-byte keys instead of 8 passes of
  // 8-byte keys; same stable permutation, so the same cells in the same member order)
  auto bits = [](long long span) {
    int b = 0;
    while (b < 40 && (1LL << b) < span + 1) ++b;
    return b;
  };
  const int bh = bits(hb[1] - hb[0]), bm = bits(hb[3] - hb[2]), bl = bits(hb[5] - hb[4]);
  const bool local32 = bh + bm + bl <= 32 && getenv("VGICP_MAP_SORT64") == nullptr;
  int m = 0;
  if (local32) {
    unsigned *lk = nullptr, *lk_sorted = nullptr, *ulk = nullptr;
    VG_CUDA(temps.alloc(&lk, (size_t)n));
    VG_CUDA(temps.alloc(&lk_sorted, (size_t)n));
    VG_CUDA(temps.alloc(&ulk, (size_t)n));
    const int sm = bl, sh = bl + bm, nbits = std::max(1, bh + bm + bl);
    k_local_keys<<<grid1(n, 256), 256, 0, st>>>(keys, n, bnd, sh, sm, lk);
    ctx->launches++;
    VG_CUDA(cudaGetLastError());
    cub::DeviceRadixSort::SortPairs(nullptr, t1, lk, lk_sorted, idx, perm, (int)n, 0, nbits, st);
    cub::DeviceRunLengthEncode::Encode(nullptr, t2, lk_sorted, ulk, counts, num_runs, (int)n, st);
    cub::DeviceScan::ExclusiveSum(nullptr, t3, counts, offsets, (int)n, st);
    tmp_bytes = std::max(std::max(t1, t2), t3);
    VG_CUDA(temps.alloc((unsigned char**)&tmp, tmp_bytes));
    VG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t1, lk, lk_sorted, idx, perm, (int)n, 0, nbits, st));
    VG_CUDA(cub::DeviceRunLengthEncode::Encode(tmp, t2, lk_sorted, ulk, counts, num_runs, (int)n, st));
    k_unlocal_keys<<<grid1(n, 256), 256, 0, st>>>(ulk, num_runs, bnd, sh, sm, ukeys);
    ctx->launches++;
    VG_CUDA(cudaGetLastError());
  } else {
    cub::DeviceRadixSort::SortPairs(nullptr, t1, keys, keys_sorted, idx, perm, (int)n, 0, 64, st);
    cub::DeviceRunLengthEncode::Encode(nullptr, t2, keys_sorted, ukeys, counts, num_runs, (int)n, st);
    cub::DeviceScan::ExclusiveSum(nullptr, t3, counts, offsets, (int)n, st);
    tmp_bytes = std::max(std::max(t1, t2), t3);
    VG_CUDA(temps.alloc((unsigned char**)&tmp, tmp_bytes));
    VG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t1, keys, keys_sorted, idx, perm, (int)n, 0, 64, st));
    VG_CUDA(cub::DeviceRunLengthEncode::Encode(tmp, t2, keys_sorted, ukeys, counts, num_runs, (int)n, st));
  }
  VG_CUDA(cudaMemcpyAsync(&m, num_runs, sizeof(int), cudaMemcpyDeviceToHost, st));
  VG_CUDA(cudaStreamSynchronize(st));
  VG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, t3, counts, offsets, m, st));
  ctx->launches += 6;  // cub: sort (>=2 passes) + rle + scan, counted conservatively
  map->m = m;
  VG_CUDA(cudaMallocAsync((void**)&map->keys, sizeof(long long) * m, st));
  VG_CUDA(cudaMallocAsync((void**)&map->means, sizeof(double) * 3 * m, st));
  VG_CUDA(cudaMallocAsync((void**)&map->covs, sizeof(double) * 9 * m, st));
  VG_CUDA(cudaMallocAsync((void**)&map->counts, sizeof(long long) * m, st));
  VG_CUDA(cudaMemcpyAsync(map->keys, ukeys, sizeof(long long) * m, cudaMemcpyDeviceToDevice, st));
  k_cell_stats<<<(m + 127) / 128, 128, 0, st>>>(offsets, counts, perm, cl->xyz64, cl->cov64, m,
                                                map->means, map->covs, map->counts);
  k_cell_stats_big<<<(m + kBigWarps - 1) / kBigWarps, kBigWarps * 32, 0, st>>>(
      offsets, counts, perm, cl->xyz64, cl->cov64, m, map->means, map->covs, map->counts);
  ctx->launches += 2;
  VG_CUDA(cudaGetLastError());
  return launch_map_finish(ctx, map, hb);
}
