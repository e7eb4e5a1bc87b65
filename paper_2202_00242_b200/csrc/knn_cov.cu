// knn_cov.cu — K6 exact k-nearest neighbours and plane-regularised point covariances.
//
// knn_search (preprocess.py:122-139): the reference takes cKDTree candidates, recomputes
// fp64 squared distances and orders them by (d2, index).  Here every query scans all points
// of its cloud through shared-memory tiles and keeps an exact top-k in registers under the
// same (d2, index) order, so the result equals the brute-force stable argsort the reference
// tests pin (test_preprocess.py:105-114).  d2 is formed as (dx*dx + dz*dz) + dy*dy with
// correctly rounded ops: the association numpy's einsum uses (checked bit for bit against
// the reference in tests/golden).
//
// Clouds of >= kKnnGridMin points use an exact uniform-grid search instead (k_knn_grid): the
// cloud is counting-sorted into cells of side h, and each query scans Chebyshev rings of cells
// around its own until the k-th best squared distance is below the distance to any unscanned
// cell; the same d2 expression and (d2, index) order give the brute-force result.
//
// estimate_covariances (preprocess.py:142-164): sample covariance / k, fp64 Jacobi
// eigen-decomposition, smallest-eigenvalue direction n, C = I - (1 - eps) n n^T (identical
// to V diag(eps, 1, 1) V^T), degenerate (lambda_max < 1e-12) -> eps * I.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace vg {

constexpr int kKnnTile = 256;

__device__ __forceinline__ bool knn_less(double da, int ia, double db, int ib) {
  return da < db || (da == db && ia < ib);
}

template <int KM>
__global__ void __launch_bounds__(kKnnTile)
    k_knn(const double* __restrict__ xyz, int n, int k, long long* __restrict__ out) {
  __shared__ double sx[kKnnTile], sy[kKnnTile], sz[kKnnTile];
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  double qx = 0.0, qy = 0.0, qz = 0.0;
  if (q < n) {
    qx = xyz[3 * (size_t)q];
    qy = xyz[3 * (size_t)q + 1];
    qz = xyz[3 * (size_t)q + 2];
  }
  // slots [0, KM-k) are -inf pads; [KM-k, KM) hold the running top-k in ascending order
  double d[KM];
  int id[KM];
#pragma unroll
  for (int j = 0; j < KM; ++j) {
    const bool pad = j < KM - k;
    d[j] = pad ? -DBL_MAX : DBL_MAX;
    id[j] = pad ? -1 : INT_MAX;
  }
  for (int base = 0; base < n; base += kKnnTile) {
    const int j = base + threadIdx.x;
    __syncthreads();
    if (j < n) {
      sx[threadIdx.x] = xyz[3 * (size_t)j];
      sy[threadIdx.x] = xyz[3 * (size_t)j + 1];
      sz[threadIdx.x] = xyz[3 * (size_t)j + 2];
    }
    __syncthreads();
    const int lim = min(kKnnTile, n - base);
    if (q >= n) continue;
    for (int u = 0; u < lim; ++u) {
      const double dx = __dsub_rn(sx[u], qx);
      const double dy = __dsub_rn(sy[u], qy);
      const double dz = __dsub_rn(sz[u], qz);
      const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dz, dz)), __dmul_rn(dy, dy));
      const int ci = base + u;
      if (knn_less(d2, ci, d[KM - 1], id[KM - 1])) {
        d[KM - 1] = d2;
        id[KM - 1] = ci;
#pragma unroll
        for (int s = KM - 1; s > 0; --s) {
          if (knn_less(d[s], id[s], d[s - 1], id[s - 1])) {
            const double td = d[s];
            d[s] = d[s - 1];
            d[s - 1] = td;
            const int ti = id[s];
            id[s] = id[s - 1];
            id[s - 1] = ti;
          }
        }
      }
    }
  }
  if (q < n) {
#pragma unroll
    for (int j = 0; j < KM; ++j)
      if (j >= KM - k) out[(size_t)q * k + (j - (KM - k))] = id[j];
  }
}

// ---- exact grid kNN ------------------------------------------------------------------------
struct KnnGrid {
  double ox, oy, oz;  // grid origin (cloud minimum)
  double h, inv_h;    // cell side
  int dx, dy, dz;     // cells per axis
};

__device__ __forceinline__ int knn_cell_axis(double v, double o, double inv_h, int d) {
  const int c = (int)floor((v - o) * inv_h);
  return min(max(c, 0), d - 1);
}

__global__ void k_bbox(const double* __restrict__ xyz, int n, double* __restrict__ out) {
  __shared__ double smin[3][256], smax[3][256];
  double lo[3] = {DBL_MAX, DBL_MAX, DBL_MAX}, hi[3] = {-DBL_MAX, -DBL_MAX, -DBL_MAX};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    for (int a = 0; a < 3; ++a) {
      const double v = xyz[3 * (size_t)i + a];
      lo[a] = fmin(lo[a], v);
      hi[a] = fmax(hi[a], v);
    }
  for (int a = 0; a < 3; ++a) {
    smin[a][threadIdx.x] = lo[a];
    smax[a][threadIdx.x] = hi[a];
  }
  __syncthreads();
  for (int s = blockDim.x / 2; s >= 1; s >>= 1) {
    if (threadIdx.x < s)
      for (int a = 0; a < 3; ++a) {
        smin[a][threadIdx.x] = fmin(smin[a][threadIdx.x], smin[a][threadIdx.x + s]);
        smax[a][threadIdx.x] = fmax(smax[a][threadIdx.x], smax[a][threadIdx.x + s]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int a = 0; a < 3; ++a) {
      out[6 * blockIdx.x + a] = smin[a][0];
      out[6 * blockIdx.x + 3 + a] = smax[a][0];
    }
}

__global__ void k_knn_cell_count(const double* __restrict__ xyz, int n, KnnGrid g,
                                 int* __restrict__ cell, int* __restrict__ counts) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int cx = knn_cell_axis(xyz[3 * (size_t)i], g.ox, g.inv_h, g.dx);
  const int cy = knn_cell_axis(xyz[3 * (size_t)i + 1], g.oy, g.inv_h, g.dy);
  const int cz = knn_cell_axis(xyz[3 * (size_t)i + 2], g.oz, g.inv_h, g.dz);
  const int c = (cx * g.dy + cy) * g.dz + cz;
  cell[i] = c;
  atomicAdd(counts + c, 1);
}

// scatter into cell order (order inside a cell is irrelevant: selection is by (d2, index))
__global__ void k_knn_scatter(const double* __restrict__ xyz, int n, const int* __restrict__ cell,
                              const int* __restrict__ start, int* __restrict__ fill,
                              double4* __restrict__ sorted) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = cell[i];
  const int pos = start[c] + atomicAdd(fill + c, 1);
  sorted[pos] = make_double4(xyz[3 * (size_t)i], xyz[3 * (size_t)i + 1], xyz[3 * (size_t)i + 2],
                             __hiloint2double(0, i));
}

template <int KM>
__global__ void __launch_bounds__(128)
    k_knn_grid(const double4* __restrict__ sorted, int n, int k, KnnGrid g,
               const int* __restrict__ start, long long* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  // queries in cell order: neighbouring threads scan the same cells
  const double4 qp = sorted[t];
  const double qx = qp.x, qy = qp.y, qz = qp.z;
  const int q = __double2loint(qp.w);
  double d[KM];
  int id[KM];
#pragma unroll
  for (int j = 0; j < KM; ++j) {
    const bool pad = j < KM - k;
    d[j] = pad ? -DBL_MAX : DBL_MAX;
    id[j] = pad ? -1 : INT_MAX;
  }
  auto consider = [&](int pos) {
    const double4 p = sorted[pos];
    const double ex = __dsub_rn(p.x, qx), ey = __dsub_rn(p.y, qy), ez = __dsub_rn(p.z, qz);
    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ez, ez)), __dmul_rn(ey, ey));
    const int ci = __double2loint(p.w);
    if (knn_less(d2, ci, d[KM - 1], id[KM - 1])) {
      d[KM - 1] = d2;
      id[KM - 1] = ci;
#pragma unroll
      for (int s = KM - 1; s > 0; --s) {
        if (knn_less(d[s], id[s], d[s - 1], id[s - 1])) {
          const double td = d[s];
          d[s] = d[s - 1];
          d[s - 1] = td;
          const int ti = id[s];
          id[s] = id[s - 1];
          id[s - 1] = ti;
        }
      }
    }
  };
  const int cx = knn_cell_axis(qx, g.ox, g.inv_h, g.dx);
  const int cy = knn_cell_axis(qy, g.oy, g.inv_h, g.dy);
  const int cz = knn_cell_axis(qz, g.oz, g.inv_h, g.dz);
  const int rmax = max(max(g.dx, g.dy), g.dz);
  // distance from the query to the nearest face of its own cell that has cells beyond it:
  // after ring R every unscanned point is at least R h + f0 away (R h alone assumes the query
  // sits on a face), so a query deep inside a dense cell stops after its own cell
  auto face = [&](double v, double o, int c, int d) {
    const double lo = o + c * g.h;
    const double a = c > 0 ? v - lo : DBL_MAX, b = c < d - 1 ? lo + g.h - v : DBL_MAX;
    return fmin(a, b);
  };
  const double f0 = fmax(fmin(fmin(face(qx, g.ox, cx, g.dx), face(qy, g.oy, cy, g.dy)),
                              face(qz, g.oz, cz, g.dz)),
                         0.0);
  for (int R = 0;; ++R) {
    // the shell of cells at Chebyshev distance R
    for (int ix = max(cx - R, 0); ix <= min(cx + R, g.dx - 1); ++ix) {
      const bool xe = ix == cx - R || ix == cx + R;
      for (int iy = max(cy - R, 0); iy <= min(cy + R, g.dy - 1); ++iy) {
        const bool ye = iy == cy - R || iy == cy + R;
        const int base = (ix * g.dy + iy) * g.dz;
        if (xe || ye) {
          const int z0 = max(cz - R, 0), z1 = min(cz + R, g.dz - 1);
          for (int pos = start[base + z0]; pos < start[base + z1 + 1]; ++pos) consider(pos);
        } else {
          if (cz - R >= 0)
            for (int pos = start[base + cz - R]; pos < start[base + cz - R + 1]; ++pos) consider(pos);
          if (R > 0 && cz + R < g.dz)
            for (int pos = start[base + cz + R]; pos < start[base + cz + R + 1]; ++pos) consider(pos);
        }
      }
    }
    // every unscanned point is farther than R h + f0 (up to the rounding of the cell
    // assignment, hence the margin); ties at the bound are scanned too
    const double bound = fmin(R * g.h + f0, 0.5 * DBL_MAX) - 2e-6 * g.h;
    if (R >= rmax || (bound > 0.0 && d[KM - 1] < bound * bound)) break;
  }
#pragma unroll
  for (int j = 0; j < KM; ++j)
    if (j >= KM - k) out[(size_t)q * k + (j - (KM - k))] = id[j];
}

// cyclic Jacobi on a symmetric 3x3 (fp64); a is destroyed, v receives eigenvectors (columns)
__device__ void jacobi3(double a[3][3], double v[3][3]) {
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) v[r][c] = (r == c) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 32; ++sweep) {
    const double off = fabs(a[0][1]) + fabs(a[0][2]) + fabs(a[1][2]);
    const double dia = fabs(a[0][0]) + fabs(a[1][1]) + fabs(a[2][2]);
    if (off <= 1e-300 || off <= 1e-18 * dia) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        const double apq = a[p][q];
        if (apq == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0);
        const double s = t * c;
        for (int k = 0; k < 3; ++k) {  // A <- A J
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {  // A <- J^T A
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          const double vkp = v[k][p], vkq = v[k][q];
          v[k][p] = c * vkp - s * vkq;
          v[k][q] = s * vkp + c * vkq;
        }
      }
  }
}

__global__ void k_cov(const double* __restrict__ xyz, const long long* __restrict__ nbrs, int n,
                      int k, double eps, double* __restrict__ covs,
                      unsigned char* __restrict__ degen) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long* nb = nbrs + (size_t)i * k;
  double mx = 0.0, my = 0.0, mz = 0.0;
  for (int j = 0; j < k; ++j) {
    const long long p = nb[j];
    mx += xyz[3 * p];
    my += xyz[3 * p + 1];
    mz += xyz[3 * p + 2];
  }
  mx /= k;
  my /= k;
  mz /= k;
  double a[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (int j = 0; j < k; ++j) {
    const long long p = nb[j];
    const double c[3] = {xyz[3 * p] - mx, xyz[3 * p + 1] - my, xyz[3 * p + 2] - mz};
    for (int r = 0; r < 3; ++r)
      for (int s = 0; s < 3; ++s) a[r][s] += c[r] * c[s];
  }
  for (int r = 0; r < 3; ++r)
    for (int s = 0; s < 3; ++s) a[r][s] /= k;
  double v[3][3];
  jacobi3(a, v);
  const double w0 = a[0][0], w1 = a[1][1], w2 = a[2][2];
  int lo = 0;
  if (w1 < w0 && w1 <= w2) lo = 1;
  else if (w2 < w0 && w2 < w1) lo = 2;
  const double wmax = fmax(w0, fmax(w1, w2));
  double* C = covs + 9 * (size_t)i;
  if (wmax < 1e-12) {  // preprocess.py:159,162-163
    for (int r = 0; r < 3; ++r)
      for (int s = 0; s < 3; ++s) C[3 * r + s] = (r == s) ? eps : 0.0;
    if (degen) degen[i] = 1;
    return;
  }
  const double nv[3] = {v[0][lo], v[1][lo], v[2][lo]};
  for (int r = 0; r < 3; ++r)
    for (int s = 0; s < 3; ++s) C[3 * r + s] = (r == s ? 1.0 : 0.0) - (1.0 - eps) * nv[r] * nv[s];
  if (degen) degen[i] = 0;
}

}  // namespace vg

using namespace vg;

static constexpr int kKnnGridMin = 4096;

// exact grid kNN: bbox -> cell side (about one cell per point, at most 4 n cells) -> counting
// sort into cells -> ring search per query
static int launch_knn_grid(vg_ctx* ctx, const vg_cloud* cl, int k, long long* nbrs_dev) {
  const int n = (int)cl->n;
  cudaStream_t st = ctx->stream;
  const int bb_blocks = 64;
  double* dbb = nullptr;
  VG_CUDA(cudaMallocAsync((void**)&dbb, sizeof(double) * 6 * bb_blocks, st));
  k_bbox<<<bb_blocks, 256, 0, st>>>(cl->xyz64, n, dbb);
  std::vector<double> hb(6 * bb_blocks);
  const cudaError_t ebb =
      cudaMemcpyAsync(hb.data(), dbb, sizeof(double) * 6 * bb_blocks, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(dbb, st);
  VG_CUDA(ebb);
  VG_CUDA(cudaStreamSynchronize(st));
  double lo[3] = {DBL_MAX, DBL_MAX, DBL_MAX}, hi[3] = {-DBL_MAX, -DBL_MAX, -DBL_MAX};
  for (int b = 0; b < bb_blocks; ++b)
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], hb[6 * b + a]);
      hi[a] = std::max(hi[a], hb[6 * b + 3 + a]);
    }
  double ext[3], emax = 0.0;
  for (int a = 0; a < 3; ++a) {
    ext[a] = hi[a] - lo[a];
    emax = std::max(emax, ext[a]);
  }
  if (!(emax > 0.0) || !std::isfinite(emax)) return -1;  // degenerate cloud: brute force
  const double floor_e = emax * 1e-3;
  double h = std::cbrt(std::max(ext[0], floor_e) * std::max(ext[1], floor_e) *
                       std::max(ext[2], floor_e) / n);
  KnnGrid g;
  long long cells = 0;
  for (int it = 0; it < 64; ++it, h *= 1.25) {
    g.dx = (int)std::min(ext[0] / h, 1e6) + 1;
    g.dy = (int)std::min(ext[1] / h, 1e6) + 1;
    g.dz = (int)std::min(ext[2] / h, 1e6) + 1;
    cells = (long long)g.dx * g.dy * g.dz;
    if (cells <= 4LL * n) break;
  }
  if (cells > 4LL * n) return -1;
  g.ox = lo[0];
  g.oy = lo[1];
  g.oz = lo[2];
  g.h = h;
  g.inv_h = 1.0 / h;
  int *cell = nullptr, *counts = nullptr, *start = nullptr, *fill = nullptr;
  double4* sorted = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  DeviceTemps temps(st);
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, start, (int)cells + 1, st);
  VG_CUDA(temps.alloc(&cell, (size_t)n));
  VG_CUDA(temps.alloc(&counts, (size_t)cells + 1));
  VG_CUDA(temps.alloc(&start, (size_t)cells + 1));
  VG_CUDA(temps.alloc(&fill, (size_t)cells));
  VG_CUDA(temps.alloc(&sorted, (size_t)n));
  VG_CUDA(temps.alloc((unsigned char**)&tmp, std::max<size_t>(tmp_bytes, 16)));
  VG_CUDA(cudaMemsetAsync(counts, 0, sizeof(int) * (cells + 1), st));
  VG_CUDA(cudaMemsetAsync(fill, 0, sizeof(int) * cells, st));
  k_knn_cell_count<<<(n + 255) / 256, 256, 0, st>>>(cl->xyz64, n, g, cell, counts);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, start, (int)cells + 1, st);
  k_knn_scatter<<<(n + 255) / 256, 256, 0, st>>>(cl->xyz64, n, cell, start, fill, sorted);
  const int blocks = (n + 127) / 128;
  if (k <= 8)
    k_knn_grid<8><<<blocks, 128, 0, st>>>(sorted, n, k, g, start, nbrs_dev);
  else if (k == 10)  // the reference's default (config.py:22): no padding slots to sort through
    k_knn_grid<10><<<blocks, 128, 0, st>>>(sorted, n, k, g, start, nbrs_dev);
  else if (k <= 16)
    k_knn_grid<16><<<blocks, 128, 0, st>>>(sorted, n, k, g, start, nbrs_dev);
  else
    k_knn_grid<32><<<blocks, 128, 0, st>>>(sorted, n, k, g, start, nbrs_dev);
  ctx->launches += 5;
  VG_CUDA(cudaGetLastError());
  return 0;
}

int launch_knn(vg_ctx* ctx, const vg_cloud* cl, int k, long long* nbrs_dev) {
  const int n = (int)cl->n;
  if (n == 0) return 0;
  static const int grid_env = [] {
    const char* e = getenv("VGICP_KNN_GRID");  // 0: always brute force
    return e ? atoi(e) : 1;
  }();
  if (grid_env && n >= kKnnGridMin && k <= 32) {
    const int rc = launch_knn_grid(ctx, cl, k, nbrs_dev);
    if (rc != -1) return rc;  // -1: grid not applicable (degenerate extent), brute force below
  }
  const int blocks = (n + kKnnTile - 1) / kKnnTile;
  if (k <= 8)
    k_knn<8><<<blocks, kKnnTile, 0, ctx->stream>>>(cl->xyz64, n, k, nbrs_dev);
  else if (k == 10)  // the reference's default: an exact-size register top-k
    k_knn<10><<<blocks, kKnnTile, 0, ctx->stream>>>(cl->xyz64, n, k, nbrs_dev);
  else if (k <= 16)
    k_knn<16><<<blocks, kKnnTile, 0, ctx->stream>>>(cl->xyz64, n, k, nbrs_dev);
  else if (k <= 32)
    k_knn<32><<<blocks, kKnnTile, 0, ctx->stream>>>(cl->xyz64, n, k, nbrs_dev);
  else {
    vg_set_error("k > 32 is not supported by the device kNN");
    return VG_ERR_INVALID;
  }
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  return 0;
}

int launch_cov(vg_ctx* ctx, const vg_cloud* cl, const long long* nbrs_dev, int k, double eps,
               double* covs_dev, unsigned char* degen_dev) {
  const int n = (int)cl->n;
  if (n == 0) return 0;
  k_cov<<<(n + 127) / 128, 128, 0, ctx->stream>>>(cl->xyz64, nbrs_dev, n, k, eps, covs_dev,
                                                   degen_dev);
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  return 0;
}
