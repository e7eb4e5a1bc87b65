// solve.cu — the LM's damped linear solve on the device.
//
// Reference: FactorGraph.optimize_lm, factor_graph.py:562-576 — per damping attempt the host
// forms h + diag(lam * diag(h)) and factors it: scipy cho_factor (dense, dim <= 600) or
// splu of its CSC form (above) — and marginal_covariance (:707-722).  At global-mapping size
// (1,000 submaps, dim 6,000) that is a 288 MB dense matrix built and factored on the host
// every attempt.
//
// Here H stays on the device:
//   * k_scatter_ne scatters a batch's block-sparse normal equations (K6 layout: 21-value upper
//     diagonal blocks, 6-value gradients, 36-value pair blocks) into dense H / g at the caller's
//     tangent offsets; every element of a layout lands on a distinct H entry, so the scatter
//     is a plain add, deterministic and race-free.  Non-matching factors' blocks come from the
//     host as a small block list (k_scatter_blocks, same rule).
//   * k_damp writes the damped diagonal of A = H + lam diag(H) + jitter I with the reference's
//     rounding sequence (lam * h_ii first, then the add; no FMA) after a copy of H.
//   * the factorization is cuSOLVER's dense Cholesky (potrf, 64-bit API) — a library
//     factorization, like cuBLAS for a plain GEMM — with a partial-pivot LU (getrf) fallback
//     for the splu branch, whose only failure is an exactly singular matrix.
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <string>
#include <vector>

#include "internal.h"
#include "vgicp.h"

struct vg_solver {
  vg_ctx* ctx = nullptr;
  long long dim = 0;
  double* H = nullptr;      // dim x dim (symmetric: row- and column-major agree)
  double* A = nullptr;      // damped copy, overwritten by the factorization
  double* g = nullptr;      // dim
  double* x = nullptr;      // solve workspace, dim x rhs_cap
  long long rhs_cap = 0;
  double* ne = nullptr;     // staging for a batch's K6 output
  long long ne_cap = 0;
  long long* offs = nullptr;  // variable tangent offsets (device)
  long long offs_cap = 0;
  int* pairs = nullptr;       // pair list (device) of the batch last scattered
  long long pairs_cap = 0;
  const vg_batch* pairs_of = nullptr;  // the pair list on the device is this batch's ...
  long long pairs_gen = -1;            // ... as of this assembly setup
  long long* blk = nullptr;   // host block descriptors (device copy)
  long long blk_cap = 0;
  double* blkv = nullptr;
  long long blkv_cap = 0;
  double* poses = nullptr;
  long long poses_cap = 0;
  int64_t* ipiv = nullptr;
  int* info = nullptr;
  void* work = nullptr;
  size_t work_bytes = 0;
  std::vector<char> hwork;
  cusolverDnHandle_t handle = nullptr;
  cusolverDnParams_t params = nullptr;
  int factored = 0;  // 0 none, 1 Cholesky (lower), 2 LU
  double cost = 0.0;
};

namespace vg {

__global__ void k_scatter_ne(const double* __restrict__ ne, int V, int P,
                             const long long* __restrict__ offs, const int* __restrict__ pairs,
                             long long dim, double* __restrict__ H, double* __restrict__ g) {
  const long long nd = 36LL * V, ng = 6LL * V, np_ = 36LL * P;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nd + ng + np_;
       e += (long long)gridDim.x * blockDim.x) {
    if (e < nd) {  // diagonal block v, element (r, c), from its upper-triangle packing
      const int v = (int)(e / 36), r = (int)(e % 36) / 6, c = (int)(e % 6);
      const int lo = min(r, c), hi = max(r, c);
      const double val = ne[2 + 21LL * v + lo * (11 - lo) / 2 + hi];
      const long long o = offs[v];
      H[(o + r) * dim + o + c] += val;
    } else if (e < nd + ng) {
      const long long k = e - nd;
      const int v = (int)(k / 6);
      g[offs[v] + k % 6] += ne[2 + 21LL * V + k];
    } else {  // pair block (a, b) element (r, c) and its transpose (:533-535)
      const long long k = e - nd - ng;
      const int p = (int)(k / 36), r = (int)(k % 36) / 6, c = (int)(k % 6);
      const double val = ne[2 + 27LL * V + k];
      const long long oa = offs[pairs[2 * p]], ob = offs[pairs[2 * p + 1]];
      H[(oa + r) * dim + ob + c] += val;
      H[(ob + c) * dim + oa + r] += val;
    }
  }
}

// one CTA per host block: block k (row0, col0, rows, cols) at values[voff[k] ..]
__global__ void k_scatter_blocks(const long long* __restrict__ desc,
                                 const double* __restrict__ values, long long dim,
                                 double* __restrict__ H) {
  const long long* d = desc + 5 * blockIdx.x;  // row0, col0, rows, cols, value offset
  const long long r0 = d[0], c0 = d[1], rows = d[2], cols = d[3], vo = d[4];
  for (long long e = threadIdx.x; e < rows * cols; e += blockDim.x)
    H[(r0 + e / cols) * dim + c0 + e % cols] += values[vo + e];
}

__global__ void k_add_vec(const double* __restrict__ src, long long n, double* __restrict__ dst) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

// A_ii = (H_ii + lam * H_ii) + jitter, rounded as numpy's h + np.diag(lam * diag) (+ jitter I)
__global__ void k_damp(const double* __restrict__ H, long long dim, double lam, double jitter,
                       double* __restrict__ A) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < dim;
       i += (long long)gridDim.x * blockDim.x) {
    const double h = H[i * dim + i];
    double a = h;
    if (lam != 0.0) a = __dadd_rn(a, __dmul_rn(lam, h));
    if (jitter != 0.0) a = __dadd_rn(a, jitter);
    A[i * dim + i] = a;
  }
}

__global__ void k_negate(const double* __restrict__ src, long long n, double* __restrict__ dst) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = -src[i];
}

}  // namespace vg

using namespace vg;

static int sfail(int code, const std::string& msg) {
  vg_set_error(msg);
  return code;
}

static int solver_status(cusolverStatus_t st, const char* what) {
  if (st == CUSOLVER_STATUS_SUCCESS) return VG_OK;
  return sfail(st == CUSOLVER_STATUS_ALLOC_FAILED ? VG_ERR_NOMEM : VG_ERR_CUDA,
               std::string(what) + ": cuSOLVER status " + std::to_string((int)st));
}
#define VG_SOLVER(call) VG_CHECK(solver_status((call), #call))

template <class T>
static int grow(vg_ctx* ctx, T** p, long long* cap, long long need) {
  if (need <= *cap) return VG_OK;
  if (*p) cudaFreeAsync(*p, ctx->stream);
  *p = nullptr;
  *cap = 0;
  VG_CUDA(cudaMallocAsync((void**)p, sizeof(T) * (size_t)need, ctx->stream));
  *cap = need;
  return VG_OK;
}

static int solver_grow_rhs(vg_solver* s, long long nrhs) {
  return grow(s->ctx, &s->x, &s->rhs_cap, nrhs * s->dim);
}

static unsigned grid_for(long long n, int threads = 256) {
  return (unsigned)std::max<long long>(1, std::min<long long>((n + threads - 1) / threads, 148LL * 16));
}

extern "C" {

int vg_solver_create(vg_ctx* ctx, int64_t dim, vg_solver** out) {
  if (!ctx || !out) return sfail(VG_ERR_INVALID, "null argument");
  *out = nullptr;
  if (dim <= 0 || dim > 60000) return sfail(VG_ERR_INVALID, "dim must be in [1, 60000]");
  vg_solver* s = new vg_solver();
  s->ctx = ctx;
  s->dim = dim;
  const size_t n2 = (size_t)dim * (size_t)dim;
  int rc = VG_OK;
  auto bail = [&](int code) {
    vg_solver_destroy(s);
    return code;
  };
  if (cudaMallocAsync((void**)&s->H, sizeof(double) * n2, ctx->stream) != cudaSuccess ||
      cudaMallocAsync((void**)&s->A, sizeof(double) * n2, ctx->stream) != cudaSuccess ||
      cudaMallocAsync((void**)&s->g, sizeof(double) * dim, ctx->stream) != cudaSuccess ||
      cudaMallocAsync((void**)&s->ipiv, sizeof(int64_t) * dim, ctx->stream) != cudaSuccess ||
      cudaMallocAsync((void**)&s->info, sizeof(int), ctx->stream) != cudaSuccess)
    return bail(sfail(VG_ERR_NOMEM, "vg_solver_create: device allocation failed"));
  rc = solver_status(cusolverDnCreate(&s->handle), "cusolverDnCreate");
  if (!rc) rc = solver_status(cusolverDnSetStream(s->handle, ctx->stream), "cusolverDnSetStream");
  if (!rc)
    rc = solver_status(cusolverDnSetDeterministicMode(s->handle, CUSOLVER_DETERMINISTIC_RESULTS),
                       "cusolverDnSetDeterministicMode");
  if (!rc) rc = solver_status(cusolverDnCreateParams(&s->params), "cusolverDnCreateParams");
  if (rc) return bail(rc);
  // one workspace sized for both factorizations
  size_t dp = 0, hp = 0, dl = 0, hl = 0;
  rc = solver_status(cusolverDnXpotrf_bufferSize(s->handle, s->params, CUBLAS_FILL_MODE_LOWER, dim,
                                                 CUDA_R_64F, s->A, dim, CUDA_R_64F, &dp, &hp),
                     "cusolverDnXpotrf_bufferSize");
  if (!rc)
    rc = solver_status(cusolverDnXgetrf_bufferSize(s->handle, s->params, dim, dim, CUDA_R_64F,
                                                   s->A, dim, CUDA_R_64F, &dl, &hl),
                       "cusolverDnXgetrf_bufferSize");
  if (rc) return bail(rc);
  s->work_bytes = std::max<size_t>(std::max(dp, dl), 16);
  s->hwork.resize(std::max<size_t>(std::max(hp, hl), 16));
  if (cudaMallocAsync(&s->work, s->work_bytes, ctx->stream) != cudaSuccess)
    return bail(sfail(VG_ERR_NOMEM, "vg_solver_create: workspace allocation failed"));
  rc = vg_solver_reset(s);
  if (rc) return bail(rc);
  *out = s;
  return VG_OK;
}

int vg_solver_destroy(vg_solver* s) {
  if (!s) return VG_OK;
  cudaStream_t st = s->ctx->stream;
  for (void* p : {(void*)s->H, (void*)s->A, (void*)s->g, (void*)s->x, (void*)s->ne,
                  (void*)s->offs, (void*)s->pairs, (void*)s->blk, (void*)s->blkv,
                  (void*)s->poses, (void*)s->ipiv, (void*)s->info, s->work})
    if (p) cudaFreeAsync(p, st);
  if (s->params) cusolverDnDestroyParams(s->params);
  if (s->handle) cusolverDnDestroy(s->handle);
  cudaStreamSynchronize(st);
  delete s;
  return VG_OK;
}

int vg_solver_reset(vg_solver* s) {
  if (!s) return sfail(VG_ERR_INVALID, "solver is null");
  cudaStream_t st = s->ctx->stream;
  VG_CUDA(cudaMemsetAsync(s->H, 0, sizeof(double) * (size_t)s->dim * (size_t)s->dim, st));
  VG_CUDA(cudaMemsetAsync(s->g, 0, sizeof(double) * (size_t)s->dim, st));
  s->cost = 0.0;
  s->factored = 0;
  return VG_OK;
}

int vg_solver_add_batch(vg_solver* s, vg_batch* b, const double* poses_host, int64_t V_poses,
                        const int64_t* offsets, double* cost_out) {
  if (!s || !b || !poses_host || !offsets) return sfail(VG_ERR_INVALID, "null argument");
  if (b->ctx != s->ctx) return sfail(VG_ERR_INVALID, "batch and solver use different contexts");
  if (b->asm_vars < 0) return sfail(VG_ERR_INVALID, "assembly not set up (vg_batch_assemble_setup)");
  if (b->asm_pidx) return sfail(VG_ERR_INVALID, "mapped assembly layouts are for sharded ranks");
  vg_ctx* ctx = s->ctx;
  const long long V = b->asm_vars, P = b->asm_pairs_n;
  for (long long v = 0; v < V; ++v)
    if (offsets[v] < 0 || offsets[v] + 6 > s->dim)
      return sfail(VG_ERR_INVALID, "variable block outside the solver's dimension");
  // every diagonal block and pair block must land on distinct entries
  std::vector<long long> so(offsets, offsets + V);
  std::sort(so.begin(), so.end());
  for (long long v = 1; v < V; ++v)
    if (so[v] < so[v - 1] + 6) return sfail(VG_ERR_INVALID, "variable blocks overlap");
  const long long total = 2 + 27 * V + 36 * P;
  VG_CHECK(grow(ctx, &s->ne, &s->ne_cap, total));
  VG_CHECK(grow(ctx, &s->poses, &s->poses_cap, 8 * V_poses));
  VG_CHECK(grow(ctx, &s->offs, &s->offs_cap, V));
  VG_CUDA(cudaMemcpyAsync(s->poses, poses_host, sizeof(double) * 8 * V_poses,
                          cudaMemcpyHostToDevice, ctx->stream));
  VG_CUDA(cudaMemcpyAsync(s->offs, offsets, sizeof(long long) * V, cudaMemcpyHostToDevice,
                          ctx->stream));
  if (s->pairs_of != b || s->pairs_gen != b->asm_gen) {
    VG_CHECK(grow(ctx, &s->pairs, &s->pairs_cap, std::max<long long>(2 * P, 1)));
    if (P)
      VG_CUDA(cudaMemcpyAsync(s->pairs, b->asm_pairs.data(), sizeof(int) * 2 * P,
                              cudaMemcpyHostToDevice, ctx->stream));
    s->pairs_of = b;
    s->pairs_gen = b->asm_gen;
  }
  VG_CHECK(vg_batch_assemble_poses_device(b, s->poses, V_poses, s->ne));
  k_scatter_ne<<<grid_for(36 * V + 6 * V + 36 * P), 256, 0, ctx->stream>>>(
      s->ne, (int)V, (int)P, s->offs, s->pairs, s->dim, s->H, s->g);
  VG_CUDA(cudaGetLastError());
  ctx->launches += 1;
  double c2[2];
  VG_CUDA(cudaMemcpyAsync(c2, s->ne, sizeof(c2), cudaMemcpyDeviceToHost, ctx->stream));
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  s->cost += c2[0];
  s->factored = 0;
  if (cost_out) *cost_out = c2[0];
  return VG_OK;
}

int vg_solver_add_blocks(vg_solver* s, int64_t nblk, const int64_t* desc, const double* values,
                         const double* g_host) {
  if (!s || nblk < 0 || (nblk && (!desc || !values))) return sfail(VG_ERR_INVALID, "null argument");
  vg_ctx* ctx = s->ctx;
  if (nblk) {
    std::vector<long long> d5(5 * (size_t)nblk);
    long long off = 0;
    for (int64_t k = 0; k < nblk; ++k) {
      const long long r0 = desc[4 * k], c0 = desc[4 * k + 1], rows = desc[4 * k + 2],
                      cols = desc[4 * k + 3];
      if (r0 < 0 || c0 < 0 || rows <= 0 || cols <= 0 || r0 + rows > s->dim || c0 + cols > s->dim)
        return sfail(VG_ERR_INVALID, "block outside the solver's dimension");
      d5[5 * k] = r0;
      d5[5 * k + 1] = c0;
      d5[5 * k + 2] = rows;
      d5[5 * k + 3] = cols;
      d5[5 * k + 4] = off;
      off += rows * cols;
    }
    VG_CHECK(grow(ctx, &s->blk, &s->blk_cap, 5 * nblk));
    VG_CHECK(grow(ctx, &s->blkv, &s->blkv_cap, off));
    VG_CUDA(cudaMemcpyAsync(s->blk, d5.data(), sizeof(long long) * d5.size(),
                            cudaMemcpyHostToDevice, ctx->stream));
    VG_CUDA(cudaMemcpyAsync(s->blkv, values, sizeof(double) * off, cudaMemcpyHostToDevice,
                            ctx->stream));
    for (int64_t k0 = 0; k0 < nblk; k0 += 65535) {
      const unsigned nb = (unsigned)std::min<int64_t>(65535, nblk - k0);
      k_scatter_blocks<<<nb, 128, 0, ctx->stream>>>(s->blk + 5 * k0, s->blkv, s->dim, s->H);
      VG_CUDA(cudaGetLastError());
      ctx->launches += 1;
    }
  }
  if (g_host) {
    VG_CHECK(solver_grow_rhs(s, 1));
    VG_CUDA(cudaMemcpyAsync(s->x, g_host, sizeof(double) * s->dim, cudaMemcpyHostToDevice,
                            ctx->stream));
    k_add_vec<<<grid_for(s->dim), 256, 0, ctx->stream>>>(s->x, s->dim, s->g);
    VG_CUDA(cudaGetLastError());
    ctx->launches += 1;
  }
  // host buffers are borrowed only for the call
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  s->factored = 0;
  return VG_OK;
}

int vg_solver_factor(vg_solver* s, double lam, double jitter, int32_t method, int64_t* info) {
  if (!s || !info) return sfail(VG_ERR_INVALID, "null argument");
  if (method != VG_SOLVE_CHOLESKY && method != VG_SOLVE_CHOLESKY_LU)
    return sfail(VG_ERR_INVALID, "unknown solve method");
  vg_ctx* ctx = s->ctx;
  const long long n = s->dim;
  const size_t bytes = sizeof(double) * (size_t)n * (size_t)n;
  auto damped = [&]() -> int {
    VG_CUDA(cudaMemcpyAsync(s->A, s->H, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    k_damp<<<grid_for(n), 256, 0, ctx->stream>>>(s->H, n, lam, jitter, s->A);
    VG_CUDA(cudaGetLastError());
    ctx->launches += 1;
    return VG_OK;
  };
  s->factored = 0;
  // the context's stream may have been rerouted (vg_ctx_set_stream) since the handle was made
  VG_SOLVER(cusolverDnSetStream(s->handle, ctx->stream));
  VG_CHECK(damped());
  VG_SOLVER(cusolverDnXpotrf(s->handle, s->params, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, s->A,
                             n, CUDA_R_64F, s->work, s->work_bytes, s->hwork.data(),
                             s->hwork.size(), s->info));
  int h_info = 0;
  VG_CUDA(cudaMemcpyAsync(&h_info, s->info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h_info == 0) {
    s->factored = 1;
    *info = 0;
    return VG_OK;
  }
  if (method == VG_SOLVE_CHOLESKY) {
    *info = h_info;
    return VG_OK;
  }
  // splu semantics: an indefinite but nonsingular damped matrix still solves
  VG_CHECK(damped());
  VG_SOLVER(cusolverDnXgetrf(s->handle, s->params, n, n, CUDA_R_64F, s->A, n, s->ipiv,
                             CUDA_R_64F, s->work, s->work_bytes, s->hwork.data(),
                             s->hwork.size(), s->info));
  VG_CUDA(cudaMemcpyAsync(&h_info, s->info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h_info == 0) s->factored = 2;
  *info = h_info;
  return VG_OK;
}

int vg_solver_solve(vg_solver* s, const double* rhs_host, int64_t nrhs, double* x_host) {
  if (!s || !x_host) return sfail(VG_ERR_INVALID, "null argument");
  if (!s->factored) return sfail(VG_ERR_INVALID, "no factorization (vg_solver_factor)");
  if (!rhs_host) nrhs = 1;
  if (nrhs <= 0) return sfail(VG_ERR_INVALID, "nrhs must be positive");
  vg_ctx* ctx = s->ctx;
  const long long n = s->dim;
  VG_CHECK(solver_grow_rhs(s, nrhs));
  VG_SOLVER(cusolverDnSetStream(s->handle, ctx->stream));
  if (rhs_host) {
    VG_CUDA(cudaMemcpyAsync(s->x, rhs_host, sizeof(double) * n * nrhs, cudaMemcpyHostToDevice,
                            ctx->stream));
  } else {
    k_negate<<<grid_for(n), 256, 0, ctx->stream>>>(s->g, n, s->x);
    VG_CUDA(cudaGetLastError());
    ctx->launches += 1;
  }
  if (s->factored == 1)
    VG_SOLVER(cusolverDnXpotrs(s->handle, s->params, CUBLAS_FILL_MODE_LOWER, n, nrhs, CUDA_R_64F,
                               s->A, n, CUDA_R_64F, s->x, n, s->info));
  else  // A is symmetric: its column-major LU solves A x = b directly
    VG_SOLVER(cusolverDnXgetrs(s->handle, s->params, CUBLAS_OP_N, n, nrhs, CUDA_R_64F, s->A, n,
                               s->ipiv, CUDA_R_64F, s->x, n, s->info));
  VG_CUDA(cudaMemcpyAsync(x_host, s->x, sizeof(double) * n * nrhs, cudaMemcpyDeviceToHost,
                          ctx->stream));
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  return VG_OK;
}

int vg_solver_export(vg_solver* s, double* h_host, double* g_host, double* cost_out) {
  if (!s) return sfail(VG_ERR_INVALID, "solver is null");
  vg_ctx* ctx = s->ctx;
  const long long n = s->dim;
  if (h_host)
    VG_CUDA(cudaMemcpyAsync(h_host, s->H, sizeof(double) * n * n, cudaMemcpyDeviceToHost,
                            ctx->stream));
  if (g_host)
    VG_CUDA(cudaMemcpyAsync(g_host, s->g, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (cost_out) *cost_out = s->cost;
  return VG_OK;
}

int vg_solver_diagonal(vg_solver* s, double* diag_host) {
  if (!s || !diag_host) return sfail(VG_ERR_INVALID, "null argument");
  const size_t pitch = sizeof(double) * (size_t)(s->dim + 1);
  VG_CUDA(cudaMemcpy2DAsync(diag_host, sizeof(double), s->H, pitch, sizeof(double),
                            (size_t)s->dim, cudaMemcpyDeviceToHost, s->ctx->stream));
  VG_CUDA(cudaStreamSynchronize(s->ctx->stream));
  return VG_OK;
}

}  // extern "C"
