// capi.cu — the extern "C" boundary (include/vgicp.h): handle lifetime, host<->device
// staging, batch flattening, and status-code error reporting.  No exception crosses the ABI.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "internal.h"
#include "vgicp.h"

using namespace vg;

static thread_local std::string g_err;

void vg_set_error(const std::string& msg) { g_err = msg; }

int vg_cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? VG_ERR_NOMEM : VG_ERR_CUDA;
}

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}


template <class T>
static int dalloc(vg_ctx* ctx, T** p, size_t count) {
  *p = nullptr;
  if (count == 0) return VG_OK;
  VG_CUDA(cudaMallocAsync((void**)p, sizeof(T) * count, ctx->stream));
  return VG_OK;
}
template <class T>
static void dfree(vg_ctx* ctx, T*& p) {
  if (p) cudaFreeAsync(p, ctx->stream);
  p = nullptr;
}

int vg_scratch(vg_ctx* ctx, size_t bytes, void** out) {
  if (bytes > ctx->scratch_bytes) {
    if (ctx->scratch) cudaFreeAsync(ctx->scratch, ctx->stream);
    size_t nb = std::max<size_t>(bytes, 4096);
    VG_CUDA(cudaMallocAsync(&ctx->scratch, nb, ctx->stream));
    ctx->scratch_bytes = nb;
  }
  *out = ctx->scratch;
  return VG_OK;
}

static int h2d(vg_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (!bytes) return VG_OK;
  VG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return VG_OK;
}
static int d2h_sync(vg_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (bytes) VG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  return VG_OK;
}

extern "C" {

int vg_abi_version(void) { return VGICP_ABI_VERSION; }

const char* vg_last_error(void) { return g_err.c_str(); }

int vg_ctx_create(int device, vg_ctx** out) {
  if (!out) return fail(VG_ERR_INVALID, "out is null");
  *out = nullptr;
  int ndev = 0;
  VG_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(VG_ERR_INVALID, "no such CUDA device");
  VG_CUDA(cudaSetDevice(device));
  int major = 0;
  VG_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  if (major != 10) return fail(VG_ERR_CUDA, "libvgicp is built for sm_100a (B200) only");
  vg_ctx* c = new vg_ctx();
  c->device = device;
  cudaError_t e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return vg_cuda_fail(e, "cudaStreamCreateWithFlags");
  }
  c->stream = c->own_stream;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = c;
  return VG_OK;
}

int vg_ctx_destroy(vg_ctx* ctx) {
  if (!ctx) return VG_OK;
  cudaSetDevice(ctx->device);
  if (ctx->scratch) cudaFreeAsync(ctx->scratch, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->side_stream) {
    cudaStreamSynchronize(ctx->side_stream);
    cudaStreamDestroy(ctx->side_stream);
    for (auto& e : ctx->events) cudaEventDestroy(e);
  }
  if (ctx->comp3) {
    cudaStreamSynchronize(ctx->comp3);
    cudaStreamDestroy(ctx->comp3);
  }
  if (ctx->comp2) {
    cudaStreamSynchronize(ctx->comp2);
    cudaStreamDestroy(ctx->comp2);
  }


  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
  return VG_OK;
}

int vg_ctx_set_stream(vg_ctx* ctx, void* stream) {
  if (!ctx) return fail(VG_ERR_INVALID, "ctx is null");
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->stream = stream ? (cudaStream_t)stream : ctx->own_stream;
  return VG_OK;
}

int vg_ctx_synchronize(vg_ctx* ctx) {
  if (!ctx) return fail(VG_ERR_INVALID, "ctx is null");
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  return VG_OK;
}

int vg_ctx_launch_count(const vg_ctx* ctx, int64_t* count) {
  if (!ctx || !count) return fail(VG_ERR_INVALID, "null argument");
  *count = ctx->launches;
  return VG_OK;
}

// ---- keys -------------------------------------------------------------------------------
int vg_pack_voxel_keys(vg_ctx* ctx, const double* xyz, int64_t n, double res, int64_t* keys_out) {
  if (!ctx || (n && (!xyz || !keys_out))) return fail(VG_ERR_INVALID, "null argument");
  if (!(res > 0.0)) return fail(VG_ERR_INVALID, "resolution must be positive");
  if (n == 0) return VG_OK;
  double* dx = nullptr;
  long long* dk = nullptr;
  VG_CHECK(dalloc(ctx, &dx, 3 * n));
  VG_CHECK(dalloc(ctx, &dk, n));
  VG_CHECK(h2d(ctx, dx, xyz, sizeof(double) * 3 * n));
  VG_CHECK(launch_pack_keys(ctx, dx, n, res, dk));
  int rc = d2h_sync(ctx, keys_out, dk, sizeof(long long) * n);
  dfree(ctx, dx);
  dfree(ctx, dk);
  return rc;
}

int vg_voxel_downsample(vg_ctx* ctx, const double* xyz, const double* stamps, int64_t n,
                        double res, double split_tol, double* xyz_out, double* stamps_out,
                        int64_t* m_out) {
  if (!ctx || !m_out || n < 0 || (n && (!xyz || !stamps || !xyz_out || !stamps_out)))
    return fail(VG_ERR_INVALID, "null argument");
  if (!(res > 0.0)) return fail(VG_ERR_INVALID, "resolution must be positive");
  if (n >= (1LL << 31)) return fail(VG_ERR_INVALID, "scan too large");
  VG_CUDA(cudaSetDevice(ctx->device));
  long long m = 0;
  VG_CHECK(launch_voxel_downsample(ctx, xyz, stamps, n, res, split_tol, xyz_out, stamps_out, &m));
  *m_out = m;
  return VG_OK;
}

int vg_deskew_points(vg_ctx* ctx, const double* xyz, const double* stamps, int64_t n,
                     const double* node_t, const double* quats, const double* trans, int64_t K,
                     double* xyz_out) {
  if (!ctx || n < 0 || (n && (!xyz || !stamps || !xyz_out)) || !node_t || !quats || !trans)
    return fail(VG_ERR_INVALID, "null argument");
  if (K < 2 || K >= (1LL << 31)) return fail(VG_ERR_INVALID, "need at least two trajectory nodes");
  for (int64_t i = 1; i < K; ++i)
    if (!(node_t[i] >= node_t[i - 1])) return fail(VG_ERR_INVALID, "node stamps must ascend");
  VG_CUDA(cudaSetDevice(ctx->device));
  return launch_deskew(ctx, xyz, stamps, n, node_t, quats, trans, (int)K, xyz_out);
}

// ---- clouds -----------------------------------------------------------------------------
int vg_cloud_create(vg_ctx* ctx, const double* xyz, const double* cov, int64_t n,
                    vg_cloud** out) {
  if (!ctx || !out || n < 0 || (n && !xyz)) return fail(VG_ERR_INVALID, "invalid cloud arguments");
  VG_CUDA(cudaSetDevice(ctx->device));
  vg_cloud* c = new vg_cloud();
  c->ctx = ctx;
  c->n = n;
  c->has_cov = cov != nullptr;
  bool exact = true;
  for (int64_t i = 0; i < 3 * n && exact; ++i) exact = ((double)(float)xyz[i] == xyz[i]);
  c->exact32 = exact;
  int rc = VG_OK;
  if (n) {
    if ((rc = dalloc(ctx, &c->xyz64, 3 * n)) || (rc = dalloc(ctx, &c->a, n)) ||
        (cov && ((rc = dalloc(ctx, &c->cov64, 9 * n)) || (rc = dalloc(ctx, &c->c0, n)) ||
                 (rc = dalloc(ctx, &c->c1, n)) || (rc = dalloc(ctx, &c->c2, n)))) ||
        (rc = h2d(ctx, c->xyz64, xyz, sizeof(double) * 3 * n)) ||
        (cov && (rc = h2d(ctx, c->cov64, cov, sizeof(double) * 9 * n))) ||
        (rc = launch_cloud_pack(ctx, c))) {
      vg_cloud_destroy(c);
      return rc;
    }
  }
  *out = c;
  return VG_OK;
}

int vg_cloud_info(const vg_cloud* c, int64_t* n, int32_t* has_cov, int32_t* exact32) {
  if (!c) return fail(VG_ERR_INVALID, "cloud is null");
  if (n) *n = c->n;
  if (has_cov) *has_cov = c->has_cov;
  if (exact32) *exact32 = c->exact32;
  return VG_OK;
}

int vg_cloud_destroy(vg_cloud* c) {
  if (!c) return VG_OK;
  vg_ctx* ctx = c->ctx;
  dfree(ctx, c->a);
  dfree(ctx, c->c0);
  dfree(ctx, c->c1);
  dfree(ctx, c->c2);
  dfree(ctx, c->xyz64);
  dfree(ctx, c->cov64);
  dfree(ctx, c->p0);
  dfree(ctx, c->p1);
  dfree(ctx, c->p2);
  delete c;
  return VG_OK;
}

// ---- maps -------------------------------------------------------------------------------
int vg_map_build(vg_ctx* ctx, const vg_cloud* cloud, double res, vg_map** out) {
  if (!ctx || !cloud || !out) return fail(VG_ERR_INVALID, "null argument");
  if (!(res > 0.0)) return fail(VG_ERR_INVALID, "resolution must be positive");
  if (cloud->n > 0 && !cloud->has_cov)  // registration.py:80-81
    return fail(VG_ERR_INVALID, "frame needs covariances before voxelization");
  if (cloud->n >= (1LL << 31)) return fail(VG_ERR_INVALID, "cloud too large for one map");
  vg_map* m = new vg_map();
  m->ctx = ctx;
  int rc = launch_map_build(ctx, cloud, res, m);
  if (rc) {
    vg_map_destroy(m);
    return rc;
  }
  *out = m;
  return VG_OK;
}

int vg_map_from_arrays(vg_ctx* ctx, double res, const int64_t* keys, const double* means,
                       const double* covs, const int64_t* counts, int64_t m, vg_map** out) {
  if (!ctx || !out || m < 0 || (m && (!keys || !means || !covs)))
    return fail(VG_ERR_INVALID, "invalid map arrays");
  if (!(res > 0.0)) return fail(VG_ERR_INVALID, "resolution must be positive");
  for (int64_t i = 1; i < m; ++i)
    if (keys[i] <= keys[i - 1])
      return fail(VG_ERR_INVALID, "GaussianVoxelMap keys must be strictly increasing");
  vg_map* mp = new vg_map();
  mp->ctx = ctx;
  mp->m = m;
  mp->res = res;
  int rc = VG_OK;
  if (m) {
    std::vector<long long> cnt(m, 1);
    if (counts) std::copy(counts, counts + m, cnt.begin());
    if ((rc = dalloc(ctx, &mp->keys, m)) || (rc = dalloc(ctx, &mp->means, 3 * m)) ||
        (rc = dalloc(ctx, &mp->covs, 9 * m)) || (rc = dalloc(ctx, &mp->counts, m)) ||
        (rc = h2d(ctx, mp->keys, keys, sizeof(long long) * m)) ||
        (rc = h2d(ctx, mp->means, means, sizeof(double) * 3 * m)) ||
        (rc = h2d(ctx, mp->covs, covs, sizeof(double) * 9 * m)) ||
        (rc = h2d(ctx, mp->counts, cnt.data(), sizeof(long long) * m)) ||
        (rc = cudaStreamSynchronize(ctx->stream) ? VG_ERR_CUDA : VG_OK)) {
      vg_map_destroy(mp);
      return rc;
    }
  }
  if ((rc = launch_map_finish(ctx, mp))) {
    vg_map_destroy(mp);
    return rc;
  }
  *out = mp;
  return VG_OK;
}

int vg_map_info(const vg_map* m, int64_t* size, double* res, int64_t* cap) {
  if (!m) return fail(VG_ERR_INVALID, "map is null");
  if (size) *size = m->m;
  if (res) *res = m->res;
  if (cap) *cap = m->capacity;
  return VG_OK;
}

int vg_map_export(vg_ctx* ctx, const vg_map* m, int64_t* keys, double* means, double* covs,
                  int64_t* counts) {
  if (!ctx || !m) return fail(VG_ERR_INVALID, "null argument");
  const long long n = m->m;
  if (n == 0) return VG_OK;
  if (keys) VG_CUDA(cudaMemcpyAsync(keys, m->keys, sizeof(long long) * n, cudaMemcpyDeviceToHost, ctx->stream));
  if (means) VG_CUDA(cudaMemcpyAsync(means, m->means, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, ctx->stream));
  if (covs) VG_CUDA(cudaMemcpyAsync(covs, m->covs, sizeof(double) * 9 * n, cudaMemcpyDeviceToHost, ctx->stream));
  if (counts) VG_CUDA(cudaMemcpyAsync(counts, m->counts, sizeof(long long) * n, cudaMemcpyDeviceToHost, ctx->stream));
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  return VG_OK;
}

int vg_map_destroy(vg_map* m) {
  if (!m) return VG_OK;
  vg_ctx* ctx = m->ctx;
  dfree(ctx, m->pkeys);
  dfree(ctx, m->prows);
  dfree(ctx, m->pkeys32);
  dfree(ctx, m->recs);
  if (m->tmap) cudaFree(m->tmap);
  dfree(ctx, m->keys);
  dfree(ctx, m->means);
  dfree(ctx, m->covs);
  dfree(ctx, m->counts);
  delete m;
  return VG_OK;
}

// ---- lookup / terms ---------------------------------------------------------------------
static const double kIdentityT[12] = {1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0};

int vg_cloud_lookup(vg_ctx* ctx, const vg_cloud* cloud, const vg_map* map, const double T[12],
                    int64_t* rows_out, int64_t* hits_out) {
  if (!ctx || !cloud || !map || !T) return fail(VG_ERR_INVALID, "null argument");
  const long long n = cloud->n;
  void* scr = nullptr;
  VG_CHECK(vg_scratch(ctx, 128, &scr));
  double* dT = (double*)scr;
  unsigned long long* dh = (unsigned long long*)((char*)scr + 96);
  VG_CHECK(h2d(ctx, dT, T, 96));
  VG_CUDA(cudaMemsetAsync(dh, 0, 8, ctx->stream));
  long long* drows = nullptr;
  if (rows_out) VG_CHECK(dalloc(ctx, &drows, n));
  VG_CHECK(launch_lookup(ctx, cloud->view(), map->view(), dT, drows, dh));
  unsigned long long hits = 0;
  if (rows_out && n) VG_CUDA(cudaMemcpyAsync(rows_out, drows, sizeof(long long) * n, cudaMemcpyDeviceToHost, ctx->stream));
  VG_CHECK(d2h_sync(ctx, &hits, dh, 8));
  dfree(ctx, drows);
  if (hits_out) *hits_out = (int64_t)hits;
  return VG_OK;
}

int vg_map_lookup(vg_ctx* ctx, const vg_map* map, const double* xyz, int64_t n, int64_t* rows_out,
                  int64_t* hits_out) {
  if (!ctx || !map || (n && !xyz)) return fail(VG_ERR_INVALID, "null argument");
  if (n == 0) {
    if (hits_out) *hits_out = 0;
    return VG_OK;
  }
  vg_cloud* c = nullptr;
  VG_CHECK(vg_cloud_create(ctx, xyz, nullptr, n, &c));
  int rc = vg_cloud_lookup(ctx, c, map, kIdentityT, rows_out, hits_out);
  vg_cloud_destroy(c);
  return rc;
}

int vg_match_terms(vg_ctx* ctx, const vg_cloud* cloud, const vg_map* map, const double T[12],
                   int64_t* rows, double* moved, double* d, double* weight, double* wd,
                   double* cost, int64_t* inliers) {
  if (!ctx || !cloud || !map || !T || !rows || !moved || !d || !weight || !wd)
    return fail(VG_ERR_INVALID, "null argument");
  if (!cloud->has_cov) return fail(VG_ERR_INVALID, "source frame has no covariances");
  const long long n = cloud->n;
  if (n == 0) {
    if (cost) *cost = 0.0;
    if (inliers) *inliers = 0;
    return VG_OK;
  }
  const int nblocks = (int)std::min<long long>((n + 255) / 256, 148 * 8);
  double *dT = nullptr, *dmoved = nullptr, *dd = nullptr, *dw = nullptr, *dwd = nullptr,
         *pc = nullptr;
  long long *drows = nullptr, *pi = nullptr;
  VG_CHECK(dalloc(ctx, &dT, 12));
  VG_CHECK(dalloc(ctx, &drows, n));
  VG_CHECK(dalloc(ctx, &dmoved, 3 * n));
  VG_CHECK(dalloc(ctx, &dd, 3 * n));
  VG_CHECK(dalloc(ctx, &dw, 9 * n));
  VG_CHECK(dalloc(ctx, &dwd, 3 * n));
  VG_CHECK(dalloc(ctx, &pc, nblocks));
  VG_CHECK(dalloc(ctx, &pi, nblocks));
  VG_CHECK(h2d(ctx, dT, T, 96));
  VG_CHECK(launch_terms(ctx, cloud->view(), map->view(), dT, drows, dmoved, dd, dw, dwd, pc, pi,
                        nblocks));
  std::vector<double> hc(nblocks);
  std::vector<long long> hi(nblocks);
  VG_CUDA(cudaMemcpyAsync(rows, drows, 8 * n, cudaMemcpyDeviceToHost, ctx->stream));
  VG_CUDA(cudaMemcpyAsync(moved, dmoved, 24 * n, cudaMemcpyDeviceToHost, ctx->stream));
  VG_CUDA(cudaMemcpyAsync(d, dd, 24 * n, cudaMemcpyDeviceToHost, ctx->stream));
  VG_CUDA(cudaMemcpyAsync(weight, dw, 72 * n, cudaMemcpyDeviceToHost, ctx->stream));
  VG_CUDA(cudaMemcpyAsync(wd, dwd, 24 * n, cudaMemcpyDeviceToHost, ctx->stream));
  VG_CUDA(cudaMemcpyAsync(hc.data(), pc, 8 * nblocks, cudaMemcpyDeviceToHost, ctx->stream));
  VG_CHECK(d2h_sync(ctx, hi.data(), pi, 8 * nblocks));
  double cs = 0.0;
  long long is = 0;
  for (int b = 0; b < nblocks; ++b) cs += hc[b], is += hi[b];
  if (cost) *cost = cs;
  if (inliers) *inliers = is;
  dfree(ctx, dT);
  dfree(ctx, drows);
  dfree(ctx, dmoved);
  dfree(ctx, dd);
  dfree(ctx, dw);
  dfree(ctx, dwd);
  dfree(ctx, pc);
  dfree(ctx, pi);
  return VG_OK;
}

int vg_linearize_terms(vg_ctx* ctx, const double T[12], const double* points, const double* weight,
                       const double* wd, int64_t n, double cost, int64_t inliers, int32_t flags,
                       int32_t min_inliers, double* out) {
  if (!ctx || !T || !out || n < 0 || (n && (!points || !weight || !wd)))
    return fail(VG_ERR_INVALID, "null argument");
  if (inliers < min_inliers)  // registration.py:213-215
    return fail(VG_ERR_DEGENERATE, std::to_string(inliers) + " inliers (minimum " +
                                       std::to_string(min_inliers) + ")");
  VG_CUDA(cudaSetDevice(ctx->device));
  FactorDev f;
  memset(&f, 0, sizeof(f));
  for (int k = 0; k < 12; ++k) f.T[k] = T[k];
  f.flags = flags;
  f.min_inliers = min_inliers;
  DeviceTemps temps(ctx->stream);
  double *dp = nullptr, *dw = nullptr, *dwd = nullptr, *dout = nullptr;
  VG_CUDA(temps.alloc(&dp, 3 * (size_t)n));
  VG_CUDA(temps.alloc(&dw, 9 * (size_t)n));
  VG_CUDA(temps.alloc(&dwd, 3 * (size_t)n));
  VG_CUDA(temps.alloc(&dout, 92));
  VG_CHECK(h2d(ctx, dp, points, sizeof(double) * 3 * n));
  VG_CHECK(h2d(ctx, dw, weight, sizeof(double) * 9 * n));
  VG_CHECK(h2d(ctx, dwd, wd, sizeof(double) * 3 * n));
  VG_CHECK(launch_terms_linearize(ctx, dp, dw, dwd, n, f, cost, (double)inliers, dout));
  return d2h_sync(ctx, out, dout, sizeof(double) * 92);
}

// ---- batches ----------------------------------------------------------------------------
int vg_batch_create(vg_ctx* ctx, const vg_factor_spec* specs, int64_t F, vg_batch** out) {
  if (!ctx || !out || F < 0 || (F && !specs)) return fail(VG_ERR_INVALID, "invalid batch arguments");
  if (F >= (1LL << 31)) return fail(VG_ERR_INVALID, "too many factors");
  std::vector<const vg_cloud*> clouds;
  std::vector<const vg_map*> maps;
  std::vector<FactorDev> fac(F);
  // dedupe clouds and maps (sort by handle address)
  std::vector<std::pair<const void*, int64_t>> ck(F), mk(F);
  bool all_covs = true;  // without covariances a batch serves VG_MODE_INLIERS only
  for (int64_t f = 0; f < F; ++f) {
    if (!specs[f].source || !specs[f].target) return fail(VG_ERR_INVALID, "factor without cloud/map");
    if (!specs[f].source->has_cov && specs[f].source->n > 0) all_covs = false;
    ck[f] = {specs[f].source, f};
    mk[f] = {specs[f].target, f};
  }
  std::vector<int> cidx(F), midx(F);
  auto dedupe = [&](std::vector<std::pair<const void*, int64_t>>& v, std::vector<int>& idx,
                    auto& uniq) {
    std::sort(v.begin(), v.end());
    for (size_t i = 0; i < v.size(); ++i) {
      if (i == 0 || v[i].first != v[i - 1].first)
        uniq.push_back((typename std::remove_reference<decltype(uniq)>::type::value_type)v[i].first);
      idx[v[i].second] = (int)uniq.size() - 1;
    }
  };
  dedupe(ck, cidx, clouds);
  dedupe(mk, midx, maps);
  long long max_var = -1;
  for (int64_t f = 0; f < F; ++f) {
    FactorDev& d = fac[f];
    memset(&d, 0, sizeof(d));
    d.T[0] = d.T[4] = d.T[8] = 1.0;
    d.cloud = cidx[f];
    d.map = midx[f];
    d.flags = specs[f].flags;
    d.min_inliers = specs[f].min_inliers;
    d.var_source = specs[f].var_source;
    d.var_target = specs[f].var_target;
    max_var = std::max<long long>(max_var, std::max(d.var_source, d.var_target));
  }
  // work items: factors ordered by target map (L1/L2 reuse of the map's slots), chunks of
  // <= kMaxChunk points, one warp per item
  std::vector<int64_t> order(F);
  std::iota(order.begin(), order.end(), 0);
  static const int order_mode = [] {
    const char* e = getenv("VGICP_ITEM_ORDER");  // 0 target-major (default), 1 source-major, 2 input
    return e ? atoi(e) : 0;
  }();
  // Stages (pipelined host output, vg_batch_linearize*): contiguous factor ranges whose
  // records are copied to the host while the next stage computes; items are stage-major.
  static const int stages_env = [] {
    // default: 6 stages from 32,768 factors, 4 from 8,192 (config 5, compact fp32 records:
    // 6 -> e2e 0.565 ms, 8 -> 0.578, 4 -> 0.596, 12 -> 0.611, 16 -> 0.621)
    const char* e = getenv("VGICP_STAGES");
    return e ? atoi(e) : -1;
  }();
  int S = (int)std::max<int64_t>(
      1, std::min<int64_t>(stages_env >= 0 ? stages_env : (F >= 32768 ? 6 : F >= 8192 ? 4 : 1),
                           16));
  // stage s holds a share proportional to ratio^s: a smaller first stage starts the copy
  // engine sooner (default 1.2 from 8 stages: config 5 e2e 0.814 -> 0.791 ms with the two
  // compute streams of run_to_host; 1.35 and beyond expose the large late stages' copies)
  static const double ratio_env = [] {
    const char* e = getenv("VGICP_STAGE_RATIO");
    return e ? atof(e) : 0.0;
  }();
  const double ratio = ratio_env > 0.0 ? ratio_env : (S >= 8 ? 1.2 : 1.0);
  // VGICP_STAGE_PROFILE="w0,w1,...": explicit relative stage sizes (overrides the count and
  // the ratio), e.g. small first and last stages (early copy start, short copy tail)
  static const std::vector<double> profile_env = [] {
    std::vector<double> v;
    const char* e = getenv("VGICP_STAGE_PROFILE");
    while (e && *e) {
      char* end = nullptr;
      const double x = strtod(e, &end);
      if (end == e) break;
      if (x > 0.0) v.push_back(x);
      e = *end == ',' ? end + 1 : end;
    }
    return v;
  }();
  std::vector<double> weights;
  if (!profile_env.empty() && F >= 8192 && stages_env != 1) {
    weights = profile_env;
    if (weights.size() > 16) weights.resize(16);  // event slots of run_to_host
  } else {
    double w = 1.0;
    for (int s = 0; s < S; ++s, w *= ratio) weights.push_back(w);
  }
  S = (int)weights.size();
  std::vector<int> stage_factors(S + 1), stage_of(F);
  {
    double tot = 0.0;
    for (double w : weights) tot += w;
    double acc = 0.0;
    stage_factors[0] = 0;
    for (int s = 1; s <= S; ++s) {
      acc += weights[s - 1];
      // interior boundaries on 64-factor windows: K5's per-window cost partials (k_finalize)
      // must not straddle two stages' launches
      stage_factors[s] = s == S ? (int)F : (int)(std::llround((double)F * acc / tot) / 64 * 64);
    }
  }
  for (int s = 0; s < S; ++s)
    for (int f = stage_factors[s]; f < stage_factors[s + 1]; ++f) stage_of[f] = s;
  if (order_mode == 0)
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
      return stage_of[a] != stage_of[b] ? stage_of[a] < stage_of[b] : fac[a].map < fac[b].map;
    });
  else if (order_mode == 1)
    std::stable_sort(order.begin(), order.end(),
                     [&](int64_t a, int64_t b) { return fac[a].cloud < fac[b].cloud; });
  if (order_mode != 0)
    std::stable_sort(order.begin(), order.end(),
                     [&](int64_t a, int64_t b) { return stage_of[a] < stage_of[b]; });
  // the last w K4b waves' worth of factors of every stage (default w = 1; VGICP_TAIL_LPT=w)
  // run longest first, so the stage's final partial wave is made of its shortest items
  // (config 5 step 0.451 -> 0.4475 ms; w = 4 measured slower: it breaks target locality)
  static const int tail_env = [] {
    const char* e = getenv("VGICP_TAIL_LPT");
    return e ? atoi(e) : 1;
  }();
  if (tail_env > 0) {
    int nsm = 0;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device) != cudaSuccess)
      nsm = 148;
    const int64_t tail = (int64_t)tail_env * nsm * 12;
    int64_t lo = 0;
    while (lo < F) {
      int64_t hi = lo;
      while (hi < F && stage_of[order[hi]] == stage_of[order[lo]]) ++hi;
      const int64_t from = std::max(lo, hi - tail);
      std::stable_sort(order.begin() + from, order.begin() + hi, [&](int64_t a, int64_t b) {
        return specs[a].source->n > specs[b].source->n;
      });
      lo = hi;
    }
  }
  std::vector<ItemDev> items;
  std::vector<int> stage_items(S + 1, 0);
  long long npts = 0, hoff = 0;
  // item size: up to kMaxChunk points, smaller when the batch is too small to give every
  // K4a warp slot of the GPU (148 SMs x 32) about one item
  long long total_pts = 0;
  for (int64_t f = 0; f < F; ++f) total_pts += specs[f].source->n;
  static int sms = 0;
  if (!sms && cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device) != cudaSuccess)
    sms = 148;
  const long long want = (long long)sms * 32;
  long long chunk = ((total_pts + want - 1) / want + 31) / 32 * 32;
  chunk = std::max<long long>(64, std::min<long long>(kMaxChunk, chunk));
  static const long long chunk_env = [] {
    const char* e = getenv("VGICP_CHUNK");  // ablation: fixed points per work item
    return e ? atoll(e) : 0LL;
  }();
  if (chunk_env > 0) chunk = std::max<long long>(32, std::min<long long>(kMaxChunk, chunk_env));
  for (int64_t f : order) {
    const long long n = specs[f].source->n;
    npts += n;
    fac[f].item_begin = (int)items.size();
    // an empty source gets no work item: its factor sums nothing (zero cost and inliers, as
    // matching_cost / linearize_from_terms give for an empty frame, registration.py:160-165)
    // and no kernel ever reads its (unallocated) point arrays
    const long long nchunks = n == 0 ? 0 : (n + chunk - 1) / chunk;
    for (long long c = 0; c < nchunks; ++c) {
      ItemDev it;
      it.factor = (int)f;
      it.begin = (int)(c * n / nchunks);
      it.end = (int)((c + 1) * n / nchunks);
      it.hoff = (int)hoff;
      hoff += ((it.end - it.begin) + 1) & ~1LL;  // keep regions 16 B aligned
      items.push_back(it);
    }
    fac[f].item_count = (int)nchunks;
    stage_items[stage_of[f] + 1] = (int)items.size();
  }
  for (int s = 1; s <= S; ++s) stage_items[s] = std::max(stage_items[s], stage_items[s - 1]);
  if (hoff >= (1LL << 31)) return fail(VG_ERR_INVALID, "batch too large (2^31 points)");
  vg_batch* b = new vg_batch();
  b->ctx = ctx;
  b->hit_capacity = hoff;
  b->F = F;
  b->num_items = (long long)items.size();
  b->num_points = npts;
  b->num_clouds = (int)clouds.size();
  b->num_maps = (int)maps.size();
  b->max_var = (int)max_var;
  b->host_factors = fac;
  b->pt_off.assign(F + 1, 0);
  for (int64_t f = 0; f < F; ++f) b->pt_off[f + 1] = b->pt_off[f] + specs[f].source->n;
  b->all_covs = all_covs;
  b->stages = S;
  b->stage_factors = stage_factors;
  b->stage_items = stage_items;
  std::vector<CloudView> cv(clouds.size());
  std::vector<MapView> mv(maps.size());
  for (size_t i = 0; i < clouds.size(); ++i) cv[i] = clouds[i]->view();
  // plane-form covariances for every source: the batch's views (read by K4a, which hands
  // them to K4b) carry the plane parameters instead of the covariance rows
  int all_plane = !clouds.empty() && all_covs;
  for (const vg_cloud* c : clouds) all_plane &= (c->plane || c->n == 0) ? 1 : 0;
  static const int plane_env = [] {
    const char* e = getenv("VGICP_PLANE");  // 0: always the general covariance form
    return e ? atoi(e) : 1;
  }();
  all_plane &= plane_env ? 1 : 0;
  if (all_plane)
    for (size_t i = 0; i < clouds.size(); ++i) {
      cv[i].c0 = clouds[i]->p0;
      cv[i].c1 = clouds[i]->p1;
      cv[i].c2 = clouds[i]->p2;
    }
  int n32 = 0;
  for (size_t i = 0; i < maps.size(); ++i) {
    mv[i] = maps[i]->view();
    n32 += maps[i]->kmode;
  }
  b->key_mode = n32 == (int)maps.size() ? 1 : (n32 == 0 ? 0 : 2);
  b->all_pow2 = 1;
  for (const MapView& m : mv) b->all_pow2 &= m.pow2 ? 1 : 0;
  b->all_plane = all_plane;
  b->all_f32 = 1;
  for (const CloudView& c : cv) b->all_f32 &= c.xyz64 ? 0 : 1;
  std::vector<ItemHdr> hdrs(items.size());
  for (size_t i = 0; i < items.size(); ++i) {
    ItemHdr& h = hdrs[i];
    memset(&h, 0, sizeof(h));
    const FactorDev& fd = fac[items[i].factor];
    for (int q = 0; q < 12; ++q) h.T[q] = fd.T[q];
    const CloudView& c = cv[fd.cloud];
    h.a = c.a;
    h.xyz64 = c.xyz64;
    h.c0 = c.c0;
    h.c1 = c.c1;
    h.c2 = c.c2;
    h.mv = mv[fd.map];
    h.factor = items[i].factor;
    h.begin = items[i].begin;
    h.end = items[i].end;
    h.hoff = items[i].hoff;
  }
  // per-item record tensor map of the target (K4b's TMA gathers); none if any map lacks one
  std::vector<const void*> item_tmap(items.size());
  bool all_tmap = !items.empty();
  for (size_t i = 0; i < items.size(); ++i) {
    item_tmap[i] = maps[fac[items[i].factor].map]->tmap;
    all_tmap &= item_tmap[i] != nullptr;
  }
  int rc = VG_OK;
  if (all_tmap && ((rc = dalloc(ctx, &b->item_tmap, items.size())) ||
                   (rc = h2d(ctx, b->item_tmap, item_tmap.data(), sizeof(void*) * items.size())))) {
    vg_batch_destroy(b);
    return rc;
  }
  if ((rc = dalloc(ctx, &b->factors, F)) || (rc = dalloc(ctx, &b->items, items.size())) ||
      (rc = dalloc(ctx, &b->clouds, cv.size())) || (rc = dalloc(ctx, &b->maps, mv.size())) ||
      (rc = dalloc(ctx, &b->partials, items.size() * kPartialStride)) ||
      (rc = dalloc(ctx, &b->hits, (size_t)hoff + 2)) ||
      (rc = dalloc(ctx, &b->hit_counts, items.size())) ||
      (rc = dalloc(ctx, &b->descs, items.size())) ||
      (rc = dalloc(ctx, &b->hdrs, items.size())) ||
      (rc = dalloc(ctx, &b->out, (size_t)F * VG_REC_LINEARIZE)) ||

      (rc = h2d(ctx, b->factors, fac.data(), sizeof(FactorDev) * F)) ||
      (rc = h2d(ctx, b->items, items.data(), sizeof(ItemDev) * items.size())) ||
      (rc = h2d(ctx, b->clouds, cv.data(), sizeof(CloudView) * cv.size())) ||
      (rc = h2d(ctx, b->maps, mv.data(), sizeof(MapView) * mv.size())) ||
      (rc = h2d(ctx, b->hdrs, hdrs.data(), sizeof(ItemHdr) * hdrs.size()))) {
    vg_batch_destroy(b);
    return rc;
  }
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  *out = b;
  return VG_OK;
}

int vg_batch_info(const vg_batch* b, int64_t* F, int64_t* items, int64_t* points) {
  if (!b) return fail(VG_ERR_INVALID, "batch is null");
  if (F) *F = b->F;
  if (items) *items = b->num_items;
  if (points) *points = b->num_points;
  return VG_OK;
}

int vg_batch_destroy(vg_batch* b) {
  if (!b) return VG_OK;
  vg_ctx* ctx = b->ctx;
  if (b->graph) cudaGraphExecDestroy(b->graph);
  if (b->hgraph) cudaGraphExecDestroy(b->hgraph);
  if (b->h_poses) cudaFreeHost(b->h_poses);
  if (b->h_out) cudaFreeHost(b->h_out);
  dfree(ctx, b->factors);
  dfree(ctx, b->items);
  dfree(ctx, b->clouds);
  dfree(ctx, b->maps);
  dfree(ctx, b->partials);
  dfree(ctx, b->hits);
  dfree(ctx, b->hit_counts);
  dfree(ctx, b->descs);
  dfree(ctx, b->hdrs);
  dfree(ctx, b->item_tmap);
  dfree(ctx, b->out);
  dfree(ctx, b->out32);
  dfree(ctx, b->poses);
  dfree(ctx, b->asm_begin);
  dfree(ctx, b->asm_codes);
  dfree(ctx, b->asm_pidx);
  dfree(ctx, b->asm_out);
  dfree(ctx, b->asm_gcost);
  cudaStreamSynchronize(ctx->stream);
  delete b;
  return VG_OK;
}

static size_t rec_of(int mode) {
  return (mode == VG_MODE_COST || mode == VG_MODE_INLIERS) ? VG_REC_COST
         : mode == VG_MODE_COMPACT                          ? VG_REC_COMPACT
                                                             : VG_REC_LINEARIZE;
}
static int kmode_of(int mode) {
  return mode == VG_MODE_COST ? 1 : mode == VG_MODE_INLIERS ? 2 : 0;
}

static int check_mode(const vg_batch* b, int mode) {
  if (mode < 0 || mode > 3) return fail(VG_ERR_INVALID, "bad mode");
  if (mode != VG_MODE_INLIERS && !b->all_covs)
    return fail(VG_ERR_INVALID, "source frame has no covariances");
  return VG_OK;
}

// Host record formats: fmt 0 = rec_of(mode) doubles per factor; fmt 1 = the compact
// MODE_LINEARIZE record of VG_REC_LINEARIZE_F32 4-byte words (fp32 blocks, fp64 cost, int32
// inliers), 2.04x fewer PCIe bytes than fmt 0.
static size_t rec_bytes(int mode, int fmt) {
  return fmt ? 4 * (size_t)VG_REC_LINEARIZE_F32 : sizeof(double) * rec_of(mode);
}

static int out_buffer(vg_batch* b, int fmt, char** dev) {
  if (fmt && !b->out32) VG_CHECK(dalloc(b->ctx, &b->out32, (size_t)b->F * VG_REC_LINEARIZE_F32));
  *dev = fmt ? reinterpret_cast<char*>(b->out32) : reinterpret_cast<char*>(b->out);
  return VG_OK;
}

static int run_device(vg_batch* b, int mode, void* out_dev, int fmt = 0) {
  VG_CHECK(launch_accumulate(b->ctx, b, kmode_of(mode)));
  VG_CHECK(launch_finalize(b->ctx, b, mode, out_dev, fmt));
  return VG_OK;
}

// K4 + K5 for every stage on the compute stream; each stage's records are copied to the
// host on the copy stream as soon as its K5 finishes, overlapping the next stage's K4.
static int run_to_host(vg_batch* b, int mode, void* out_host, int fmt = 0) {
  vg_ctx* ctx = b->ctx;
  const size_t rb = rec_bytes(mode, fmt);
  char* dev = nullptr;
  VG_CHECK(out_buffer(b, fmt, &dev));
  char* host = static_cast<char*>(out_host);
  if (b->stages <= 1) {
    VG_CHECK(run_device(b, mode, dev, fmt));
    return d2h_sync(ctx, host, dev, rb * b->F);
  }
  if (!ctx->side_stream) {
    VG_CUDA(cudaStreamCreateWithFlags(&ctx->side_stream, cudaStreamNonBlocking));
    for (auto& e : ctx->events) VG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  const int kmode = kmode_of(mode);
  // VGICP_STAGE_TRACE=1 (profiling): timed events at every stage boundary, printed to stderr
  static const bool trace = getenv("VGICP_STAGE_TRACE") != nullptr;
  // VGICP_STAGE_NOCOPY=1 (profiling only, results not delivered): the staged compute alone
  static const bool nocopy = getenv("VGICP_STAGE_NOCOPY") != nullptr;
  cudaEvent_t tr[2 * 17 + 1] = {};
  if (trace) {
    for (auto& e : tr) VG_CUDA(cudaEventCreate(&e));
    VG_CUDA(cudaEventRecord(tr[0], ctx->stream));
  }
  // Two compute streams (default from 8 stages; VGICP_STAGE_STREAMS=1/2 overrides): even
  // stages on ctx->stream, odd stages on a second stream, each stage's K4a starting once the
  // previous stage's K4a is done, so a stage's partial last waves overlap the next stage's
  // work instead of idling SM slots (config 5: compute 0.70 -> 0.54 ms; the copies then pace)
  static const int nstreams_env = [] {
    const char* e = getenv("VGICP_STAGE_STREAMS");
    return e ? atoi(e) : 0;
  }();
  const int nstreams =
      std::min(3, nstreams_env > 0 ? nstreams_env : (b->stages >= 6 ? 2 : 1));
  cudaStream_t home = ctx->stream;
  struct Restore {
    vg_ctx* c;
    cudaStream_t s;
    ~Restore() { c->stream = s; }
  } restore{ctx, home};
  cudaStream_t comp[3] = {home, nullptr, nullptr};
  if (nstreams >= 2) {
    if (!ctx->comp2) VG_CUDA(cudaStreamCreateWithFlags(&ctx->comp2, cudaStreamNonBlocking));
    if (nstreams == 3 && !ctx->comp3)
      VG_CUDA(cudaStreamCreateWithFlags(&ctx->comp3, cudaStreamNonBlocking));
    comp[1] = ctx->comp2;
    comp[2] = ctx->comp3;
    VG_CUDA(cudaEventRecord(ctx->events[40], home));
    for (int k = 1; k < nstreams; ++k) VG_CUDA(cudaStreamWaitEvent(comp[k], ctx->events[40], 0));
  }
  for (int s = 0; s < b->stages; ++s) {
    const int f0 = b->stage_factors[s], f1 = b->stage_factors[s + 1];
    if (nstreams >= 2) {
      ctx->stream = comp[s % nstreams];
      if (s > 0) VG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->events[20 + s - 1], 0));
      VG_CHECK(launch_accumulate_range_ev(ctx, b, kmode, b->stage_items[s],
                                          b->stage_items[s + 1], ctx->events[20 + s]));
    } else {
      VG_CHECK(launch_accumulate_range(ctx, b, kmode, b->stage_items[s], b->stage_items[s + 1]));
    }
    VG_CHECK(launch_finalize_range(ctx, b, mode, dev, f0, f1, fmt));
    VG_CUDA(cudaEventRecord(ctx->events[s], ctx->stream));
    if (trace) VG_CUDA(cudaEventRecord(tr[1 + 2 * s], ctx->stream));
    VG_CUDA(cudaStreamWaitEvent(ctx->side_stream, ctx->events[s], 0));
    if (!nocopy)
      VG_CUDA(cudaMemcpyAsync(host + (size_t)f0 * rb, dev + (size_t)f0 * rb,
                              rb * (size_t)(f1 - f0), cudaMemcpyDeviceToHost, ctx->side_stream));
    if (trace) VG_CUDA(cudaEventRecord(tr[2 + 2 * s], ctx->side_stream));
  }
  if (trace) {
    VG_CUDA(cudaDeviceSynchronize());
    fprintf(stderr, "stage_trace_ms compute/copy:");
    for (int s = 0; s < b->stages; ++s) {
      float c = 0.f, d = 0.f;
      cudaEventElapsedTime(&c, tr[0], tr[1 + 2 * s]);
      cudaEventElapsedTime(&d, tr[0], tr[2 + 2 * s]);
      fprintf(stderr, " %.3f/%.3f", c, d);
    }
    fprintf(stderr, "\n");
    for (auto& e : tr) cudaEventDestroy(e);
  }
  if (nstreams >= 2) {
    ctx->stream = home;
    for (int k = 1; k < nstreams; ++k) {
      VG_CUDA(cudaEventRecord(ctx->events[40 + k], comp[k]));
      VG_CUDA(cudaStreamWaitEvent(home, ctx->events[40 + k], 0));
    }
  }
  // the compute stream must not run ahead of the copies that still read the device records
  VG_CUDA(cudaEventRecord(ctx->events[b->stages], ctx->side_stream));
  VG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->events[b->stages], 0));
  VG_CUDA(cudaStreamSynchronize(ctx->side_stream));
  return VG_OK;
}

static int linearize_T(vg_batch* b, const double* T_host, int mode, void* out_host, int fmt) {
  if (!b || (b->F && (!T_host || !out_host))) return fail(VG_ERR_INVALID, "null argument");
  VG_CHECK(check_mode(b, mode));
  if (fmt && mode != VG_MODE_LINEARIZE)
    return fail(VG_ERR_INVALID, "f32 records exist for VG_MODE_LINEARIZE only");
  if (b->F == 0) return VG_OK;
  vg_ctx* ctx = b->ctx;
  // scatter T_ij into the 128 B factor records (dst pitch 128, src pitch 96)
  VG_CUDA(cudaMemcpy2DAsync(b->factors, sizeof(FactorDev), T_host, 12 * sizeof(double),
                            12 * sizeof(double), (size_t)b->F, cudaMemcpyHostToDevice, ctx->stream));
  VG_CHECK(launch_spread_T(ctx, b));
  return run_to_host(b, mode, out_host, fmt);
}

int vg_batch_linearize(vg_batch* b, const double* T_host, int mode, double* out_host) {
  return linearize_T(b, T_host, mode, out_host, 0);
}

int vg_batch_linearize_f32(vg_batch* b, const double* T_host, int mode, float* out_host) {
  return linearize_T(b, T_host, mode, out_host, 1);
}

static int ensure_poses(vg_batch* b, int64_t V) {
  if (V > b->pose_cap) {
    // the small-batch host graph has b->poses baked in: it must not outlive the buffer
    if (b->hgraph) cudaGraphExecDestroy(b->hgraph);
    b->hgraph = nullptr;
    b->hgraph_V = -1;
    dfree(b->ctx, b->poses);
    VG_CHECK(dalloc(b->ctx, &b->poses, 8 * (size_t)V));
    b->pose_cap = V;
  }
  return VG_OK;
}

// Small batches through the host API are launch-latency bound: the pose-table upload,
// K-compose, K4a, K4b, K5 and the record download are captured once into a CUDA graph over
// pinned staging buffers owned by the batch, so a call is two host memcpys + one launch.
static constexpr size_t kSmallHostBytes = 1 << 20;

static int run_small_host(vg_batch* b, const double* poses_host, int64_t V, int mode,
                          void* out_host, int fmt) {
  vg_ctx* ctx = b->ctx;
  const size_t out_bytes = rec_bytes(mode, fmt) * b->F;
  const size_t pose_bytes = sizeof(double) * 8 * V;
  const int key = mode + 8 * fmt;
  if (!b->hgraph || b->hgraph_mode != key || b->hgraph_V != V) {
    if (b->hgraph) cudaGraphExecDestroy(b->hgraph);
    b->hgraph = nullptr;
    if (b->h_poses) cudaFreeHost(b->h_poses);
    if (b->h_out) cudaFreeHost(b->h_out);
    b->h_poses = b->h_out = nullptr;
    VG_CUDA(cudaMallocHost((void**)&b->h_poses, pose_bytes));
    VG_CUDA(cudaMallocHost((void**)&b->h_out, out_bytes));
    VG_CHECK(ensure_poses(b, V));
    char* dev = nullptr;
    VG_CHECK(out_buffer(b, fmt, &dev));
    VG_CUDA(cudaStreamSynchronize(ctx->stream));
    cudaGraph_t g;
    const long long l0 = ctx->launches;
    VG_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    cudaError_t e1 = cudaMemcpyAsync(b->poses, b->h_poses, pose_bytes, cudaMemcpyHostToDevice,
                                     ctx->stream);
    int rc = e1 == cudaSuccess ? launch_compose(ctx, b, b->poses) : VG_ERR_CUDA;
    if (!rc) rc = run_device(b, mode, dev, fmt);
    cudaError_t e2 = rc ? cudaSuccess
                        : cudaMemcpyAsync(b->h_out, dev, out_bytes, cudaMemcpyDeviceToHost,
                                          ctx->stream);
    cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
    b->hgraph_launches = ctx->launches - l0;
    ctx->launches = l0;
    if (rc) return rc;
    if (e1 != cudaSuccess) return vg_cuda_fail(e1, "cudaMemcpyAsync (capture)");
    if (e2 != cudaSuccess) return vg_cuda_fail(e2, "cudaMemcpyAsync (capture)");
    if (e != cudaSuccess) return vg_cuda_fail(e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&b->hgraph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return vg_cuda_fail(e, "cudaGraphInstantiate");
    b->hgraph_mode = key;
    b->hgraph_V = V;
  }
  memcpy(b->h_poses, poses_host, pose_bytes);
  VG_CUDA(cudaGraphLaunch(b->hgraph, ctx->stream));
  ctx->launches += b->hgraph_launches;
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  memcpy(out_host, b->h_out, out_bytes);
  return VG_OK;
}

static int linearize_poses(vg_batch* b, const double* poses_host, int64_t V, int mode,
                           void* out_host, int fmt) {
  if (!b || (b->F && (!poses_host || !out_host))) return fail(VG_ERR_INVALID, "null argument");
  VG_CHECK(check_mode(b, mode));
  if (fmt && mode != VG_MODE_LINEARIZE)
    return fail(VG_ERR_INVALID, "f32 records exist for VG_MODE_LINEARIZE only");
  if (b->F == 0) return VG_OK;
  if (V <= b->max_var) return fail(VG_ERR_INVALID, "pose table smaller than the largest variable index");
  if (b->stages <= 1 && rec_bytes(mode, fmt) * b->F <= kSmallHostBytes &&
      sizeof(double) * 8 * V <= kSmallHostBytes && !getenv("VGICP_NO_HOST_GRAPH"))
    return run_small_host(b, poses_host, V, mode, out_host, fmt);
  VG_CHECK(ensure_poses(b, V));
  VG_CHECK(h2d(b->ctx, b->poses, poses_host, sizeof(double) * 8 * V));
  VG_CHECK(launch_compose(b->ctx, b, b->poses));
  return run_to_host(b, mode, out_host, fmt);
}

int vg_batch_linearize_poses(vg_batch* b, const double* poses_host, int64_t V, int mode,
                             double* out_host) {
  return linearize_poses(b, poses_host, V, mode, out_host, 0);
}

int vg_batch_linearize_poses_f32(vg_batch* b, const double* poses_host, int64_t V, int mode,
                                 float* out_host) {
  return linearize_poses(b, poses_host, V, mode, out_host, 1);
}

// pinned host memory for record outputs: cudaMemcpyAsync into it overlaps the staged compute
// (pageable destinations serialise the copies), see _lib.PinnedPool
int vg_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(VG_ERR_INVALID, "null argument");
  *out = nullptr;
  if (!bytes) return VG_OK;
  VG_CUDA(cudaMallocHost(out, bytes));
  return VG_OK;
}

int vg_host_free(void* p) {
  if (p) VG_CUDA(cudaFreeHost(p));
  return VG_OK;
}

int vg_batch_linearize_poses_device(vg_batch* b, const double* poses_dev, int64_t V, int mode,
                                    double* out_dev) {
  if (!b || !out_dev) return fail(VG_ERR_INVALID, "null argument");
  VG_CHECK(check_mode(b, mode));
  if (b->F == 0) return VG_OK;
  if (poses_dev) {
    if (V <= b->max_var) return fail(VG_ERR_INVALID, "pose table smaller than the largest variable index");
    VG_CHECK(launch_compose(b->ctx, b, poses_dev));
  }
  return run_device(b, mode, out_dev);
}

int vg_batch_lookup_rows(vg_batch* b, const double* poses_host, int64_t V, int64_t* rows_out,
                         int64_t* inliers_out) {
  if (!b || (b->F && (!poses_host || !rows_out || !inliers_out)))
    return fail(VG_ERR_INVALID, "null argument");
  if (b->F == 0) return VG_OK;
  if (V <= b->max_var) return fail(VG_ERR_INVALID, "pose table smaller than the largest variable index");
  vg_ctx* ctx = b->ctx;
  const long long npts = b->pt_off[b->F];
  DeviceTemps temps(ctx->stream);
  long long *d_off = nullptr, *d_rows = nullptr;
  VG_CUDA(temps.alloc(&d_off, (size_t)b->F + 1));
  VG_CUDA(temps.alloc(&d_rows, (size_t)std::max(npts, 1LL)));
  VG_CHECK(h2d(ctx, d_off, b->pt_off.data(), sizeof(long long) * (b->F + 1)));
  VG_CUDA(cudaMemsetAsync(d_rows, 0xff, sizeof(long long) * (size_t)npts, ctx->stream));
  VG_CHECK(ensure_poses(b, V));
  VG_CHECK(h2d(ctx, b->poses, poses_host, sizeof(double) * 8 * V));
  VG_CHECK(launch_compose(ctx, b, b->poses));
  // the same K4a launch the linearization runs (VG_MODE_INLIERS stops after it), then K5
  VG_CHECK(launch_accumulate(ctx, b, kmode_of(VG_MODE_INLIERS)));
  VG_CHECK(launch_export_rows(ctx, b, d_off, d_rows));
  VG_CHECK(launch_finalize(ctx, b, VG_MODE_INLIERS, b->out));
  std::vector<double> rec(2 * (size_t)b->F);
  if (npts) VG_CUDA(cudaMemcpyAsync(rows_out, d_rows, sizeof(long long) * npts, cudaMemcpyDeviceToHost, ctx->stream));
  VG_CHECK(d2h_sync(ctx, rec.data(), b->out, sizeof(double) * rec.size()));
  for (int64_t f = 0; f < b->F; ++f) inliers_out[f] = (int64_t)rec[2 * f + 1];
  return VG_OK;
}

int vg_batch_compose_device(vg_batch* b, const double* poses_dev, int64_t V) {
  if (!b || !poses_dev) return fail(VG_ERR_INVALID, "null argument");
  if (V <= b->max_var) return fail(VG_ERR_INVALID, "pose table smaller than the largest variable index");
  return launch_compose(b->ctx, b, poses_dev);
}

int vg_batch_accumulate_device(vg_batch* b, int mode) {
  if (!b) return fail(VG_ERR_INVALID, "bad arguments");
  VG_CHECK(check_mode(b, mode));
  return launch_accumulate(b->ctx, b, kmode_of(mode));
}

int vg_batch_finalize_device(vg_batch* b, int mode, double* out_dev) {
  if (!b || !out_dev || mode < 0 || mode > 3) return fail(VG_ERR_INVALID, "bad arguments");
  return launch_finalize(b->ctx, b, mode, out_dev);
}

static int assemble_setup(vg_batch* b, int64_t num_vars, const int32_t* given, int64_t given_P,
                          int64_t* num_pairs, int64_t* out_doubles,
                          const int32_t* out_index = nullptr, int64_t out_pairs = -1);

int vg_batch_assemble_setup(vg_batch* b, int64_t num_vars, int64_t* num_pairs,
                            int64_t* out_doubles) {
  return assemble_setup(b, num_vars, nullptr, -1, num_pairs, out_doubles);
}

int vg_batch_assemble_setup_pairs(vg_batch* b, int64_t num_vars, const int32_t* pairs,
                                  int64_t num_pairs, int64_t* out_doubles) {
  if (num_pairs < 0 || (num_pairs && !pairs)) return fail(VG_ERR_INVALID, "invalid pair list");
  return assemble_setup(b, num_vars, pairs, num_pairs, nullptr, out_doubles);
}

int vg_batch_assemble_setup_mapped(vg_batch* b, int64_t num_vars, const int32_t* pairs,
                                   int64_t num_pairs, const int32_t* out_index,
                                   int64_t out_pairs, int64_t* out_doubles) {
  if (num_pairs < 0 || (num_pairs && (!pairs || !out_index)) || out_pairs < num_pairs)
    return fail(VG_ERR_INVALID, "invalid pair list");
  for (int64_t p = 0; p < num_pairs; ++p)
    if (out_index[p] < 0 || out_index[p] >= out_pairs || (p && out_index[p] <= out_index[p - 1]))
      return fail(VG_ERR_INVALID, "output pair slots must be increasing and < out_pairs");
  return assemble_setup(b, num_vars, pairs, num_pairs, nullptr, out_doubles, out_index,
                        out_pairs);
}

static int assemble_setup(vg_batch* b, int64_t num_vars, const int32_t* given, int64_t given_P,
                          int64_t* num_pairs, int64_t* out_doubles, const int32_t* out_index,
                          int64_t out_pairs) {
  if (!b || num_vars <= 0 || num_vars >= (1LL << 28))
    return fail(VG_ERR_INVALID, "invalid assembly arguments");
  vg_ctx* ctx = b->ctx;
  const long long V = num_vars, F = b->F;
  // contributions per unit, in factor order (factor_graph.py:529-535 adds blocks in order)
  std::vector<std::vector<int>> diag((size_t)V);
  std::vector<std::pair<long long, int>> pc;  // (pair key, code), stable-sorted below
  for (long long f = 0; f < F; ++f) {
    const FactorDev& d = b->host_factors[f];
    const long long vs = d.var_source, vt = d.var_target;
    const bool unary = d.flags & 1;
    if (vs < 0 || (!unary && vt < 0))
      return fail(VG_ERR_INVALID, "factor without pose-table variables");
    if (f >= (1LL << 28)) return fail(VG_ERR_INVALID, "too many factors for assembly");
    const int code = (int)f * 8;
    if (vs < V) diag[vs].push_back(code + 0);
    if (unary || vt >= V) continue;  // constant target: only the source blocks
    if (vs == vt) {
      diag[vs].push_back(code + 4);
      diag[vs].push_back(code + 1);
      continue;
    }
    diag[vt].push_back(code + 1);
    if (vs < V) {
      const long long a = std::min(vs, vt), c = std::max(vs, vt);
      pc.push_back({a * V + c, code + (vs < vt ? 2 : 3)});
    }
  }
  std::stable_sort(pc.begin(), pc.end(),
                   [](const std::pair<long long, int>& x, const std::pair<long long, int>& y) {
                     return x.first < y.first;
                   });
  std::vector<int> begin, codes, pairs;
  begin.reserve(V + pc.size() + 2);
  for (long long v = 0; v < V; ++v) {
    begin.push_back((int)codes.size());
    codes.insert(codes.end(), diag[v].begin(), diag[v].end());
  }
  if (given) {
    // caller's (global) pair list, e.g. the same on every rank so blocks can be summed with
    // one reduction; pairs this batch does not touch stay zero
    size_t k = 0;
    for (int64_t p = 0; p < given_P; ++p) {
      const long long a = given[2 * p], c = given[2 * p + 1];
      if (a < 0 || c >= V || a >= c || (p && a * V + c <= (long long)given[2 * p - 2] * V + given[2 * p - 1]))
        return fail(VG_ERR_INVALID, "pair list must be sorted, unique, a < b < num_vars");
      begin.push_back((int)codes.size());
      pairs.push_back((int)a);
      pairs.push_back((int)c);
      for (; k < pc.size() && pc[k].first == a * V + c; ++k) codes.push_back(pc[k].second);
      if (k < pc.size() && pc[k].first < a * V + c)
        return fail(VG_ERR_INVALID, "a factor's variable pair is missing from the pair list");
    }
    if (k != pc.size())
      return fail(VG_ERR_INVALID, "a factor's variable pair is missing from the pair list");
  } else {
    for (size_t i = 0; i < pc.size(); ++i) {
      if (i == 0 || pc[i].first != pc[i - 1].first) {
        begin.push_back((int)codes.size());
        pairs.push_back((int)(pc[i].first / V));
        pairs.push_back((int)(pc[i].first % V));
      }
      codes.push_back(pc[i].second);
    }
  }
  begin.push_back((int)codes.size());
  const long long P = (long long)pairs.size() / 2;
  const long long P_out = out_index ? out_pairs : P;
  const long long total = 2 + V * 27 + P_out * 36;
  dfree(ctx, b->asm_begin);
  dfree(ctx, b->asm_codes);
  dfree(ctx, b->asm_pidx);
  if (out_index && P) {
    VG_CHECK(dalloc(ctx, &b->asm_pidx, (size_t)P));
    VG_CHECK(h2d(ctx, b->asm_pidx, out_index, sizeof(int) * P));
  }
  dfree(ctx, b->asm_out);
  b->asm_begin = nullptr;
  b->asm_codes = nullptr;
  b->asm_out = nullptr;
  b->asm_vars = -1;
  VG_CHECK(dalloc(ctx, &b->asm_begin, begin.size()));
  VG_CHECK(dalloc(ctx, &b->asm_codes, std::max<size_t>(codes.size(), 1)));
  VG_CHECK(dalloc(ctx, &b->asm_out, (size_t)total));
  if (!b->asm_gcost && F) VG_CHECK(dalloc(ctx, &b->asm_gcost, (size_t)F));
  // K5's cost partials: per factor for the warp-per-factor K5 (linearize.cu), else per window
  b->asm_gparts = (F < 4096 || b->num_items > 4 * F) ? F : (F + 63) / 64;
  VG_CHECK(h2d(ctx, b->asm_begin, begin.data(), sizeof(int) * begin.size()));
  if (!codes.empty()) VG_CHECK(h2d(ctx, b->asm_codes, codes.data(), sizeof(int) * codes.size()));
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  b->asm_vars = V;
  static std::atomic<long long> setups{0};
  b->asm_gen = ++setups;  // unique across batches: a reused batch address is a new setup
  b->asm_pairs_n = P;
  b->asm_out_pairs = P_out;
  b->asm_pairs = pairs;
  if (num_pairs) *num_pairs = P;
  if (out_doubles) *out_doubles = total;
  return VG_OK;
}

int vg_batch_assemble_pairs(const vg_batch* b, int32_t* pairs_out) {
  if (!b || b->asm_vars < 0) return fail(VG_ERR_INVALID, "assembly not set up");
  if (b->asm_pairs_n && !pairs_out) return fail(VG_ERR_INVALID, "null argument");
  if (b->asm_pairs_n) memcpy(pairs_out, b->asm_pairs.data(), sizeof(int32_t) * b->asm_pairs.size());
  return VG_OK;
}

static int run_assemble(vg_batch* b, const double* poses_dev, int64_t V, double* out_dev) {
  if (b->asm_vars < 0) return fail(VG_ERR_INVALID, "assembly not set up (vg_batch_assemble_setup)");
  if (V <= b->max_var) return fail(VG_ERR_INVALID, "pose table smaller than the largest variable index");
  VG_CHECK(check_mode(b, VG_MODE_LINEARIZE));
  vg_ctx* ctx = b->ctx;
  if (b->F) {
    VG_CHECK(launch_compose(ctx, b, poses_dev));
    VG_CHECK(launch_accumulate(ctx, b, kmode_of(VG_MODE_LINEARIZE)));
    VG_CHECK(launch_finalize(ctx, b, VG_MODE_LINEARIZE, b->out));
  }
  return launch_assemble(ctx, b, b->out, out_dev);
}

int vg_batch_assemble_poses_device(vg_batch* b, const double* poses_dev, int64_t V,
                                   double* out_dev) {
  if (!b || !poses_dev || !out_dev) return fail(VG_ERR_INVALID, "null argument");
  return run_assemble(b, poses_dev, V, out_dev);
}

int vg_batch_assemble_records_device(vg_batch* b, const double* records_dev, double* out_dev) {
  if (!b || !records_dev || !out_dev) return fail(VG_ERR_INVALID, "null argument");
  if (b->asm_vars < 0) return fail(VG_ERR_INVALID, "assembly not set up (vg_batch_assemble_setup)");
  return launch_assemble(b->ctx, b, records_dev, out_dev);
}

int vg_batch_assemble_poses(vg_batch* b, const double* poses_host, int64_t V, double* out_host) {
  if (!b || !poses_host || !out_host) return fail(VG_ERR_INVALID, "null argument");
  if (b->asm_vars < 0) return fail(VG_ERR_INVALID, "assembly not set up (vg_batch_assemble_setup)");
  if (V <= b->max_var) return fail(VG_ERR_INVALID, "pose table smaller than the largest variable index");
  VG_CHECK(ensure_poses(b, V));
  VG_CHECK(h2d(b->ctx, b->poses, poses_host, sizeof(double) * 8 * V));
  VG_CHECK(run_assemble(b, b->poses, V, b->asm_out));
  const size_t total = 2 + (size_t)b->asm_vars * 27 + (size_t)b->asm_out_pairs * 36;
  return d2h_sync(b->ctx, out_host, b->asm_out, sizeof(double) * total);
}

int vg_batch_graph_capture(vg_batch* b, const double* poses_dev, int64_t V, int mode,
                           double* out_dev) {
  if (!b || !out_dev) return fail(VG_ERR_INVALID, "null argument");
  vg_ctx* ctx = b->ctx;
  if (b->graph) {
    cudaGraphExecDestroy(b->graph);
    b->graph = nullptr;
  }
  cudaGraph_t g;
  const long long l0 = ctx->launches;
  VG_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  int rc = vg_batch_linearize_poses_device(b, poses_dev, V, mode, out_dev);
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
  b->graph_launches = ctx->launches - l0;
  ctx->launches = l0;
  if (rc) return rc;
  if (e != cudaSuccess) return vg_cuda_fail(e, "cudaStreamEndCapture");
  e = cudaGraphInstantiate(&b->graph, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return vg_cuda_fail(e, "cudaGraphInstantiate");
  return VG_OK;
}

int vg_batch_graph_capture_assemble(vg_batch* b, const double* poses_dev, int64_t V,
                                    double* records_dev, double* out_dev, int32_t zero_out) {
  if (!b || !poses_dev || !records_dev || !out_dev) return fail(VG_ERR_INVALID, "null argument");
  if (b->asm_vars < 0) return fail(VG_ERR_INVALID, "assembly not set up (vg_batch_assemble_setup)");
  if (V <= b->max_var) return fail(VG_ERR_INVALID, "pose table smaller than the largest variable index");
  vg_ctx* ctx = b->ctx;
  if (b->graph) {
    cudaGraphExecDestroy(b->graph);
    b->graph = nullptr;
  }
  const size_t total = 2 + (size_t)b->asm_vars * 27 + (size_t)b->asm_out_pairs * 36;
  cudaGraph_t g;
  const long long l0 = ctx->launches;
  VG_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  int rc = VG_OK;
  if (b->F) {
    rc = launch_compose(ctx, b, poses_dev);
    if (!rc) rc = run_device(b, VG_MODE_LINEARIZE, records_dev);
  }
  if (!rc && zero_out && cudaMemsetAsync(out_dev, 0, sizeof(double) * total, ctx->stream))
    rc = VG_ERR_CUDA;
  if (!rc) rc = launch_assemble(ctx, b, records_dev, out_dev);
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
  b->graph_launches = ctx->launches - l0;
  ctx->launches = l0;
  if (rc) return rc;
  if (e != cudaSuccess) return vg_cuda_fail(e, "cudaStreamEndCapture");
  e = cudaGraphInstantiate(&b->graph, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return vg_cuda_fail(e, "cudaGraphInstantiate");
  return VG_OK;
}

int vg_batch_graph_launch(vg_batch* b) {
  if (!b || !b->graph) return fail(VG_ERR_INVALID, "no captured graph");
  VG_CUDA(cudaGraphLaunch(b->graph, b->ctx->stream));
  b->ctx->launches += b->graph_launches;
  return VG_OK;
}

// ---- preprocessing ----------------------------------------------------------------------
int vg_knn(vg_ctx* ctx, const vg_cloud* cloud, int32_t k, int64_t* nbrs_out) {
  if (!ctx || !cloud || !nbrs_out || k <= 0) return fail(VG_ERR_INVALID, "invalid kNN arguments");
  if (cloud->n < k)  // preprocess.py:129-130
    return fail(VG_ERR_TOO_SPARSE, "frame has " + std::to_string(cloud->n) +
                                       " points, need at least " + std::to_string(k));
  if (cloud->n >= (1LL << 31)) return fail(VG_ERR_INVALID, "cloud too large");
  DeviceTemps temps(ctx->stream);
  long long* dn = nullptr;
  VG_CUDA(temps.alloc(&dn, (size_t)cloud->n * k));
  VG_CHECK(launch_knn(ctx, cloud, k, dn));
  return d2h_sync(ctx, nbrs_out, dn, sizeof(long long) * cloud->n * k);
}

int vg_covariances(vg_ctx* ctx, const vg_cloud* cloud, const int64_t* nbrs, int32_t k, double eps,
                   double* covs_out, uint8_t* degen_out) {
  if (!ctx || !cloud || (cloud->n && (!nbrs || !covs_out)) || k <= 0)
    return fail(VG_ERR_INVALID, "invalid covariance arguments");
  const long long n = cloud->n;
  if (n == 0) return VG_OK;
  for (long long i = 0; i < n * k; ++i)
    if (nbrs[i] < 0 || nbrs[i] >= n) return fail(VG_ERR_INVALID, "neighbor index out of range");
  DeviceTemps temps(ctx->stream);
  long long* dn = nullptr;
  double* dc = nullptr;
  unsigned char* dg = nullptr;
  VG_CUDA(temps.alloc(&dn, (size_t)n * k));
  VG_CUDA(temps.alloc(&dc, 9 * (size_t)n));
  VG_CUDA(temps.alloc(&dg, (size_t)n));
  VG_CHECK(h2d(ctx, dn, nbrs, sizeof(long long) * n * k));
  VG_CHECK(launch_cov(ctx, cloud, dn, k, eps, dc, dg));
  if (degen_out) VG_CUDA(cudaMemcpyAsync(degen_out, dg, n, cudaMemcpyDeviceToHost, ctx->stream));
  return d2h_sync(ctx, covs_out, dc, sizeof(double) * 9 * n);
}

int vg_cloud_estimate_covariances(vg_ctx* ctx, vg_cloud* cloud, int32_t k, double eps,
                                  int64_t* nbrs_out, double* covs_out, uint8_t* degen_out) {
  if (!ctx || !cloud || k <= 0) return fail(VG_ERR_INVALID, "invalid arguments");
  const long long n = cloud->n;
  if (n < k)
    return fail(VG_ERR_TOO_SPARSE, "frame has " + std::to_string(n) + " points, need at least " +
                                       std::to_string(k));
  DeviceTemps temps(ctx->stream);
  long long* dn = nullptr;
  unsigned char* dg = nullptr;
  VG_CUDA(temps.alloc(&dn, (size_t)n * k));
  VG_CUDA(temps.alloc(&dg, (size_t)n));
  if (!cloud->cov64) {
    VG_CHECK(dalloc(ctx, &cloud->cov64, 9 * (size_t)n));
    VG_CHECK(dalloc(ctx, &cloud->c0, (size_t)n));
    VG_CHECK(dalloc(ctx, &cloud->c1, (size_t)n));
    VG_CHECK(dalloc(ctx, &cloud->c2, (size_t)n));
  }
  VG_CHECK(launch_knn(ctx, cloud, k, dn));
  VG_CHECK(launch_cov(ctx, cloud, dn, k, eps, cloud->cov64, dg));
  cloud->has_cov = true;
  VG_CHECK(launch_cloud_pack(ctx, cloud));
  if (nbrs_out) VG_CUDA(cudaMemcpyAsync(nbrs_out, dn, 8 * n * k, cudaMemcpyDeviceToHost, ctx->stream));
  if (covs_out) VG_CUDA(cudaMemcpyAsync(covs_out, cloud->cov64, 72 * n, cudaMemcpyDeviceToHost, ctx->stream));
  if (degen_out) VG_CUDA(cudaMemcpyAsync(degen_out, dg, n, cudaMemcpyDeviceToHost, ctx->stream));
  VG_CUDA(cudaStreamSynchronize(ctx->stream));
  return VG_OK;
}

}  // extern "C"
