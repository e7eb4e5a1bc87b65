// internal.h — host-side objects behind the opaque C-ABI handles and the kernel launchers.
#pragma once
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"
#include "vgicp.h"

struct vg_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;  // where all work is enqueued
  cudaStream_t side_stream = nullptr;  // host-output copies of the staged pipeline
  cudaStream_t comp2 = nullptr;        // second compute stream (odd stages, overlapped)
  cudaStream_t comp3 = nullptr;        // third compute stream (VGICP_STAGE_STREAMS=3)
  cudaEvent_t events[65] = {};
  long long launches = 0;         // kernels launched (bench evidence)
  // scratch (grown on demand, stream-ordered reuse)
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
};

struct vg_cloud {
  vg_ctx* ctx = nullptr;
  long long n = 0;
  bool has_cov = false;
  bool exact32 = true;
  float4* a = nullptr;       // x, y, z fp32
  double2* c0 = nullptr;     // covariance SoA (fp64)
  double2* c1 = nullptr;
  double2* c2 = nullptr;
  double* xyz64 = nullptr;  // always kept: fp64 points (map build, kNN)
  double* cov64 = nullptr;  // n*9 fp64 covariances (bit-exact map build), or null
  double2* p0 = nullptr;    // plane form alpha I - kappa n n^T of every covariance (map_build.cu)
  double2* p1 = nullptr;
  double2* p2 = nullptr;
  bool plane = false;       // every covariance has the plane form
  vg::CloudView view() const {
    vg::CloudView v;
    v.a = a;
    v.c0 = has_cov ? c0 : nullptr;
    v.c1 = has_cov ? c1 : nullptr;
    v.c2 = has_cov ? c2 : nullptr;
    v.xyz64 = exact32 ? nullptr : xyz64;
    v.n = n;
    return v;
  }
};

struct vg_map {
  vg_ctx* ctx = nullptr;
  long long m = 0;
  double res = 1.0;
  unsigned capacity = 0;
  int log2cap = 0;
  long long* pkeys = nullptr;     // kmode 0 probe keys (capacity)
  int* prows = nullptr;           // kmode 0 row per slot (capacity)
  unsigned* pkeys32 = nullptr;    // kmode 1 keys (capacity)
  vg::VoxelRec* recs = nullptr;   // kmode 1: capacity, slot-indexed; kmode 0: m, row-indexed
  void* tmap = nullptr;           // device CUtensorMap of recs (rows x 16 fp64, box 10 x 1) for
                                  // K4b's TMA gather4 record fetches, or null
  long long empty_key = 0;
  int kmode = 0;
  int bx = 0, by = 0, bz = 0, ex = 0, ey = 0, ez = 0;
  // reference arrays (device, fp64/int64): keys sorted ascending, means m*3, covs m*9
  long long* keys = nullptr;
  double* means = nullptr;
  double* covs = nullptr;
  long long* counts = nullptr;
  vg::MapView view() const {
    vg::MapView v;
    v.keys = pkeys;
    v.rows = prows;
    v.keys32 = pkeys32;
    v.recs = recs;
    v.empty_key = empty_key;
    v.kmode = kmode;
    v.bx = bx;
    v.by = by;
    v.bz = bz;
    v.ex = ex;
    v.ey = ey;
    v.ez = ez;
    v.res = res;
    v.inv_res = 1.0 / res;
    v.mask = (capacity / (kmode ? vg::kBucket32 : vg::kBucket)) - 1;
    v.shift = kmode ? 32 - (log2cap - 2) : 64 - (log2cap - 3);
    v.m = (int)m;
    int e2 = 0;
    v.pow2 = (std::frexp(res, &e2) == 0.5) ? 1 : 0;
    return v;
  }
};

struct vg_batch {
  vg_ctx* ctx = nullptr;
  long long F = 0;
  long long num_items = 0;
  long long num_points = 0;
  int num_clouds = 0;
  int num_maps = 0;
  int max_var = -1;
  int key_mode = 2;                   // 1: all maps 32-bit local keys, 0: all int64, 2: mixed
  int all_pow2 = 0;                   // every map's resolution is a power of two
  int all_f32 = 0;                    // every source point is fp32-exact (no xyz64 copy)
  int all_plane = 0;                  // every source covariance has the plane form (c0..c2 of
                                      // the batch's cloud views then point at p0..p2)
  bool all_covs = true;               // every source has covariances (else INLIERS mode only)
  vg::FactorDev* factors = nullptr;   // F
  vg::ItemDev* items = nullptr;       // num_items (ordered by target map, then factor)
  vg::CloudView* clouds = nullptr;    // num_clouds
  vg::MapView* maps = nullptr;        // num_maps
  double* partials = nullptr;         // num_items * kPartialStride
  int2* hits = nullptr;               // compacted (point, slot) hits, per-item regions
  int* hit_counts = nullptr;          // num_items
  vg::AccDesc* descs = nullptr;       // num_items (K4a -> K4b)
  vg::ItemHdr* hdrs = nullptr;        // num_items (K4a fast-path headers; T refreshed per step)
  const void** item_tmap = nullptr;   // num_items: the target map's record tensor map (TMA)
  long long hit_capacity = 0;
  double* poses = nullptr;            // pose table (device), capacity pose_cap
  long long pose_cap = 0;
  double* out = nullptr;              // device output (F * 92)
  unsigned* out32 = nullptr;          // device output of the f32 records (F * 94 words, lazy)
  // pipelined host-output path: stage s = factors [stage_factors[s], stage_factors[s+1]),
  // whose items are exactly [stage_items[s], stage_items[s+1]) (items are stage-major)
  int stages = 1;
  std::vector<int> stage_factors, stage_items;
  cudaGraphExec_t graph = nullptr;
  long long graph_launches = 0;
  // small-batch host path: graph over pinned staging (see run_small_host in capi.cu)
  cudaGraphExec_t hgraph = nullptr;
  long long hgraph_launches = 0;
  int hgraph_mode = -1;
  long long hgraph_V = -1;
  double* h_poses = nullptr;
  double* h_out = nullptr;
  std::vector<vg::FactorDev> host_factors;
  std::vector<long long> pt_off;      // F + 1: first point of each factor in spec order
                                      // (vg_batch_lookup_rows output layout)
  // normal-equation assembly (vg_batch_assemble_*): CSR of contributions per output unit
  long long asm_vars = -1;            // variables (pose-table rows < asm_vars); -1: not set up
  long long asm_gen = 0;              // unique id of the current assembly setup (consumers' caches)
  long long asm_pairs_n = 0;
  std::vector<int> asm_pairs;         // P x 2 (a < b)
  int* asm_begin = nullptr;           // units + 1
  int* asm_codes = nullptr;           // factor * 8 + role
  int* asm_pidx = nullptr;            // P: output slot of each pair block (mapped setup) or null
  long long asm_out_pairs = 0;        // pair blocks in the output layout (>= asm_pairs_n)
  double* asm_out = nullptr;          // device output (host-buffer entry point)
  double2* asm_gcost = nullptr;       // gated (cost, count) partials written by K5: one per
                                      // 64-factor window (k_finalize) or per factor (warp K5)
  long long asm_gparts = 0;           // how many (K6's cost unit sums them)
};

// Programmatic dependent launch: the kernel may be scheduled while its stream predecessor
// drains (it waits in griddepcontrol.wait before touching the predecessor's results), hiding
// the launch gap between the kernels of a step.
template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_release() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Stream-ordered device temporaries of one call, released on every exit path.
struct DeviceTemps {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit DeviceTemps(cudaStream_t s) : st(s) {}
  DeviceTemps(const DeviceTemps&) = delete;
  DeviceTemps& operator=(const DeviceTemps&) = delete;
  template <class T>
  cudaError_t alloc(T** p, size_t count) {
    *p = nullptr;
    if (count == 0) return cudaSuccess;
    const cudaError_t e = cudaMallocAsync((void**)p, sizeof(T) * count, st);
    if (e == cudaSuccess) ptrs.push_back((void*)*p);
    return e;
  }
  ~DeviceTemps() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};

// error plumbing (capi.cu)
void vg_set_error(const std::string& msg);
int vg_cuda_fail(cudaError_t e, const char* what);
#define VG_CUDA(call)                                        \
  do {                                                       \
    cudaError_t _e = (call);                                 \
    if (_e != cudaSuccess) return vg_cuda_fail(_e, #call);   \
  } while (0)

#define VG_CHECK(x)               \
  do {                            \
    int _rc = (x);                \
    if (_rc != VG_OK) return _rc; \
  } while (0)

// scratch helpers
int vg_scratch(vg_ctx* ctx, size_t bytes, void** out);

// ---- launchers (each returns VG_OK or an error code; all stream-ordered on ctx) ----
int launch_pack_keys(vg_ctx* ctx, const double* xyz_dev, long long n, double res,
                     long long* keys_dev);
int launch_cloud_pack(vg_ctx* ctx, vg_cloud* cloud);  // fp64 xyz/cov -> fp32 SoA
int launch_map_build(vg_ctx* ctx, const vg_cloud* cloud, double res, vg_map* map);
// per-point deskew (preprocess.py:218-231) from host arrays into host outputs
int launch_deskew(vg_ctx* ctx, const double* xyz, const double* stamps, long long n,
                  const double* node_t, const double* quats, const double* trans, int K,
                  double* xyz_out);
// voxel_downsample (preprocess.py:73-119) from host arrays into host outputs (capacity n)
int launch_voxel_downsample(vg_ctx* ctx, const double* xyz, const double* stamps, long long n,
                            double res, double tol, double* xyz_out, double* stamps_out,
                            long long* m_out);
// fp64 arrays -> slots + hash; bounds: k_key_bounds' output when the build has it, else null
int launch_map_finish(vg_ctx* ctx, vg_map* map, const long long* bounds = nullptr);
int launch_lookup(vg_ctx* ctx, const vg::CloudView& cv, const vg::MapView& mv,
                  const double* T_dev, long long* rows_dev, unsigned long long* hits_dev);
int launch_terms(vg_ctx* ctx, const vg::CloudView& cv, const vg::MapView& mv,
                 const double* T_dev, long long* rows, double* moved, double* d, double* w,
                 double* wd, double* partial_cost, long long* partial_inl, int nblocks);
int launch_compose(vg_ctx* ctx, vg_batch* b, const double* poses_dev);
// linearize_from_terms over explicit per-point terms (vg_linearize_terms)
int launch_terms_linearize(vg_ctx* ctx, const double* mu_dev, const double* W_dev,
                           const double* wd_dev, long long n, const vg::FactorDev& f,
                           double cost, double inliers, double* out_dev);
int launch_spread_T(vg_ctx* ctx, vg_batch* b);  // FactorDev.T -> ItemHdr.T (explicit-T mode)
int launch_accumulate(vg_ctx* ctx, vg_batch* b, int kmode);  // K4a + K4b
// K5; f32: MODE_LINEARIZE records in the compact host format (VG_REC_LINEARIZE_F32 words)
int launch_finalize(vg_ctx* ctx, vg_batch* b, int mode, void* out_dev, int f32 = 0);
int launch_finalize_range(vg_ctx* ctx, vg_batch* b, int mode, void* out_dev, int f0, int f1,
                          int f32 = 0);
int launch_assemble(vg_ctx* ctx, vg_batch* b, const double* rec, double* out_dev);  // K6
int launch_accumulate_range(vg_ctx* ctx, vg_batch* b, int kmode, int lo, int hi);  // K4a + K4b
// scatter the last K4a pass's hit lists as reference rows (vg_batch_lookup_rows)
int launch_export_rows(vg_ctx* ctx, vg_batch* b, const long long* pt_off_dev, long long* rows_dev);
// the same, recording `after_lookup` on ctx->stream between K4a and K4b
int launch_accumulate_range_ev(vg_ctx* ctx, vg_batch* b, int kmode, int lo, int hi,
                               cudaEvent_t after_lookup);
int launch_knn(vg_ctx* ctx, const vg_cloud* cloud, int k, long long* nbrs_dev);
int launch_cov(vg_ctx* ctx, const vg_cloud* cloud, const long long* nbrs_dev, int k,
               double eps, double* covs_dev, unsigned char* degen_dev);
