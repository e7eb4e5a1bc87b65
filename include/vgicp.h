/*
 * vgicp.h — C-ABI of the B200-native VGICP matching-cost path (libvgicp.so).
 *
 * This is the drop-in boundary for the hot path of arXiv 2202.00242 as restated by the
 * reference package `limapper` (pure Python/NumPy).  Every entry point below replaces one
 * reference function; the citation is `file:line` under /root/reference/pkg/src/limapper/.
 * The Python mirror of the reference API (paper_2202_00242_b200/registration.py,
 * preprocess.py, factor_graph.py) binds these with ctypes.
 *
 * Conventions
 *   - Plain pointers and sizes only; no torch/CUDA types in signatures (streams are void*).
 *   - Host arrays are C-contiguous float64 / int64, caller-owned and only borrowed for the
 *     duration of the call.  Device objects (ctx, cloud, map, batch) are owned by handles.
 *   - A rigid transform "T" is 12 doubles: R row-major (9) then t (3); p' = R p + t.
 *   - A pose-table entry is 8 doubles: quaternion (x, y, z, w) then translation (3), then
 *     one pad — the layout of limapper.geometry.Se3Pose (geometry.py:47-60,208-237).
 *   - Every function returns a status code (VG_OK == 0).  vg_last_error() returns a
 *     thread-local message for the last failure.  Nothing throws or longjmps across the ABI.
 *   - Results are deterministic: fixed-order reductions, no floating-point atomics.
 */
#ifndef VGICP_H_
#define VGICP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VGICP_ABI_VERSION 1

/* status codes; the Python wrapper maps each to the reference exception type */
#define VG_OK 0
#define VG_ERR_INVALID 1    /* ValueError (registration.py:80-81, preprocess.py:149-150) */
#define VG_ERR_CUDA 2       /* RuntimeError: a CUDA call failed */
#define VG_ERR_DEGENERATE 3 /* DegenerateConstraint (errors.py:24-25, registration.py:213-215) */
#define VG_ERR_TOO_SPARSE 4 /* FrameTooSparse (errors.py:8-9, preprocess.py:129-130) */
#define VG_ERR_NOMEM 5      /* MemoryError: device allocation failed */

/* batch evaluation modes and per-factor output record sizes (doubles) */
#define VG_MODE_LINEARIZE 0 /* blocks: H_ii(21) H_ij(36) H_jj(21) b_i(6) b_j(6) cost inliers */
#define VG_MODE_COST 1      /* cost inliers */
#define VG_MODE_COMPACT 2   /* H'(21) b'(6) cost inliers: pre-adjoint record */
#define VG_MODE_INLIERS 3   /* 0 inliers: correspondence counts only (overlap gating) */
#define VG_REC_LINEARIZE 92
#define VG_REC_COST 2
#define VG_REC_COMPACT 29
/* compact host record of VG_MODE_LINEARIZE (the *_f32 entry points), 94 4-byte words:
 * words 0-89 the blocks H_ii(21) H_ij(36) H_jj(21) b_i(6) b_j(6) in fp32 (the north_star's
 * fp32 H/b, each within 1e-4 rel / 1e-6 abs of the fp64 reference), words 90-91 the cost as
 * fp64 (low word first), word 92 the inlier count (int32), word 93 zero padding. */
#define VG_REC_LINEARIZE_F32 94

/* factor flags */
#define VG_FACTOR_UNARY 1 /* target pose fixed (factor_graph.py:219-245) */

typedef struct vg_ctx vg_ctx;
typedef struct vg_cloud vg_cloud;
typedef struct vg_map vg_map;
typedef struct vg_batch vg_batch;

typedef struct vg_factor_spec {
  const vg_cloud* source; /* MatchingCostFactor.source (factor_graph.py:219-229) */
  const vg_map* target;   /* MatchingCostFactor.target_map */
  int32_t flags;          /* VG_FACTOR_UNARY or 0 */
  int32_t min_inliers;    /* MatchingCostFactor.min_inliers (default 10, registration.py:26) */
  int32_t var_source;     /* pose-table index of the source variable (pose-table mode) */
  int32_t var_target;     /* pose-table index of the target variable / fixed pose */
} vg_factor_spec;

/* ---- library / context ---------------------------------------------------------------- */
int vg_abi_version(void);
const char* vg_last_error(void);
int vg_ctx_create(int device, vg_ctx** out);
int vg_ctx_destroy(vg_ctx* ctx);
/* route all work of ctx onto an existing cudaStream_t (NULL = the context's own stream) */
int vg_ctx_set_stream(vg_ctx* ctx, void* stream);
int vg_ctx_synchronize(vg_ctx* ctx);
/* number of kernels this library has launched on ctx so far (bench evidence) */
int vg_ctx_launch_count(const vg_ctx* ctx, int64_t* count);

/* ---- voxel keys ------------------------------------------------------------------------ */
/* replaces pack_voxel_keys (preprocess.py:21-22,68-70): floor(p/res)+2^20 packed 21 bits/axis */
int vg_pack_voxel_keys(vg_ctx* ctx, const double* xyz, int64_t n, double resolution,
                       int64_t* keys_out);
/* replaces voxel_downsample (preprocess.py:73-119): per packed voxel key (ascending), the
 * mean position and mean stamp of its points; a voxel whose stamp spread exceeds split_tol
 * (the reference passes scan.duration / 10) is split into a primary and an overflow cell by
 * the running-mean rule, primary first.  Bit-identical to the reference (its summation
 * orders included).  xyz_out (n x 3) and stamps_out (n) need room for n cells; *m_out
 * receives the cell count.  VG_ERR_INVALID when resolution <= 0. */
int vg_voxel_downsample(vg_ctx* ctx, const double* xyz, const double* stamps, int64_t n,
                        double resolution, double split_tol, double* xyz_out,
                        double* stamps_out, int64_t* m_out);

/* replaces the per-point half of deskew (preprocess.py:218-231): each point's segment of the
 * node trajectory (node_t ascending, K >= 2; searchsorted side="right", clipped), the slerped
 * node quaternion (xyzw, _slerp_batch :167-178) and linearly interpolated translation at its
 * stamp, and p' = p + 2w(u x p) + 2u x (u x p) + t.  The node trajectory is what the
 * reference integrates on the host from the IMU (:199-216).  xyz_out: n x 3. */
int vg_deskew_points(vg_ctx* ctx, const double* xyz, const double* stamps, int64_t n,
                     const double* node_t, const double* quats, const double* trans, int64_t K,
                     double* xyz_out);

/* ---- clouds (Frame: preprocess.py:46-60) ----------------------------------------------- */
/* xyz: n x 3; cov: n x 3 x 3 or NULL.  Points exactly representable in fp32 take the fast
 * fast path: 64 B/point SoA in HBM (float4 xyz + the covariance as three fp64 double2 rows);
 * any other input also keeps an fp64 xyz copy so voxel keys stay exact. */
int vg_cloud_create(vg_ctx* ctx, const double* xyz, const double* cov, int64_t n,
                    vg_cloud** out);
int vg_cloud_info(const vg_cloud* cloud, int64_t* n, int32_t* has_cov, int32_t* exact_fp32);
int vg_cloud_destroy(vg_cloud* cloud);

/* ---- Gaussian voxel maps (GaussianVoxelMap: registration.py:29-71) --------------------- */
/* replaces build_voxelmap (registration.py:74-98); exported arrays are bit-identical */
int vg_map_build(vg_ctx* ctx, const vg_cloud* cloud, double resolution, vg_map** out);
/* adopt reference arrays (GaussianVoxelMap.__init__, registration.py:36-42); row = index */
int vg_map_from_arrays(vg_ctx* ctx, double resolution, const int64_t* keys,
                       const double* means, const double* covs, const int64_t* counts,
                       int64_t m, vg_map** out);
int vg_map_info(const vg_map* map, int64_t* m, double* resolution, int64_t* table_capacity);
/* any output pointer may be NULL */
int vg_map_export(vg_ctx* ctx, const vg_map* map, int64_t* keys, double* means, double* covs,
                  int64_t* counts);
int vg_map_destroy(vg_map* map);

/* ---- correspondence lookup ------------------------------------------------------------- */
/* replaces GaussianVoxelMap.lookup (registration.py:47-55): row per point or -1 */
int vg_map_lookup(vg_ctx* ctx, const vg_map* map, const double* xyz, int64_t n,
                  int64_t* rows_out, int64_t* hits_out);
/* transform + lookup of a device cloud: overlap_rate (registration.py:168-173) and the
 * hit count of _try_binary_factor (odometry.py:335-346); rows_out may be NULL */
int vg_cloud_lookup(vg_ctx* ctx, const vg_cloud* cloud, const vg_map* map, const double T[12],
                    int64_t* rows_out, int64_t* hits_out);

/* ---- per-point terms ------------------------------------------------------------------- */
/* replaces match_terms (registration.py:146-157).  Per source point (n rows, miss rows are
 * zero): rows (n), moved (n x 3), d (n x 3), weight (n x 3 x 3), wd (n x 3).  The caller
 * compacts by rows >= 0 to obtain MatchTerms.  cost/inliers are the fixed-order sums. */
int vg_match_terms(vg_ctx* ctx, const vg_cloud* cloud, const vg_map* map, const double T[12],
                   int64_t* rows, double* moved, double* d, double* weight, double* wd,
                   double* cost, int64_t* inliers);

/* replaces linearize_from_terms (registration.py:207-248) for a MatchTerms that carries the
 * per-point terms but not the voxel map (e.g. one built by the reference's own match_terms):
 * points = the hit source points (n x 3), weight (n x 3 x 3), wd (n x 3), T = T_ij; cost and
 * inliers as in the terms.  out: one VG_MODE_LINEARIZE record (92 doubles).  Returns
 * VG_ERR_DEGENERATE when inliers < min_inliers. */
int vg_linearize_terms(vg_ctx* ctx, const double T[12], const double* points,
                       const double* weight, const double* wd, int64_t n, double cost,
                       int64_t inliers, int32_t flags, int32_t min_inliers, double* out);

/* ---- batched linearization (the hot path) ---------------------------------------------- */
/* A batch is the set of MatchingCostFactors of one graph (factor_graph.py:209-308); it is
 * flattened once into (factor, chunk) work items resident in HBM. */
int vg_batch_create(vg_ctx* ctx, const vg_factor_spec* specs, int64_t num_factors,
                    vg_batch** out);
int vg_batch_info(const vg_batch* batch, int64_t* num_factors, int64_t* num_items,
                  int64_t* num_points);
int vg_batch_destroy(vg_batch* batch);

/* explicit transforms: T_ij = T_j^-1 T_i per factor (registration.py:264), F x 12 host
 * doubles.  out: F x record(mode) host doubles.  One call = match_terms +
 * linearize_from_terms (registration.py:146-157,207-248) for every factor. */
int vg_batch_linearize(vg_batch* batch, const double* T_host, int mode, double* out_host);

/* the same with the compact fp32 record (VG_REC_LINEARIZE_F32 words per factor; mode must be
 * VG_MODE_LINEARIZE): half the device->host bytes of the fp64 records */
int vg_batch_linearize_f32(vg_batch* batch, const double* T_host, int mode, float* out_host);

/* pose-table mode: poses V x 8 (quat xyzw, t, pad).  T_ij is composed on the device from
 * var_source / var_target exactly as pose_compose(pose_inverse(t_j), t_i). */
int vg_batch_linearize_poses(vg_batch* batch, const double* poses_host, int64_t num_poses,
                             int mode, double* out_host);

/* pose-table mode with the compact fp32 record (VG_REC_LINEARIZE_F32 words per factor) */
int vg_batch_linearize_poses_f32(vg_batch* batch, const double* poses_host, int64_t num_poses,
                                 int mode, float* out_host);

/* pinned (page-locked) host memory for outputs: device->host copies into it overlap the staged
 * computation, copies into pageable memory do not */
int vg_host_alloc(size_t bytes, void** out);
int vg_host_free(void* ptr);

/* correspondence rows of every factor at the pose table (GaussianVoxelMap.lookup of the moved
 * source points, registration.py:47-55,149): rows_out holds sum(n_f) int64 in factor (spec)
 * order, factor f's n_f points contiguous, the reference row of each hit or -1; inliers_out
 * (F) the hit count per factor (MatchTerms.inliers, :157).  Runs K-compose and the very K4a
 * launch the linearization runs, then scatters its compacted (point, record) hit lists: the
 * correspondences K4b consumes, exported for bit-exact checking. */
int vg_batch_lookup_rows(vg_batch* batch, const double* poses_host, int64_t num_poses,
                         int64_t* rows_out, int64_t* inliers_out);

/* device-resident variant: all pointers are device pointers on ctx's device; no host sync.
 * poses_dev may be NULL to reuse the poses of the previous call. */
int vg_batch_linearize_poses_device(vg_batch* batch, const double* poses_dev,
                                    int64_t num_poses, int mode, double* out_dev);
/* the three stages of vg_batch_linearize_poses_device, exposed separately so a caller can
 * time each kernel with events on the same stream: K-compose (T_ij from the pose table),
 * K4 (fused per-point accumulate into per-item partials), K5 (fixed-order finalize). */
int vg_batch_compose_device(vg_batch* batch, const double* poses_dev, int64_t num_poses);
int vg_batch_accumulate_device(vg_batch* batch, int mode);
int vg_batch_finalize_device(vg_batch* batch, int mode, double* out_dev);
/* capture compose + accumulate + finalize into a CUDA graph and replay it */
int vg_batch_graph_capture(vg_batch* batch, const double* poses_dev, int64_t num_poses,
                           int mode, double* out_dev);
int vg_batch_graph_launch(vg_batch* batch);
/* capture one rank's whole normal-equation step — K-compose, K4, K5 into records_dev, an
 * optional zeroing of out_dev, K6 into out_dev (the set-up layout) — as the batch's graph
 * (vg_batch_graph_launch replays it): the multi-GPU step between the pose broadcast and the
 * reduction, one launch instead of six */
int vg_batch_graph_capture_assemble(vg_batch* batch, const double* poses_dev, int64_t num_poses,
                                    double* records_dev, double* out_dev, int32_t zero_out);

/* ---- normal equations (FactorGraph._assemble_dense, factor_graph.py:522-536) ------------
 * Sums every factor's blocks into the block-sparse system the LM solves,
 * on the device and in a fixed order (factor order per block), so only the system crosses
 * PCIe.  Variables are pose-table rows 0 .. num_vars-1; rows >= num_vars are constants (the
 * fixed targets of unary factors), whose blocks are dropped as the reference's unary factors
 * do (factor_graph.py:296-297).  Factors below their min_inliers contribute nothing
 * (:282-291).  Output (doubles): [0] cost, [1] factors contributing, then
 *   diag  num_vars x 21  upper triangle (row-major) of each variable's 6x6 H block,
 *   grad  num_vars x 6   g,
 *   pairs P x 36          H block (a, b), row-major, for each variable pair a < b
 * with the pair list from vg_batch_assemble_pairs().  6-dof blocks: a caller with 15-dof
 * frame-state keys embeds them top-left (factor_graph.py:292-308). */
int vg_batch_assemble_setup(vg_batch* batch, int64_t num_vars, int64_t* num_pairs,
                            int64_t* out_doubles);
/* same with a caller-given pair list (sorted, unique, a < b): every rank of a sharded graph
 * passes the global list, so the per-rank systems share one layout and one sum-reduction
 * combines them.  Pairs of this batch missing from the list: VG_ERR_INVALID. */
int vg_batch_assemble_setup_pairs(vg_batch* batch, int64_t num_vars, const int32_t* pairs,
                                  int64_t num_pairs, int64_t* out_doubles);
/* the batch's own pair list, each block written at out_index[p] of an output layout with
 * out_pairs pair slots (increasing): a rank of a pair-disjoint shard writes its blocks
 * straight into the global layout (slots of other ranks' pairs stay untouched, i.e. zero in a
 * zeroed buffer), so one sum-reduction yields the global system */
int vg_batch_assemble_setup_mapped(vg_batch* batch, int64_t num_vars, const int32_t* pairs,
                                   int64_t num_pairs, const int32_t* out_index,
                                   int64_t out_pairs, int64_t* out_doubles);
int vg_batch_assemble_pairs(const vg_batch* batch, int32_t* pairs_out /* P x 2 */);
int vg_batch_assemble_poses(vg_batch* batch, const double* poses_host, int64_t num_poses,
                            double* out_host);
int vg_batch_assemble_poses_device(vg_batch* batch, const double* poses_dev,
                                   int64_t num_poses, double* out_dev);
/* K6 alone, over records the last vg_batch_finalize_device (VG_MODE_LINEARIZE) wrote:
 * lets a caller time K-compose / K4 / K5 separately and still assemble (bench.py, N > 1) */
int vg_batch_assemble_records_device(vg_batch* batch, const double* records_dev,
                                     double* out_dev);

/* ---- damped normal-equation solve ------------------------------------
 * Replaces the LM's linear solve, factor_graph.py:565-576 — `cho_factor(h + diag(lam *
 * diag(h)))` for dim <= dense_threshold, `splu(csc(h + diag(lam * diag(h))))` above — and the
 * factorizations of marginal_covariance (:707-722).  H (dim x dim, dense fp64) and g stay on
 * the device: the batch's block-sparse normal equations (K6) are scattered into H there, the
 * host adds only the few non-matching factors' blocks (priors, IMU), and each damping attempt
 * copies 8 * dim bytes of solution back instead of 8 * dim^2 bytes of H. */
typedef struct vg_solver vg_solver;
#define VG_SOLVE_CHOLESKY 0    /* cho_factor semantics: not positive definite -> info > 0 */
#define VG_SOLVE_CHOLESKY_LU 1 /* splu semantics: Cholesky, else partial-pivot LU; info > 0
                                  only when the damped matrix is exactly singular */
int vg_solver_create(vg_ctx* ctx, int64_t dim, vg_solver** out);
int vg_solver_destroy(vg_solver* solver);
/* H := 0, g := 0, cost := 0 */
int vg_solver_reset(vg_solver* solver);
/* add the batch's normal equations at the pose table (K-compose .. K6, vg_batch_assemble_setup
 * first): variable v's 6x6 block at tangent offset offsets[v] (factor_graph.py:292-308 puts
 * the pose block top-left of a 15-dof frame state); *cost_out = the batch's gated cost sum */
int vg_solver_add_batch(vg_solver* solver, vg_batch* batch, const double* poses_host,
                        int64_t num_poses, const int64_t* offsets, double* cost_out);
/* add host blocks (the reference's per-factor scatter of other factors, :529-535): block k is
 * desc[4k .. 4k+3] = (row0, col0, rows, cols), its values row-major at consecutive positions
 * of `values`; blocks must not overlap each other.  g_host (dim) is added when non-null. */
int vg_solver_add_blocks(vg_solver* solver, int64_t num_blocks, const int64_t* desc,
                         const double* values, const double* g_host);
/* factor A = H + lam * diag(H) + jitter * I (method VG_SOLVE_*); *info = 0 on success, else
 * the failing minor (Cholesky) / pivot (LU) — the reference's LinAlgError / RuntimeError */
int vg_solver_factor(vg_solver* solver, double lam, double jitter, int32_t method,
                     int64_t* info);
/* solve A X = B with the last factorization: B = rhs_host (dim x nrhs, column-major), or -g
 * when rhs_host is NULL (nrhs 1); X to x_host (dim x nrhs, column-major) */
int vg_solver_solve(vg_solver* solver, const double* rhs_host, int64_t nrhs, double* x_host);
/* copy H (dim x dim, symmetric), g (dim) and the accumulated cost to the host; any may be NULL */
int vg_solver_export(vg_solver* solver, double* h_host, double* g_host, double* cost_out);
/* diag(H) (dim) to the host: the jitter scale of marginal_covariance (:716-717) */
int vg_solver_diagonal(vg_solver* solver, double* diag_host);

/* ---- preprocessing (preprocess.py:122-164) --------------------------------------------- */
/* replaces knn_search (preprocess.py:122-139): exact k nearest (self included), ordered by
 * (squared distance, index).  Returns VG_ERR_TOO_SPARSE when n < k. */
int vg_knn(vg_ctx* ctx, const vg_cloud* cloud, int32_t k, int64_t* neighbors_out);
/* replaces estimate_covariances (preprocess.py:142-164): plane-regularised covariances */
int vg_covariances(vg_ctx* ctx, const vg_cloud* cloud, const int64_t* neighbors, int32_t k,
                   double plane_eps, double* covs_out, uint8_t* degenerate_out);
/* fused kNN + covariance on a device cloud; results stay on the device and are attached
 * to the cloud (so vg_map_build / linearization use them without a host round trip);
 * neighbors_out / covs_out / degenerate_out may be NULL. */
int vg_cloud_estimate_covariances(vg_ctx* ctx, vg_cloud* cloud, int32_t k, double plane_eps,
                                  int64_t* neighbors_out, double* covs_out,
                                  uint8_t* degenerate_out);

#ifdef __cplusplus
}
#endif
#endif /* VGICP_H_ */
