// common.cuh — device data layouts and helpers shared by every libvgicp kernel.
//
// HBM layouts:
//   cloud  : SoA, 64 B/point: a[i] = (x, y, z) fp32, covariance as three fp64 double2 arrays
//            + optional fp64 xyz (n x 3) when the points are not exactly fp32 (keys stay exact)
//   map    : open-addressing hash table of 16 B slots (key -> row, load factor <= 0.5) and a
//            row-indexed array of 64 B voxel records (cell-local fp32 mean + fp64 covariance).
//   work   : (factor, chunk) items, one warp per item; fp64 partials, fixed-order reduce.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace vg {

constexpr int kKeyOffset = 1 << 20;   // preprocess.py:21-22
constexpr int kWarpsPerBlock = 8;
constexpr int kPartialStride = 32;    // doubles per work-item partial (29 used)
constexpr int kMaxChunk = 512;        // points per work item => <= 16 points per lane

// 16-byte hash slot: packed key -> reference row.  row < 0 marks an empty slot (any int64
// can be a key, so emptiness is not encoded in the key).
struct __align__(16) Slot {
  long long key;  // packed voxel key (registration.py:36-42 `keys`)
  int row;        // rank of the key in ascending order == reference row index
  int pad;
};
static_assert(sizeof(Slot) == 16, "slot must be 16 B");

// 64-byte voxel record, gathered by row.  Covariances stay fp64: a cell's fused covariance
// C' + R C R^T has condition ~1e3 for plane-like neighbourhoods, and fp32 storage alone
// perturbs W = F^-1 by ~3e-5 relative — enough to break the per-element 1e-4 parity bar on
// cancelling H entries (tests/kernel_model.py quantifies it).
struct __align__(64) VoxelRec {
  float4 mean;    // voxel mean relative to the cell centre (x, y, z), pad
  double2 c0;     // c00 c01
  double2 c1;     // c02 c11
  double2 c2;     // c12 c22
};
static_assert(sizeof(VoxelRec) == 64, "voxel record must be 64 B");

struct CloudView {
  const float4* a;      // n: x, y, z (fp32), pad
  const double2* c0;    // n: c00 c01   (null when the cloud has no covariances)
  const double2* c1;    // n: c02 c11
  const double2* c2;    // n: c12 c22
  const double* xyz64;  // n*3 or null (exact fp32 fast path)
  long long n;
};

struct MapView {
  const Slot* table;
  const VoxelRec* vox;
  double res;
  double inv_res;
  unsigned mask;        // capacity - 1
  int shift;            // 64 - log2(capacity)
  int m;                // occupied cells
  int pad;
};

// Per-factor record resident in HBM (128 B).  T = T_ij (R row-major, t), fp64.
struct __align__(16) FactorDev {
  double T[12];
  int cloud;
  int map;
  int flags;
  int min_inliers;
  int item_begin;
  int item_count;
  int var_source;
  int var_target;
};
static_assert(sizeof(FactorDev) == 128, "factor record must be 128 B");

struct __align__(16) ItemDev {
  int factor;
  int begin;
  int end;
  int pad;
};

// ---------------------------------------------------------------------------------------
// voxel keys: floor(p / res) (IEEE true division, as numpy) + 2^20, 21 bits per axis
// (preprocess.py:68-70).  x * (1/res) is used unless the quotient is within 1e-12 of an
// integer, where the correctly rounded quotient decides — so the floor is bit-identical to
// numpy's floor(p / res) for every input.
__device__ __forceinline__ double floor_div(double x, double res, double inv_res) {
  double q = x * inv_res;
  double f = floor(q);
  double frac = q - f;
  double tol = 1e-12 * fabs(q);
  if (frac <= tol || 1.0 - frac <= tol) f = floor(__ddiv_rn(x, res));
  return f;
}

__device__ __forceinline__ long long pack_key(double fx, double fy, double fz) {
  unsigned long long ux = (unsigned long long)((long long)fx + kKeyOffset);
  unsigned long long uy = (unsigned long long)((long long)fy + kKeyOffset);
  unsigned long long uz = (unsigned long long)((long long)fz + kKeyOffset);
  return (long long)((ux << 42) | (uy << 21) | uz);
}

__device__ __forceinline__ unsigned slot_of(long long key, int shift) {
  return (unsigned)(((unsigned long long)key * 0x9E3779B97F4A7C15ull) >> shift);
}

// Probe for `key`; returns the reference row or -1 (one 16 B load per probe).  Average probe length <= 1.5 on hits
// (load factor <= 0.5).
__device__ __forceinline__ int probe(const MapView& mv, long long key) {
  if (mv.m == 0) return -1;
  unsigned h = slot_of(key, mv.shift);
  for (;;) {
    const int4 s = __ldg(reinterpret_cast<const int4*>(mv.table + h));
    const long long k = ((long long)(unsigned)s.y << 32) | (unsigned)s.x;
    if (s.z < 0) return -1;
    if (k == key) return s.z;
    h = (h + 1) & mv.mask;
  }
}

// Reference-exact fp64 helpers (no FMA contraction), used where numpy's rounding must be
// reproduced bit for bit (voxel map statistics, registration.py:87-97).
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

}  // namespace vg
