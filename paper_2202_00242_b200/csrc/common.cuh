// common.cuh — device data layouts and helpers shared by every libvgicp kernel.
//
// HBM layouts:
//   cloud  : SoA, 64 B/point: a[i] = (x, y, z) fp32, covariance as three fp64 double2 arrays
//            + optional fp64 xyz (n x 3) when the points are not exactly fp32 (keys stay exact)
//   map    : open-addressing hash table (load factor <= 0.5) of 96 B slots carrying the
//            voxel's key, reference row and fp64 Gaussian.
//   work   : (factor, chunk) items, one warp per item; fp64 partials, fixed-order reduce.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace vg {

constexpr int kKeyOffset = 1 << 20;   // preprocess.py:21-22
constexpr int kWarpsPerBlock = 4;
constexpr int kPartialStride = 32;    // doubles per work-item partial (29 used)
constexpr int kMaxChunk = 512;        // points per work item => <= 16 points per lane

// 96-byte inline hash slot: packed key, reference row and the voxel Gaussian in fp64.
// row < 0 marks an empty slot (any int64 can be a key).  A hit reads exactly the slot's
// three 32 B sectors with no dependent second gather.  Mean and covariance stay fp64: the
// fused covariance C' + R C R^T has condition ~1e3 for plane-like cells and the parity bar
// is per element (1e-4 rel) on H/b entries that cancel by up to ~1e5 — fp32 storage or fp32
// per-point math exceeds it (tests/kernel_model.py, tests/test_host_logic.py quantify it).
struct __align__(32) Slot {
  long long key;    // packed voxel key (registration.py:36-42 `keys`)
  int row;          // rank of the key in ascending order == reference row index
  int pad0;
  double mean[3];   // voxel mean (registration.py:90-92)
  double cov[6];    // voxel covariance c00 c01 c02 c11 c12 c22 (registration.py:93-97)
  double pad1;
};
static_assert(sizeof(Slot) == 96, "slot must be 96 B");

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
  double res;
  double inv_res;
  unsigned mask;        // capacity - 1
  int shift;            // 64 - log2(capacity)
  int m;                // occupied cells
  int pow2;             // res is a power of two: x * (1/res) == x / res exactly
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
__device__ __forceinline__ double floor_div(double x, double res, double inv_res, int pow2) {
  double q = x * inv_res;
  double f = floor(q);
  if (pow2) return f;
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

// Probe for `key`; returns the slot index or -1 (one 16 B header load per probe; average
// probe length <= 1.5 on hits at load factor <= 0.5).
__device__ __forceinline__ int probe(const MapView& mv, long long key) {
  if (mv.m == 0) return -1;
  unsigned h = slot_of(key, mv.shift);
  for (;;) {
    const int4 s = __ldg(reinterpret_cast<const int4*>(mv.table + h));
    const long long k = ((long long)(unsigned)s.y << 32) | (unsigned)s.x;
    if (s.z < 0) return -1;
    if (k == key) return (int)h;
    h = (h + 1) & mv.mask;
  }
}

// Reference-exact fp64 helpers (no FMA contraction), used where numpy's rounding must be
// reproduced bit for bit (voxel map statistics, registration.py:87-97).
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

}  // namespace vg
