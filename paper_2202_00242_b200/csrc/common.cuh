// common.cuh — device data layouts and helpers shared by every libvgicp kernel.
//
// HBM layouts:
//   cloud  : SoA, 64 B/point: a[i] = (x, y, z) fp32, covariance as three fp64 double2 arrays
//            + optional fp64 xyz (n x 3) when the points are not exactly fp32 (keys stay exact)
//   map    : bucketized open-addressing hash table (load factor <= 0.25): dense int64 key
//            array in 64 B buckets of 8 slots + parallel 96 B records (row, fp64 Gaussian).
//   work   : (factor, chunk) items, one warp per item; fp64 partials, fixed-order reduce.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace vg {

constexpr int kKeyOffset = 1 << 20;   // preprocess.py:21-22
constexpr int kWarpsPerBlock = 4;
constexpr int kPartialStride = 32;    // doubles per work-item partial (29 used)
constexpr int kMaxChunk = 512;        // points per work item => <= 16 points per lane

// Voxel map on the device = open-addressing hash table in two parallel arrays indexed by
// slot: a dense int64 key array (probed one 64 B bucket at a time) and 96 B records carrying the
// reference row and the voxel Gaussian in fp64.  Empty slots hold `empty_key`, a value that is
// not a key of this map.  Mean and covariance stay fp64: the fused covariance C' + R C R^T
// has condition ~1e3 for plane-like cells and the parity bar is per element (1e-4 rel) on
// H/b entries that cancel by up to ~1e5 — fp32 storage or fp32 per-point math exceeds it
// (tests/kernel_model.py, tests/test_host_logic.py quantify it).
struct __align__(32) VoxelRec {
  double mean[3];   // voxel mean (registration.py:90-92)          offsets  0..24
  double cov[6];    // covariance c00 c01 c02 c11 c12 c22 (:93-97)  offsets 24..72
  int row;          // rank of the key in ascending order == reference row index
  int pad0;
  double pad1[2];
};
static_assert(sizeof(VoxelRec) == 96, "voxel record must be 96 B");
static_assert(offsetof(VoxelRec, mean) % 16 == 0 && offsetof(VoxelRec, cov) % 16 == 8,
              "double2 loads at mean[0], mean[2], cov[1], cov[3] must be 16 B aligned");

struct CloudView {
  const float4* a;      // n: x, y, z (fp32), pad
  const double2* c0;    // n: c00 c01   (null when the cloud has no covariances)
  const double2* c1;    // n: c02 c11
  const double2* c2;    // n: c12 c22
  const double* xyz64;  // n*3 or null (exact fp32 fast path)
  long long n;
};

struct MapView {
  const long long* keys;    // capacity (multiple of 4), 32 B aligned
  const VoxelRec* recs;     // capacity, parallel to keys
  long long empty_key;
  double res;
  double inv_res;
  unsigned mask;        // buckets - 1
  int shift;            // 64 - log2(buckets)
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
  int begin;  // point range [begin, end) of the factor's source cloud
  int end;
  int hoff;   // offset of this item's region in the batch hit list (even, 16 B aligned)
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

// Bucketized open addressing: a key hashes to a 64 B bucket of 8 slots (two 256-bit loads);
// insertion fills the home bucket before spilling to the next one, so a lookup resolves in
// its home bucket unless that bucket is full (load factor <= 0.25: ~0.1% of lookups).
// Returns the slot index or -1.  Lookups of any key (including empty_key) terminate.
constexpr int kBucket = 8;
struct ProbeGroup {
  long long k[kBucket];
};
__device__ __forceinline__ void ld256(const void* p, long long& a, long long& b, long long& c,
                                      long long& d) {
  asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
               : "l"(p));
}
__device__ __forceinline__ ProbeGroup probe_load(const MapView& mv, unsigned bucket) {
  ProbeGroup g;
  const long long* p = mv.keys + (size_t)bucket * kBucket;
  ld256(p, g.k[0], g.k[1], g.k[2], g.k[3]);
  ld256(p + 4, g.k[4], g.k[5], g.k[6], g.k[7]);
  return g;
}
// 1 found (slot set), 0 missing, -1 continue with the next bucket
__device__ __forceinline__ int probe_scan(const MapView& mv, const ProbeGroup& g,
                                          unsigned bucket, long long key, int& slot) {
  int found = -1;
  bool empty = false;
#pragma unroll
  for (int j = kBucket - 1; j >= 0; --j) {
    if (g.k[j] == key) found = j;
    empty |= (g.k[j] == mv.empty_key);
  }
  if (found >= 0) {
    slot = (int)(bucket * kBucket + found);
    return 1;
  }
  return empty ? 0 : -1;
}
__device__ __forceinline__ unsigned bucket_of(long long key, const MapView& mv) {
  return slot_of(key, mv.shift);  // shift = 64 - log2(#buckets)
}
__device__ __forceinline__ unsigned next_bucket(unsigned b, const MapView& mv) {
  return (b + 1) & mv.mask;  // mask = #buckets - 1
}
__device__ __forceinline__ int probe(const MapView& mv, long long key) {
  if (mv.m == 0) return -1;
  unsigned b = bucket_of(key, mv);
  for (;;) {
    const ProbeGroup g = probe_load(mv, b);
    int slot = -1;
    const int r = probe_scan(mv, g, b, key, slot);
    if (r >= 0) return r ? slot : -1;
    b = next_bucket(b, mv);
  }
}

// Reference-exact fp64 helpers (no FMA contraction), used where numpy's rounding must be
// reproduced bit for bit (voxel map statistics, registration.py:87-97).
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

// 1/a: hardware approximation + two Newton steps (error squares each step), no slow path
__device__ __forceinline__ double rcp64(double a) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  double e = fma(-a, r, 1.0);
  r = fma(r, e, r);
  e = fma(-a, r, 1.0);
  return fma(r, e, r);
}

// 32 values reduced across 32 lanes in 31 shuffle steps; lane L returns the sum of value L.
__device__ __forceinline__ double warp_transpose_reduce32(double (&v)[32], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const double send = up ? v[i] : v[i + s];
      const double keep = up ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

}  // namespace vg
