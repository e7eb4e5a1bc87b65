// common.cuh — device data layouts and helpers shared by every libvgicp kernel.
//
// HBM layouts:
//   cloud  : SoA, 64 B/point: a[i] = (x, y, z) fp32, covariance as three fp64 double2 arrays
//            + optional fp64 xyz (n x 3) when the points are not exactly fp32 (keys stay exact)
//   map    : bucketized open-addressing hash: 32-bit cell-local keys in 32 B buckets of 8
//            (load <= 0.25, ~16 B/cell: the probe arrays of all maps stay L2-resident) with
//            128 B fp64 records parallel to the slots; maps that do not fit the local frame
//            use int64 keys (64 B buckets) + a row array and row-indexed records.
//   work   : (factor, chunk) items, one warp per item; fp64 partials, fixed-order reduce.
#pragma once
#include <cstdio>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace vg {

// Device-side bounds / invariant checks, compiled in by the checked build
// (tools/build_variant.sh checked "-DVG_CHECKS=1"): the memory-safety net used in place of
// compute-sanitizer, which is closed on this GPU pool.  A failed check prints and traps (the
// launch fails with cudaErrorLaunchFailure / illegal instruction; the library returns
// VG_ERR_CUDA), so a test run against the checked library fails loudly on a violation.
#ifndef VG_CHECKS
#define VG_CHECKS 0
#endif
#if VG_CHECKS
#define VG_DEVICE_CHECK(cond, what)                                                       \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("VG_DEVICE_CHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__,   \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                                \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define VG_DEVICE_CHECK(cond, what) \
  do {                              \
  } while (0)
#endif

constexpr int kKeyOffset = 1 << 20;   // preprocess.py:21-22
constexpr int kWarpsPerBlock = 4;
constexpr int kPartialStride = 32;    // doubles per work-item partial (29 used)
constexpr int kMaxChunk = 1024;       // points per work item (whole factors at config 5:
                                      // 512 measured 2.7% slower per step, 256 11%)

// Voxel map on the device = open-addressing hash table (key -> reference row) + dense,
// row-indexed, line-aligned voxel records.  Each record is one 128 B cache line, so a
// cooperative gather touches one line per record.  Mean and covariance stay fp64: the fused
// covariance C' + R C R^T has condition ~1e3 for plane-like cells and the parity bar is per
// element (1e-4 rel) on H/b entries that cancel by up to ~1e5 — fp32 storage or fp32
// per-point math exceeds it (tests/kernel_model.py, tests/test_host_logic.py quantify it).
struct __align__(128) VoxelRec {
  double mean[3];   // voxel mean (registration.py:90-92)                 bytes  0..24
  double cov[6];    // covariance c00 c01 c02 c11 c12 c22 (:93-97)        bytes 24..72
  long long row;    // reference row (kmode 1 records sit at hash slots)  bytes 72..80
  double pad[6];
};
static_assert(sizeof(VoxelRec) == 128, "voxel record must be one 128 B line");
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
  const long long* keys;    // kmode 0: int64 packed keys, buckets of 8 (64 B)
  const int* rows;          // kmode 0: reference row per slot (parallel to keys)
  const unsigned* keys32;   // kmode 1: 32-bit cell-local keys, buckets of 8 (32 B)
  const VoxelRec* recs;     // kmode 1: parallel to keys32 (slot-indexed); kmode 0: row-indexed
  long long empty_key;      // kmode 0 empty marker (a value that is not a key of the map)
  double res;
  double inv_res;
  unsigned mask;        // buckets - 1
  int shift;            // kmode 0: 64 - log2(buckets); kmode 1: 32 - log2(buckets)
  int m;                // occupied cells
  int pow2;             // res is a power of two: x * (1/res) == x / res exactly
  int kmode;            // 1: every cell fits the 11/11/10-bit local frame below
  int bx, by, bz;       // local frame origin (min cell index)
  int ex, ey, ez;       // local frame extents (cells)
};

// Per-item header for the fused kernel (256 B, one coalesced load by 16 lanes): T_ij (written
// by K-compose every step) + the static views of the item's source cloud and target map.
struct __align__(16) ItemHdr {
  double T[12];
  const float4* a;
  const double* xyz64;
  const double2* c0;
  const double2* c1;
  const double2* c2;
  MapView mv;
  int factor;
  int begin;
  int end;
  int hoff;
};
static_assert(sizeof(ItemHdr) == 256, "item header must be 256 B");

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

// Per-item descriptor written by K4a for K4b: everything K4b's prologue needs in one
// broadcast load (instead of item -> factor -> cloud/map view dependency chains).
struct __align__(16) AccDesc {
  double T[12];            // T_ij of the item's factor
  const float4* a;         // source points (fp32)
  const double* xyz64;     // source points (fp64 path) or null
  const double2* c0;       // source covariance SoA
  const double2* c1;
  const double2* c2;
  const struct VoxelRec* recs;  // target map records
  int hoff;                // hit-list offset
  int n;                   // hits
  int pad[2];
};

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

// Bucketized open addressing: a key hashes to a bucket; insertion fills the home bucket
// before spilling to the next one, so a lookup resolves in its home bucket unless that
// bucket is full.  Two key encodings:
//   kmode 1 — 32-bit cell-local keys (lx | ly << 11 | lz << 22 relative to the map's min
//             cell); a bucket of 4 keys is 16 B = one 128-bit load.  Load <= 0.25, so ~0.4% of
//             buckets overflow into the next one.  The probe returns the slot; the record sits
//             at the same slot (it carries the row).
//   kmode 0 — the reference's packed int64 keys in 64 B buckets of 8 (two 256-bit loads,
//             load <= 0.25); the probe returns the slot, a parallel array gives the row and
//             records are row-indexed.
// The local key is built from decode(pack(floor)) — the reference's own key round trip —
// so aliasing of out-of-range indices behaves exactly as the reference's packed keys.
constexpr int kBucket = 8;    // kmode 0: int64 keys, 64 B buckets
constexpr int kBucket32 = 4;  // kmode 1: 32-bit keys, 16 B buckets (one 128-bit load)
constexpr unsigned kEmpty32 = 0xffffffffu;

// kmode 1 home bucket of a cell-local key (lx | ly << 11 | lz << 22).  VG_BLOCK_HASH: the
// 2x2x2 block of the cell picks a 128 B line (8 buckets), the cell's coordinate parities the
// bucket inside it, so probes of neighbouring cells share lines (needs >= 16 buckets)
#ifndef VG_BLOCK_HASH
#define VG_BLOCK_HASH 0
#endif
__host__ __device__ __forceinline__ unsigned bucket32(unsigned k32, int shift) {
#if VG_BLOCK_HASH
  const unsigned sub = (k32 & 1u) | ((k32 >> 10) & 2u) | ((k32 >> 20) & 4u);
  const unsigned blk = k32 & ~(1u | (1u << 11) | (1u << 22));
  return (((blk * 0x9E3779B9u) >> (shift + 3)) << 3) | sub;
#else
  return (k32 * 0x9E3779B9u) >> shift;
#endif
}

struct Query {
  long long key;   // packed reference key
  unsigned k32;    // local key (kmode 1)
  unsigned bucket;
  bool inside;     // kmode 1: cell lies in the map's local frame (else certainly a miss)
};
struct ProbeGroup {
  long long k[kBucket];  // kmode 0: 8 keys; kmode 1: k[0..3] hold 8 packed 32-bit keys
};

__device__ __forceinline__ void ld256(const void* p, long long& a, long long& b, long long& c,
                                      long long& d) {
  asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
               : "l"(p));
}

// `kmode` is mv.kmode, passed separately so callers specialised on a key encoding fold it
__device__ __forceinline__ Query make_query(const MapView& mv, double fx, double fy, double fz,
                                            int kmode) {
  Query q;
  q.key = pack_key(fx, fy, fz);
  if (kmode) {
    const long long dx = (q.key >> 42) - kKeyOffset;
    const long long dy = ((q.key >> 21) & ((1LL << 21) - 1)) - kKeyOffset;
    const long long dz = (q.key & ((1LL << 21) - 1)) - kKeyOffset;
    const unsigned long long lx = (unsigned long long)(dx - mv.bx);
    const unsigned long long ly = (unsigned long long)(dy - mv.by);
    const unsigned long long lz = (unsigned long long)(dz - mv.bz);
    q.inside = lx < (unsigned long long)mv.ex && ly < (unsigned long long)mv.ey &&
               lz < (unsigned long long)mv.ez;
    q.k32 = (unsigned)lx | ((unsigned)ly << 11) | ((unsigned)lz << 22);
    q.bucket = bucket32(q.k32, mv.shift);
  } else {
    q.inside = true;
    q.k32 = 0;
    q.bucket = slot_of(q.key, mv.shift);
  }
  return q;
}

// kmode 1 fast path: for |floor| < 2^20 the reference's pack/unpack round trip is the
// identity, so the local key comes straight from the floors; otherwise defer to make_query
// (which reproduces the reference's aliasing of out-of-range indices).
__device__ __forceinline__ Query make_query_local(const MapView& mv, double fx, double fy,
                                                  double fz) {
  if (fmax(fabs(fx), fmax(fabs(fy), fabs(fz))) < 1048576.0) {
    Query q;
    q.key = 0;
    const unsigned lx = (unsigned)(__double2int_rz(fx) - mv.bx);
    const unsigned ly = (unsigned)(__double2int_rz(fy) - mv.by);
    const unsigned lz = (unsigned)(__double2int_rz(fz) - mv.bz);
    q.inside = lx < (unsigned)mv.ex && ly < (unsigned)mv.ey && lz < (unsigned)mv.ez;
    q.k32 = lx | (ly << 11) | (lz << 22);
    q.bucket = bucket32(q.k32, mv.shift);
    return q;
  }
  return make_query(mv, fx, fy, fz, 1);
}

__device__ __forceinline__ ProbeGroup probe_load(const MapView& mv, unsigned bucket, int kmode) {
  ProbeGroup g;
  if (kmode) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(mv.keys32 + (size_t)bucket * kBucket32));
    g.k[0] = (long long)((unsigned long long)v.x | ((unsigned long long)v.y << 32));
    g.k[1] = (long long)((unsigned long long)v.z | ((unsigned long long)v.w << 32));
  } else {
    const long long* p = mv.keys + (size_t)bucket * kBucket;
    ld256(p, g.k[0], g.k[1], g.k[2], g.k[3]);
    ld256(p + 4, g.k[4], g.k[5], g.k[6], g.k[7]);
  }
  return g;
}

// 1 found (`slot` set), 0 missing, -1 next bucket
__device__ __forceinline__ int probe_scan(const MapView& mv, const ProbeGroup& g,
                                          unsigned bucket, const Query& q, int& slot,
                                          int kmode) {
  int found = -1;
  bool empty = false;
  if (kmode) {
#pragma unroll
    for (int j = kBucket32 - 1; j >= 0; --j) {
      const unsigned kj = (unsigned)((unsigned long long)g.k[j >> 1] >> (32 * (j & 1)));
      if (kj == q.k32) found = j;
      empty |= (kj == kEmpty32);
    }
  } else {
#pragma unroll
    for (int j = kBucket - 1; j >= 0; --j) {
      if (g.k[j] == q.key) found = j;
      empty |= (g.k[j] == mv.empty_key);
    }
  }
  if (found >= 0) {
    slot = (int)(bucket * (kmode ? kBucket32 : kBucket) + found);
    return 1;
  }
  return empty ? 0 : -1;
}

__device__ __forceinline__ unsigned next_bucket(unsigned b, const MapView& mv) {
  return (b + 1) & mv.mask;  // mask = #buckets - 1
}

// probe result (slot) -> index of the voxel record to gather
__device__ __forceinline__ int rec_index(const MapView& mv, int slot, int kmode) {
  return kmode ? slot : __ldg(mv.rows + slot);
}
// probe result (slot) -> reference row
__device__ __forceinline__ int slot_row(const MapView& mv, int slot, int kmode) {
  return kmode ? (int)__ldg(&mv.recs[slot].row) : __ldg(mv.rows + slot);
}

// full lookup: slot or -1
__device__ __forceinline__ int probe_query(const MapView& mv, const Query& q) {
  if (mv.m == 0 || !q.inside) return -1;
  unsigned b = q.bucket;
  for (unsigned probes = 0;; ++probes) {
    VG_DEVICE_CHECK(probes <= mv.mask, "probe_query: every bucket visited");
    const ProbeGroup g = probe_load(mv, b, mv.kmode);
    int slot = -1;
    const int r = probe_scan(mv, g, b, q, slot, mv.kmode);
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
