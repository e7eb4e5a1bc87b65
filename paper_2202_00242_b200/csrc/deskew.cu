// deskew.cu — per-point half of deskew (preprocess.py:181-232) on the device.
//
// The host integrates the IMU across the scan (integration_nodes + propagate_state, as the
// reference does: preprocess.py:199-216) into a short node trajectory (node stamps, xyzw
// quaternions and translations relative to the scan-start pose).  Every point then finds its
// segment (searchsorted side="right", :218-219), interpolates the pose (shortest-arc slerp of
// the node quaternions, linear translation, :220-224; _slerp_batch :167-178) and is moved into
// the scan-start frame (p' = p + 2w(u x p) + 2u x (u x p) + t, :226-231).  One thread per
// point; the node table is staged in shared memory when it fits.  Arithmetic follows NumPy's
// operation order without FMA contraction; acos/sin/sqrt are CUDA's (<= 2 ulp), so results
// agree with the reference to ~1e-15 relative (tests allow 1e-9 m).
#include "common.cuh"
#include "internal.h"

namespace vg {

constexpr int kDeskewSmemNodes = 2048;

__device__ __forceinline__ void cross_rn(const double a[3], const double b[3], double o[3]) {
  o[0] = sub_rn(mul_rn(a[1], b[2]), mul_rn(a[2], b[1]));
  o[1] = sub_rn(mul_rn(a[2], b[0]), mul_rn(a[0], b[2]));
  o[2] = sub_rn(mul_rn(a[0], b[1]), mul_rn(a[1], b[0]));
}

__global__ void k_deskew(const double* __restrict__ xyz, const double* __restrict__ stamps,
                         long long n, const double* __restrict__ node_t,
                         const double* __restrict__ quats, const double* __restrict__ trans,
                         int K, double* __restrict__ out) {
  __shared__ double s_t[kDeskewSmemNodes];
  const bool staged = K <= kDeskewSmemNodes;
  if (staged)
    for (int i = threadIdx.x; i < K; i += blockDim.x) s_t[i] = node_t[i];
  __syncthreads();
  const double* nt = staged ? s_t : node_t;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
       p += (long long)gridDim.x * blockDim.x) {
    const double ts = stamps[p];
    // searchsorted(node_t, ts, side="right") - 1, clipped to [0, K-2]
    int lo = 0, hi = K;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (nt[mid] <= ts) lo = mid + 1;
      else hi = mid;
    }
    int seg = lo - 1;
    seg = seg < 0 ? 0 : (seg > K - 2 ? K - 2 : seg);
    const double t0 = nt[seg], t1 = nt[seg + 1];
    const double span = sub_rn(t1, t0);
    double alpha = span > 0.0 ? __ddiv_rn(sub_rn(ts, t0), span) : 0.0;
    alpha = alpha < 0.0 ? 0.0 : (alpha > 1.0 ? 1.0 : alpha);
    // _slerp_batch (preprocess.py:167-178)
    double qa[4], qb[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      qa[j] = quats[4 * seg + j];
      qb[j] = quats[4 * (seg + 1) + j];
    }
    double dot = add_rn(add_rn(add_rn(mul_rn(qa[0], qb[0]), mul_rn(qa[1], qb[1])),
                               mul_rn(qa[2], qb[2])), mul_rn(qa[3], qb[3]));
    if (dot < 0.0)
#pragma unroll
      for (int j = 0; j < 4; ++j) qb[j] = -qb[j];
    dot = fabs(dot);
    const double theta = acos(fmin(fmax(dot, -1.0), 1.0));
    const double st = sin(theta);
    const bool near = dot > 1.0 - 1e-12;
    const double den = st == 0.0 ? 1.0 : st;
    const double oma = sub_rn(1.0, alpha);
    const double w0 = near ? oma : __ddiv_rn(sin(mul_rn(oma, theta)), den);
    const double w1 = near ? alpha : __ddiv_rn(sin(mul_rn(alpha, theta)), den);
    double q[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) q[j] = add_rn(mul_rn(w0, qa[j]), mul_rn(w1, qb[j]));
    const double nrm = __dsqrt_rn(add_rn(add_rn(add_rn(add_rn(0.0, mul_rn(q[0], q[0])),
                                                       mul_rn(q[1], q[1])),
                                                mul_rn(q[2], q[2])), mul_rn(q[3], q[3])));
#pragma unroll
    for (int j = 0; j < 4; ++j) q[j] = __ddiv_rn(q[j], nrm);
    // t = (1 - alpha) trans[seg] + alpha trans[seg + 1]
    double tr[3];
#pragma unroll
    for (int j = 0; j < 3; ++j)
      tr[j] = add_rn(mul_rn(oma, trans[3 * seg + j]), mul_rn(alpha, trans[3 * (seg + 1) + j]));
    // p' = p + w c1 + u x c1 + t, c1 = 2 (u x p)
    const double pt[3] = {xyz[3 * p], xyz[3 * p + 1], xyz[3 * p + 2]};
    double c1[3], c2[3];
    cross_rn(q, pt, c1);
#pragma unroll
    for (int j = 0; j < 3; ++j) c1[j] = mul_rn(2.0, c1[j]);
    cross_rn(q, c1, c2);
#pragma unroll
    for (int j = 0; j < 3; ++j)
      out[3 * p + j] = add_rn(add_rn(add_rn(pt[j], mul_rn(q[3], c1[j])), c2[j]), tr[j]);
  }
}

}  // namespace vg

using namespace vg;

int launch_deskew(vg_ctx* ctx, const double* xyz, const double* stamps, long long n,
                  const double* node_t, const double* quats, const double* trans, int K,
                  double* xyz_out) {
  if (n == 0) return 0;
  cudaStream_t st = ctx->stream;
  double *dx = nullptr, *ds = nullptr, *dn = nullptr, *dq = nullptr, *dt = nullptr,
         *dout = nullptr;
  DeviceTemps temps(st);
  VG_CUDA(temps.alloc(&dx, 3 * (size_t)n));
  VG_CUDA(temps.alloc(&ds, (size_t)n));
  VG_CUDA(temps.alloc(&dn, (size_t)K));
  VG_CUDA(temps.alloc(&dq, 4 * (size_t)K));
  VG_CUDA(temps.alloc(&dt, 3 * (size_t)K));
  VG_CUDA(temps.alloc(&dout, 3 * (size_t)n));
  VG_CUDA(cudaMemcpyAsync(dx, xyz, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
  VG_CUDA(cudaMemcpyAsync(ds, stamps, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  VG_CUDA(cudaMemcpyAsync(dn, node_t, sizeof(double) * K, cudaMemcpyHostToDevice, st));
  VG_CUDA(cudaMemcpyAsync(dq, quats, sizeof(double) * 4 * K, cudaMemcpyHostToDevice, st));
  VG_CUDA(cudaMemcpyAsync(dt, trans, sizeof(double) * 3 * K, cudaMemcpyHostToDevice, st));
  const long long blocks = (n + 255) / 256;
  k_deskew<<<(unsigned)(blocks < 148 * 8 ? blocks : 148 * 8), 256, 0, st>>>(dx, ds, n, dn, dq,
                                                                           dt, K, dout);
  ctx->launches++;
  VG_CUDA(cudaGetLastError());
  VG_CUDA(cudaMemcpyAsync(xyz_out, dout, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, st));
  VG_CUDA(cudaStreamSynchronize(st));
  return 0;
}
