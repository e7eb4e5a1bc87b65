// Microbenchmark: K4b per-hit fp64 math throughput with data already in shared memory
// (no global traffic).  Answers "is the math itself latency/occupancy bound at 12 warps/SM?"
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2202_00242_b200/csrc
//        -I../../include mathbench.cu -o mathbench
#include <cstdio>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace vg;

struct Stage {
  float4 pt[2][32];
  float4 cov[3][32];
  float4 rec[32][5];
};

template <int MODE>
__device__ __forceinline__ void hit_math(const Stage& st, int lane, const double (&R)[9],
                                         const double (&t)[3], double (&acc)[28]) {
  const float4 a = st.pt[0][lane];
  const double px = a.x, py = a.y, pz = a.z;
  const double2 s0 = *reinterpret_cast<const double2*>(&st.cov[0][lane]);
  const double2 s1 = *reinterpret_cast<const double2*>(&st.cov[1][lane]);
  const double2 s2 = *reinterpret_cast<const double2*>(&st.cov[2][lane]);
  const double2 m01 = *reinterpret_cast<const double2*>(&st.rec[lane][0]);
  const double2 m2c0 = *reinterpret_cast<const double2*>(&st.rec[lane][1]);
  const double2 c12 = *reinterpret_cast<const double2*>(&st.rec[lane][2]);
  const double2 c34 = *reinterpret_cast<const double2*>(&st.rec[lane][3]);
  const double v5 = reinterpret_cast<const double*>(&st.rec[lane][4])[0];
  const double x = fma(R[0], px, fma(R[1], py, R[2] * pz)) + t[0];
  const double y = fma(R[3], px, fma(R[4], py, R[5] * pz)) + t[1];
  const double z = fma(R[6], px, fma(R[7], py, R[8] * pz)) + t[2];
  const double d0 = m01.x - x, d1 = m01.y - y, d2 = m2c0.x - z;
  const double C00 = s0.x, C01 = s0.y, C02 = s1.x, C11 = s1.y, C12 = s2.x, C22 = s2.y;
  double A[9];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const double r0 = R[3 * q], r1 = R[3 * q + 1], r2 = R[3 * q + 2];
    A[3 * q + 0] = fma(r0, C00, fma(r1, C01, r2 * C02));
    A[3 * q + 1] = fma(r0, C01, fma(r1, C11, r2 * C12));
    A[3 * q + 2] = fma(r0, C02, fma(r1, C12, r2 * C22));
  }
  auto arT = [&](int a_, int c_) {
    return fma(A[3 * a_], R[3 * c_], fma(A[3 * a_ + 1], R[3 * c_ + 1], A[3 * a_ + 2] * R[3 * c_ + 2]));
  };
  const double fa = m2c0.y + arT(0, 0), fb = c12.x + arT(0, 1), fc = c12.y + arT(0, 2);
  const double fd = c34.x + arT(1, 1), fe = c34.y + arT(1, 2), ff = v5 + arT(2, 2);
  const double i00 = fma(fd, ff, -fe * fe), i01 = fma(fc, fe, -fb * ff),
               i02 = fma(fb, fe, -fc * fd), i11 = fma(fa, ff, -fc * fc),
               i12 = fma(fb, fc, -fa * fe), i22 = fma(fa, fd, -fb * fb);
  const double inv = rcp64(fma(fa, i00, fma(fb, i01, fc * i02)));
  const double W00 = i00 * inv, W01 = i01 * inv, W02 = i02 * inv, W11 = i11 * inv,
               W12 = i12 * inv, W22 = i22 * inv;
  const double wd0 = fma(W00, d0, fma(W01, d1, W02 * d2));
  const double wd1 = fma(W01, d0, fma(W11, d1, W12 * d2));
  const double wd2 = fma(W02, d0, fma(W12, d1, W22 * d2));
  acc[27] += fma(d0, wd0, fma(d1, wd1, d2 * wd2));
  if (MODE == 0) {
    const double vx = x - t[0], vy = y - t[1], vz = z - t[2];
    const double N00 = fma(-vz, W01, vy * W02), N01 = fma(-vz, W11, vy * W12), N02 = fma(-vz, W12, vy * W22);
    const double N10 = fma(vz, W00, -vx * W02), N11 = fma(vz, W01, -vx * W12), N12 = fma(vz, W02, -vx * W22);
    const double N20 = fma(-vy, W00, vx * W01), N21 = fma(-vy, W01, vx * W11), N22 = fma(-vy, W02, vx * W12);
    acc[0] += fma(-vz, N01, vy * N02); acc[1] += fma(vz, N00, -vx * N02); acc[2] += fma(-vy, N00, vx * N01);
    acc[3] += fma(vz, N10, -vx * N12); acc[4] += fma(-vy, N10, vx * N11); acc[5] += fma(-vy, N20, vx * N21);
    acc[6] += N00; acc[7] += N01; acc[8] += N02; acc[9] += N10; acc[10] += N11; acc[11] += N12;
    acc[12] += N20; acc[13] += N21; acc[14] += N22;
    acc[15] += W00; acc[16] += W01; acc[17] += W02; acc[18] += W11; acc[19] += W12; acc[20] += W22;
    acc[21] += fma(vy, wd2, -vz * wd1); acc[22] += fma(vz, wd0, -vx * wd2); acc[23] += fma(vx, wd1, -vy * wd0);
    acc[24] += wd0; acc[25] += wd1; acc[26] += wd2;
  }
}

template <int MODE, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) k_math(int rounds, double* out) {
  __shared__ Stage st[WARPS];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  Stage& s = st[wib];
  // plausible data: plane-like covariances, points ~10 m
  for (int u = 0; u < 2; ++u) s.pt[u][lane] = make_float4(10.f + lane * 0.1f, -3.f, 1.f, 0.f);
  double* c = reinterpret_cast<double*>(&s.cov[0][lane]);
  c[0] = 1.0; c[1] = 0.01;
  c = reinterpret_cast<double*>(&s.cov[1][lane]); c[0] = 0.02; c[1] = 1.0;
  c = reinterpret_cast<double*>(&s.cov[2][lane]); c[0] = 0.01; c[1] = 0.001;
  double* r = reinterpret_cast<double*>(&s.rec[lane][0]);
  r[0] = 10.1; r[1] = -2.9; r[2] = 1.05; r[3] = 0.5; r[4] = 0.01; r[5] = 0.02;
  r[6] = 0.6; r[7] = 0.01; r[8] = 0.003; r[9] = 0.0;
  __syncwarp();
  double R[9] = {0.99, -0.1, 0.0, 0.1, 0.99, 0.0, 0.0, 0.0, 1.0}, t[3] = {0.1, 0.2, 0.0};
  R[0] += 1e-9 * blockIdx.x;
  double acc[28];
#pragma unroll
  for (int k = 0; k < 28; ++k) acc[k] = 0.0;
  for (int i = 0; i < rounds; ++i) {
    hit_math<MODE>(s, (lane + i) & 31, R, t, acc);  // lane-rotating reads: no hoisting
    t[0] += 1e-12;
  }
  double sum = 0.0;
#pragma unroll
  for (int k = 0; k < 28; ++k) sum += acc[k];
  if (sum == 1234.5) out[0] = sum;
}

template <int MODE, int WARPS, int MINB>
float run(int blocks, int rounds) {
  double* out;
  cudaMalloc(&out, 8);
  k_math<MODE, WARPS, MINB><<<blocks, WARPS * 32>>>(rounds, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_math<MODE, WARPS, MINB><<<blocks, WARPS * 32>>>(rounds, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(out);
  return ms;
}

int main() {
  // 14M hits = 437.5k warp-rounds, as in config 5
  const long long warp_rounds = 437500;
  for (int warps_per_sm : {4, 8, 12, 16}) {
    const int blocks = 148 * warps_per_sm / 4;
    const int rounds = (int)(warp_rounds / (blocks * 4));
    const float ms = warps_per_sm <= 12 ? run<0, 4, 3>(blocks, rounds) : run<0, 4, 4>(blocks, rounds);
    printf("linearize math, %2d warps/SM: %.3f ms for %lld warp-rounds\n", warps_per_sm, ms,
           (long long)blocks * 4 * rounds);
  }
  const int blocks = 148 * 12 / 4;
  printf("cost math, 12 warps/SM: %.3f ms\n", run<1, 4, 3>(blocks, (int)(warp_rounds / (blocks * 4))));
  return 0;
}
