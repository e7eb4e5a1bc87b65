// Microbenchmark: random-gather ceiling of the B200 memory system (L2-resident and HBM-sized
// tables), for 32 B / 64 B / 128 B records gathered with 16 B loads by cooperating lanes.
// Answers "what sector rate can K4a/K4b's random accesses reach at best?"
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

// each group of G lanes gathers one REC-byte record (REC/16 units spread over the group)
template <int REC>
__global__ void k_gather(const int4* __restrict__ tab, uint32_t nrec, long long nreq,
                         unsigned long long* out) {
  constexpr int U = REC / 16;
  int4 acc = make_int4(0, 0, 0, 0);
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nthreads = (long long)gridDim.x * blockDim.x;
  // thread t handles unit (t % U) of record request (t / U)
  for (long long u = tid; u < nreq * U; u += nthreads) {
    const long long req = u / U;
    const uint32_t rec = hash32((uint32_t)req * 2654435761u) % nrec;
    const int4 v = __ldg(tab + (size_t)rec * U + (u % U));
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678) out[0] = 1;
}

template <int REC>
void run(size_t table_bytes, long long nreq) {
  int4* tab;
  cudaMalloc(&tab, table_bytes);
  cudaMemset(tab, 1, table_bytes);
  unsigned long long* out;
  cudaMalloc(&out, 8);
  const uint32_t nrec = (uint32_t)(table_bytes / REC);
  const int blocks = 148 * 8, threads = 256;
  k_gather<REC><<<blocks, threads>>>(tab, nrec, nreq, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_gather<REC><<<blocks, threads>>>(tab, nrec, nreq, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double sectors = (double)nreq * ((REC + 31) / 32);
  printf("rec %3d B, table %6.0f MB: %.3f ms, %.1f Grec/s, %.0f sectors/ns (%.2f TB/s of sectors)\n",
         REC, table_bytes / 1e6, ms, nreq / ms / 1e6, sectors / ms / 1e6, sectors * 32 / ms / 1e9);
  cudaFree(tab);
  cudaFree(out);
}

int main() {
  const long long nreq = 20000000;
  for (size_t tb : {(size_t)32 << 20, (size_t)64 << 20, (size_t)512 << 20}) {
    run<32>(tb, nreq);
    run<64>(tb, nreq);
    run<128>(tb, nreq);
  }
  return 0;
}
