// Zero-copy write bandwidth probe: SM stores into mapped pinned host memory vs a copy-engine
// D2H memcpy of the same bytes (18.8 MB = config 5's compact fp32 records).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zc_probe zc_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_write(unsigned* __restrict__ dst, size_t words, int rec_words) {
  // one warp per 94-word record, like a K4b epilogue
  const size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const size_t base = w * rec_words;
  if (base >= words) return;
  for (int k = lane; k < rec_words; k += 32) dst[base + k] = (unsigned)(base + k);
}

int main() {
  const int F = 50000, RW = 94;
  const size_t words = (size_t)F * RW, bytes = words * 4;
  unsigned *h = nullptr, *d = nullptr;
  cudaMallocHost(&h, bytes);
  cudaMalloc(&d, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best_zc = 1e9, best_dev = 1e9, best_cp = 1e9;
  for (int rep = 0; rep < 20; ++rep) {
    const int threads = 128, blocks = (F * 32 + threads - 1) / threads;
    cudaEventRecord(a);
    k_write<<<blocks, threads>>>(h, words, RW);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best_zc) best_zc = ms;
    cudaEventRecord(a);
    k_write<<<blocks, threads>>>(d, words, RW);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best_dev) best_dev = ms;
    cudaEventRecord(a);
    cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best_cp) best_cp = ms;
  }
  bool ok = true;
  for (size_t i = 0; i < words; i += 9973) ok &= h[i] == (unsigned)i;
  printf("{\"bytes\": %zu, \"zero_copy_ms\": %.4f, \"zero_copy_gbs\": %.1f, \"device_write_ms\": %.4f, "
         "\"memcpy_d2h_ms\": %.4f, \"memcpy_gbs\": %.1f, \"ok\": %d}\n",
         bytes, best_zc, bytes / best_zc / 1e6, best_dev, best_cp, bytes / best_cp / 1e6, ok);
  return 0;
}
