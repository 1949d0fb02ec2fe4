// Shared-memory atomic throughput on one B200 SM set: ATOMS.ADD with return (the scatter's rank),
// RED.ADD / RED.OR without return, and plain LDS + STS, on random words of a 16 KiB table.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/atoms_bench tools/atoms_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t h32(uint32_t x) { x ^= x >> 16; x *= 0x45d9f3bu; x ^= x >> 16; return x; }

template <int MODE>
__global__ void __launch_bounds__(1024) k(uint32_t iters, uint32_t words, uint32_t* out) {
  extern __shared__ uint32_t t[];
  for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) t[i] = 0;
  __syncthreads();
  uint32_t acc = 0, x = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  for (uint32_t i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    const uint32_t a = h32(x) & (words - 1);
    if (MODE == 0) acc += atomicAdd(&t[a], 1u);
    else if (MODE == 1) atomicAdd(&t[a], 1u);              // result unused: RED
    else if (MODE == 2) atomicOr(&t[a], 1u << (x & 31));   // RED.OR
    else { acc += t[a]; t[(a + 7) & (words - 1)] = acc; }
  }
  __syncthreads();
  if (acc == 0x12345678u) out[0] = acc + t[0];
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out; cudaMalloc(&out, 4);
  const uint32_t iters = 4096, words = 4096;
  const char* names[] = {"atoms_add_return", "red_shared_add", "red_shared_or", "lds_sts"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int threads : {256, 1024}) {
      auto launch = [&]() {
        if (mode == 0) k<0><<<sms * (1024 / threads), threads, words * 4>>>(iters, words, out);
        if (mode == 1) k<1><<<sms * (1024 / threads), threads, words * 4>>>(iters, words, out);
        if (mode == 2) k<2><<<sms * (1024 / threads), threads, words * 4>>>(iters, words, out);
        if (mode == 3) k<3><<<sms * (1024 / threads), threads, words * 4>>>(iters, words, out);
      };
      launch();
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double ops = (double)sms * 1024 * iters;   // lane operations
      int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      printf("{\"op\": \"%s\", \"threads_per_cta\": %d, \"ms\": %.4f, \"G_lane_ops_per_s\": %.1f, \"lanes_per_clk_per_sm\": %.3f}\n",
             names[mode], threads, ms, ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk * 1e3));
    }
  }
  return 0;
}
