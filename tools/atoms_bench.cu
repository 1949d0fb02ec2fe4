// Shared-memory rank primitives on one B200: ATOMS.ADD with return (the scatter's rank), RED.ADD /
// RED.OR without return, plain LDS + STS, and a warp-level multisplit rank (10 ballots → the lanes of the
// warp with the same 10-bit bin, one leader updates a warp-private 1024-counter histogram): random keys
// over 1024 or 4096 words.  Prints lane operations per clock per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/atoms_bench tools/atoms_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t h32(uint32_t x) { x ^= x >> 16; x *= 0x45d9f3bu; x ^= x >> 16; return x; }

template <int MODE>
__global__ void __launch_bounds__(1024) k(uint32_t iters, uint32_t words, uint32_t* out) {
  extern __shared__ uint32_t t[];
  const uint32_t tot = MODE == 4 ? 1024u * (blockDim.x >> 5) : words;
  for (uint32_t i = threadIdx.x; i < tot; i += blockDim.x) t[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t* wh = t + (threadIdx.x >> 5) * 1024u;
  uint32_t acc = 0, x = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  for (uint32_t i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    const uint32_t a = h32(x) & (words - 1);
    if (MODE == 0) acc += atomicAdd(&t[a], 1u);
    else if (MODE == 1) atomicAdd(&t[a], 1u);              // result unused: RED
    else if (MODE == 2) atomicOr(&t[a], 1u << (x & 31));   // RED.OR
    else if (MODE == 3) { acc += t[a]; t[(a + 7) & (words - 1)] = acc; }
    else {   // warp multisplit over 1024 bins
      const uint32_t b = a & 1023u;
      uint32_t peers = 0xffffffffu;
#pragma unroll
      for (int j = 0; j < 10; ++j) {
        const uint32_t m = __ballot_sync(0xffffffffu, (b >> j) & 1u);
        peers &= ((b >> j) & 1u) ? m : ~m;
      }
      const uint32_t lt = peers & ((1u << lane) - 1u);
      const uint32_t cnt = wh[b];
      __syncwarp();
      if (lt == 0) wh[b] = cnt + __popc(peers);
      __syncwarp();
      acc += cnt + __popc(lt);
    }
  }
  __syncthreads();
  if (acc == 0x12345678u) out[0] = acc + t[0];
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out; cudaMalloc(&out, 4);
  const uint32_t iters = 4096;
  const char* names[] = {"atoms_add_return", "red_shared_add", "red_shared_or", "lds_sts", "warp_multisplit_1024"};
  cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  for (int mode = 0; mode < 5; ++mode) {
    for (uint32_t words : {1024u, 4096u}) {
      if (mode == 4 && words != 1024u) continue;
      for (int threads : {256, 512, 1024}) {
        const size_t smem = mode == 4 ? 4096u * (threads / 32) : words * 4;
        auto launch = [&]() {
          const int grid = sms * (2048 / threads);
          if (mode == 0) k<0><<<grid, threads, smem>>>(iters, words, out);
          if (mode == 1) k<1><<<grid, threads, smem>>>(iters, words, out);
          if (mode == 2) k<2><<<grid, threads, smem>>>(iters, words, out);
          if (mode == 3) k<3><<<grid, threads, smem>>>(iters, words, out);
          if (mode == 4) k<4><<<grid, threads, smem>>>(iters, words, out);
        };
        launch();
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double ops = (double)sms * 2048 * iters;   // lane operations
        int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        const cudaError_t e = cudaGetLastError();
        printf("{\"op\": \"%s\", \"words\": %u, \"threads_per_cta\": %d, \"ms\": %.4f, \"G_lane_ops_per_s\": %.1f, "
               "\"lanes_per_clk_per_sm\": %.3f, \"err\": \"%s\"}\n",
               names[mode], words, threads, ms, ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk * 1e3),
               cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
