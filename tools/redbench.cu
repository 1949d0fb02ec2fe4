// L2 atomic (RED) throughput microbenchmark for the CBAA update roofline.
// the update kernel is bound by random single-word
// red.global.or.b32 into the cube; its peak is not in MEASURED_PEAKS.json,
// so it is measured here on the box.  Standalone: nvcc -o redbench redbench.cu
#include <cstdio>
#include <cstdint>
#include <string>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hmix(uint32_t h) {
  h ^= h >> 16; h *= 0x7feb352dU; h ^= h >> 15; h *= 0x846ca68bU; h ^= h >> 16; return h;
}

// mode 0: RED.OR random word; 1: RED with L2 evict_last hint; 2: LDG random word;
// 3: ATOM.OR with return (forces round trip); 4: LDG through L1 (ld.global.ca)
template <int MODE>
__global__ void k_rand(uint32_t* buf, uint32_t words_mask, uint64_t ops_per_thread, uint32_t seed, uint32_t* sink) {
  uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  for (uint64_t i = 0; i < ops_per_thread; i += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint32_t h = hmix(tid * 0x9E3779B1U + (uint32_t)(i + u) * 0x85EBCA6BU + seed);
      uint32_t w = h & words_mask;
      uint32_t m = 1u << (hmix(h) & 31);
      if (MODE == 0) {
        asm volatile("red.global.or.b32 [%0], %1;" :: "l"(buf + w), "r"(m) : "memory");
      } else if (MODE == 1) {
        asm volatile("red.global.L2::cache_hint.or.b32 [%0], %1, %2;" :: "l"(buf + w), "r"(m), "l"(pol) : "memory");
      } else if (MODE == 2) {
        uint32_t v;
        asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(buf + w));
        acc += v;
      } else if (MODE == 4) {
        uint32_t v;
        asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(v) : "l"(buf + w));
        acc += v;
      } else {
        acc += atomicOr(buf + w, m);
      }
    }
  }
  if (acc == 0xdeadbeef) sink[0] = acc;
}

// Streams 8 B/pair of input (u32 src/dst SoA, ld.global.cs) and issues 4 REDs per pair into the cube,
// like the update but with a trivial hash: isolates the stream+RED mix.
__global__ void k_stream_red(const uint4* __restrict__ src, const uint4* __restrict__ dst, uint64_t n4,
                             uint32_t* cube, uint32_t words_mask) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    uint4 s = __ldcs(src + i), d = __ldcs(dst + i);
    uint32_t ss[4] = {s.x, s.y, s.z, s.w}, dd[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      uint32_t h = hmix(ss[p]);
      uint32_t row = hmix(dd[p]) & 4095;
      uint32_t base = (h & words_mask) & ~127u;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        uint32_t w = (base ^ (hmix(h + a) & words_mask & ~127u)) | (row >> 5);
        asm volatile("red.global.or.b32 [%0], %1;" :: "l"(cube + (w & words_mask)), "r"(1u << (row & 31)) : "memory");
      }
    }
  }
}

__global__ void k_fill(uint32_t* p, uint64_t n, uint32_t seed) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) p[i] = hmix((uint32_t)i ^ seed) * 2654435761u;
}

int main(int argc, char** argv) {
  const bool quick = argc > 1 && std::string(argv[1]) == "--quick";
  int dev = 0, sms = 0, l2 = 0, persist = 0, clk = 0;
  CK(cudaSetDevice(dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  cudaDeviceGetAttribute(&persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"sms\": %d, \"l2_bytes\": %d, \"max_persist_l2\": %d, \"clock_khz\": %d}\n", sms, l2, persist, clk);
  uint32_t* buf; uint32_t* sink;
  const uint64_t maxbytes = 1ull << 30;
  CK(cudaMalloc(&buf, maxbytes)); CK(cudaMalloc(&sink, 64));
  CK(cudaMemset(buf, 0, maxbytes));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = sms * 8, threads = 256;
  uint64_t nthreads = (uint64_t)blocks * threads;
  const uint64_t opt = 1024;  // ops per thread
  uint64_t sizes_kb[] = {16, 128, 1024, 4096, 16384, 32768, 65536, 98304, 131072, 262144, 1048576};
  const char* names[] = {"red", "red_evict_last", "ldg", "atom_ret", "ldg_ca"};
  if (quick) {  // roofline denominators: random single-word RED.OR and LDG over an L2-resident 64 MiB buffer
    const uint32_t mask = (uint32_t)((64ull << 20) / 4) - 1;
    for (int mode : {0, 2, 4}) {
      float best = 1e30f;
      for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k_rand<0><<<blocks, threads>>>(buf, mask, opt, rep, sink);
        else if (mode == 2) k_rand<2><<<blocks, threads>>>(buf, mask, opt, rep, sink);
        else k_rand<4><<<blocks, threads>>>(buf, mask, opt, rep, sink);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
      }
      printf("{\"mode\": \"%s\", \"buf_mb\": 64, \"ms\": %.4f, \"Gops\": %.2f}\n", names[mode], best,
             (double)nthreads * opt / best / 1e6);
    }
    return 0;
  }
  for (int mode = 0; mode < 5; ++mode) {
    for (uint64_t kb : sizes_kb) {
      uint32_t words = (uint32_t)((kb << 10) / 4);
      uint32_t mask = words - 1;
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k_rand<0><<<blocks, threads>>>(buf, mask, opt, rep, sink);
        if (mode == 1) k_rand<1><<<blocks, threads>>>(buf, mask, opt, rep, sink);
        if (mode == 2) k_rand<2><<<blocks, threads>>>(buf, mask, opt, rep, sink);
        if (mode == 3) k_rand<3><<<blocks, threads>>>(buf, mask, opt, rep, sink);
        if (mode == 4) k_rand<4><<<blocks, threads>>>(buf, mask, opt, rep, sink);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
      }
      double ops = (double)nthreads * opt;
      printf("{\"mode\": \"%s\", \"buf_kb\": %llu, \"ms\": %.4f, \"Gops\": %.2f}\n", names[mode],
             (unsigned long long)kb, best, ops / best / 1e6);
    }
  }
  // stream + RED: 100M pairs (800 MB) into a 128 MiB cube, like C2
  {
    uint64_t n = 100000000ull, n4 = n / 4;
    uint32_t *src, *dst;
    CK(cudaMalloc(&src, n * 4)); CK(cudaMalloc(&dst, n * 4));
    k_fill<<<blocks, threads>>>(src, n, 1); k_fill<<<blocks, threads>>>(dst, n, 2);
    uint64_t cube_mb[] = {32, 64, 128, 256};
    for (uint64_t mb : cube_mb) {
      uint32_t mask = (uint32_t)((mb << 20) / 4) - 1;
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaMemsetAsync(buf, 0, mb << 20);
        cudaEventRecord(e0);
        k_stream_red<<<blocks, threads>>>((const uint4*)src, (const uint4*)dst, n4, buf, mask);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
      }
      printf("{\"mode\": \"stream_red\", \"cube_mb\": %llu, \"ms\": %.4f, \"Gpairs\": %.2f, \"Gred\": %.2f}\n",
             (unsigned long long)mb, best, n / best / 1e6, 4.0 * n / best / 1e6);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
