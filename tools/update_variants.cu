// Experimental update-kernel variants, built as a separate tools/libvariants.so that contains the
// whole product library (single translation unit) plus cbaa_x_update(h, variant, ...).  Used only by
// tools/variants.py to decide what goes into the product kernel; never by tests or the bench.
#include "../paper_1901_06207_b200/csrc/cbaa.cu"

namespace cbaa {

// V1: eight pairs per thread per step (two uint4 per array), test-and-set.
template <bool DUMMY>
__global__ void __launch_bounds__(kThreads) kx_update8(const __grid_constant__ Geo G, const uint32_t* __restrict__ src,
                                                       const uint32_t* __restrict__ dst, uint64_t n8,
                                                       uint32_t* __restrict__ cube, uint32_t lo, uint32_t span) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t skip = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += stride) {
    uint4 s0 = ld_stream4(src + 8 * i), s1 = ld_stream4(src + 8 * i + 4);
    uint4 d0 = ld_stream4(dst + 8 * i), d1 = ld_stream4(dst + 8 * i + 4);
    uint32_t ss[4] = {s0.x, s0.y, s0.z, s0.w}, dd[4] = {d0.x, d0.y, d0.z, d0.w};
    uint32_t ss1[4] = {s1.x, s1.y, s1.z, s1.w}, dd1[4] = {d1.x, d1.y, d1.z, d1.w};
    set_quad<3, 1, CBAA_UPDATE_TEST_SET, false>(G, ss, dd, cube, lo, span, skip);
    set_quad<3, 1, CBAA_UPDATE_TEST_SET, false>(G, ss1, dd1, cube, lo, span, skip);
  }
}

// V2: the product kernel body with a register cap for higher occupancy.
__global__ void __launch_bounds__(kThreads, 6) kx_update_occ(const __grid_constant__ Geo G, const uint32_t* __restrict__ src,
                                                             const uint32_t* __restrict__ dst, uint64_t n4,
                                                             uint32_t* __restrict__ cube, uint32_t lo, uint32_t span) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t skip = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    uint4 s = ld_stream4(src + 4 * i), d = ld_stream4(dst + 4 * i);
    uint32_t ss[4] = {s.x, s.y, s.z, s.w}, dd[4] = {d.x, d.y, d.z, d.w};
    set_quad<3, 1, CBAA_UPDATE_TEST_SET, false>(G, ss, dd, cube, lo, span, skip);
  }
}

// V3: test-and-set behind a per-CTA shared-memory filter of words already seen all-ones (FULL words).
// A hit skips the global access entirely (one LDS instead of one random L1 sector).  Entries hold a
// word index whose word was observed == 0xffffffff; since bits only go 0 -> 1, that stays true.
template <int LOG_T>
__global__ void __launch_bounds__(kThreads) kx_update_filter(const __grid_constant__ Geo G,
                                                             const uint32_t* __restrict__ src,
                                                             const uint32_t* __restrict__ dst, uint64_t n4,
                                                             uint32_t* __restrict__ cube, uint32_t lo, uint32_t span) {
  constexpr uint32_t T = 1u << LOG_T;
  __shared__ uint32_t full[T];
  for (uint32_t k = threadIdx.x; k < T; k += kThreads) full[k] = kNoWord;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    uint4 s = ld_stream4(src + 4 * i), d = ld_stream4(dst + 4 * i);
    uint32_t ss[4] = {s.x, s.y, s.z, s.w}, dd[4] = {d.x, d.y, d.z, d.w};
    uint32_t w[4][4], bit[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) bit[p] = pair_targets<3, 1>(G, ss[p], dd[p], lo, span, w[p]);
    uint32_t v[4][4];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        uint32_t x = w[p][a];
        bool hit = x == kNoWord || full[(x ^ (x >> LOG_T)) & (T - 1)] == x;
        v[p][a] = hit ? 0xffffffffu : __ldca(cube + x);
      }
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        uint32_t x = w[p][a];
        if (x == kNoWord) continue;
        if (v[p][a] == 0xffffffffu) {
          full[(x ^ (x >> LOG_T)) & (T - 1)] = x;
        } else if (!(v[p][a] & bit[p])) {
          red_or(cube + x, bit[p]);
        }
      }
  }
}

// V4: single pass, cube loads and REDs with an L2 evict_last policy (cube kept, input evict_first).
__device__ __forceinline__ uint32_t ld_ca_keep(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.ca.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void red_keep(uint32_t* p, uint32_t v, uint64_t pol) {
  asm volatile("red.relaxed.gpu.global.or.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__global__ void __launch_bounds__(kThreads) kx_update_keep(const __grid_constant__ Geo G, const uint32_t* __restrict__ src,
                                                           const uint32_t* __restrict__ dst, uint64_t n4,
                                                           uint32_t* __restrict__ cube, uint32_t lo, uint32_t span) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    uint4 s = ld_stream4(src + 4 * i), d = ld_stream4(dst + 4 * i);
    uint32_t ss[4] = {s.x, s.y, s.z, s.w}, dd[4] = {d.x, d.y, d.z, d.w};
    uint32_t w[4][4], bit[4], v[4][4];
#pragma unroll
    for (int p = 0; p < 4; ++p) bit[p] = pair_targets<3, 1>(G, ss[p], dd[p], lo, span, w[p]);
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int a = 0; a < 4; ++a) v[p][a] = w[p][a] != kNoWord ? ld_ca_keep(cube + w[p][a], pol) : bit[p];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int a = 0; a < 4; ++a)
        if (!(v[p][a] & bit[p])) red_keep(cube + w[p][a], bit[p], pol);
  }
}

}  // namespace cbaa

extern "C" int cbaa_x_update(cbaa_handle* h, int variant, int passes, int blocks_per_sm, const uint32_t* src,
                             const uint32_t* dst, uint64_t n, cbaa_stream stream) {
  using namespace cbaa;
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t W = h->cube_words;
  for (int p = 0; p < passes; ++p) {
    uint32_t lo = (uint32_t)(W * p / passes), hi = (uint32_t)(W * (p + 1) / passes);
    int grid = h->sms * blocks_per_sm;
    switch (variant) {
      case 1: kx_update8<true><<<grid, kThreads, 0, s>>>(h->G, src, dst, n / 8, h->cube, lo, hi - lo); break;
      case 2: kx_update_occ<<<grid, kThreads, 0, s>>>(h->G, src, dst, n / 4, h->cube, lo, hi - lo); break;
      case 3: kx_update_filter<12><<<grid, kThreads, 0, s>>>(h->G, src, dst, n / 4, h->cube, lo, hi - lo); break;
      case 4: kx_update_filter<13><<<grid, kThreads, 0, s>>>(h->G, src, dst, n / 4, h->cube, lo, hi - lo); break;
      case 5: kx_update_keep<<<grid, kThreads, 0, s>>>(h->G, src, dst, n / 4, h->cube, lo, hi - lo); break;
      case 6:
      case 7: {  // product kernel with the smem carveout forced to 0 (max L1) / to max smem (min L1)
        cudaFuncSetAttribute(k_update<3, 1, CBAA_UPDATE_TEST_SET, false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             variant == 6 ? 0 : 100);
        k_update<3, 1, CBAA_UPDATE_TEST_SET, false><<<grid, kThreads, 0, s>>>(h->G, src, dst, 0, n / 4, n, h->cube, lo,
                                                                               hi - lo, nullptr);
        cudaFuncSetAttribute(k_update<3, 1, CBAA_UPDATE_TEST_SET, false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             -1);
        break;
      }
      default:
        k_update<3, 1, CBAA_UPDATE_TEST_SET, false><<<grid, kThreads, 0, s>>>(h->G, src, dst, 0, n / 4, n, h->cube, lo,
                                                                               hi - lo, nullptr);
    }
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -3;
}
