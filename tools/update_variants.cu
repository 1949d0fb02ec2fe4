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

// V8: input tiles staged into shared memory by the TMA bulk-copy engine (cp.async.bulk + mbarrier),
// double-buffered; the L1/LSU miss path then carries only the random cube accesses.
constexpr int kTile = 2048;   // pairs per tile: 8 KB src + 8 KB dst per stage

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
__global__ void __launch_bounds__(kThreads) kx_update_tma(const __grid_constant__ Geo G, const uint32_t* __restrict__ src,
                                                          const uint32_t* __restrict__ dst, uint64_t n,
                                                          uint32_t* __restrict__ cube, uint32_t lo, uint32_t span) {
  __shared__ __align__(128) uint32_t s_src[2][kTile];
  __shared__ __align__(128) uint32_t s_dst[2][kTile];
  __shared__ __align__(8) uint64_t bar[2];
  const uint64_t n_tiles = n / kTile;
  uint32_t skip = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t tile = blockIdx.x;
  if (threadIdx.x == 0 && tile < n_tiles) {
    mbar_expect_tx(&bar[0], 2 * kTile * 4);
    bulk_g2s(s_src[0], src + tile * kTile, kTile * 4, &bar[0]);
    bulk_g2s(s_dst[0], dst + tile * kTile, kTile * 4, &bar[0]);
  }
  uint32_t it = 0;
  for (; tile < n_tiles; tile += gridDim.x, ++it) {
    const int st = it & 1;
    const uint64_t next = tile + gridDim.x;
    if (threadIdx.x == 0 && next < n_tiles) {   // stage st^1 was released by the __syncthreads below
      mbar_expect_tx(&bar[st ^ 1], 2 * kTile * 4);
      bulk_g2s(s_src[st ^ 1], src + next * kTile, kTile * 4, &bar[st ^ 1]);
      bulk_g2s(s_dst[st ^ 1], dst + next * kTile, kTile * 4, &bar[st ^ 1]);
    }
    mbar_wait(&bar[st], (it >> 1) & 1);
    const uint4* S4 = reinterpret_cast<const uint4*>(s_src[st]);
    const uint4* D4 = reinterpret_cast<const uint4*>(s_dst[st]);
    uint4 sa = S4[threadIdx.x], sb = S4[threadIdx.x + kThreads];
    uint4 da = D4[threadIdx.x], db = D4[threadIdx.x + kThreads];
    uint32_t ss[4] = {sa.x, sa.y, sa.z, sa.w}, dd[4] = {da.x, da.y, da.z, da.w};
    uint32_t ss2[4] = {sb.x, sb.y, sb.z, sb.w}, dd2[4] = {db.x, db.y, db.z, db.w};
    __syncthreads();   // everyone has its 8 pairs in registers: the stage can be refilled
    set_quad<3, 1, CBAA_UPDATE_TEST_SET, false>(G, ss, dd, cube, lo, span, skip);
    set_quad<3, 1, CBAA_UPDATE_TEST_SET, false>(G, ss2, dd2, cube, lo, span, skip);
  }
  // remainder pairs (< one tile) one per thread
  const uint64_t rem0 = n_tiles * kTile;
  for (uint64_t k = rem0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x)
    set_pair_generic<CBAA_UPDATE_TEST_SET>(G, src[k], dst[k], cube, lo, span);
}

// V9/V10: the product's 8-pair body with the input read L1::no_allocate (it never pollutes L1);
// V10 additionally marks cube loads L1::evict_last.
__device__ __forceinline__ uint4 ld_in_noalloc(const uint32_t* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_cube_keep(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.L1::evict_last.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_cube_first(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.L1::evict_first.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_cube_nc(const uint32_t* p) { return __ldg(p); }
__device__ __forceinline__ uint32_t ld_cube_cg(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ uint32_t ld_cube_unchanged(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.L1::evict_unchanged.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
template <int KEEP>
__global__ void __launch_bounds__(kThreads) kx_update_na(const __grid_constant__ Geo G, const uint32_t* __restrict__ src,
                                                         const uint32_t* __restrict__ dst, uint64_t n8,
                                                         uint32_t* __restrict__ cube, uint32_t lo, uint32_t span) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += stride) {
    uint4 s0 = ld_in_noalloc(src + 8 * i), s1 = ld_in_noalloc(src + 8 * i + 4);
    uint4 d0 = ld_in_noalloc(dst + 8 * i), d1 = ld_in_noalloc(dst + 8 * i + 4);
    uint32_t ss[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
    uint32_t dd[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
    uint32_t w[8][4], bit[8], v[8][4];
#pragma unroll
    for (int p = 0; p < 8; ++p) bit[p] = pair_targets<3, 1>(G, ss[p], dd[p], lo, span, w[p]);
#pragma unroll
    for (int p = 0; p < 8; ++p)
#pragma unroll
      for (int a = 0; a < 4; ++a)
        v[p][a] = w[p][a] == kNoWord ? bit[p]
                  : (KEEP == 1 ? ld_cube_keep(cube + w[p][a])
                     : KEEP == 2 ? ld_cube_first(cube + w[p][a])
                     : KEEP == 3 ? ld_cube_unchanged(cube + w[p][a])
                     : KEEP == 4 ? ld_cube_nc(cube + w[p][a])
                     : KEEP == 5 ? ld_cube_cg(cube + w[p][a]) : __ldca(cube + w[p][a]));
#pragma unroll
    for (int p = 0; p < 8; ++p)
#pragma unroll
      for (int a = 0; a < 4; ++a)
        if (!(v[p][a] & bit[p])) red_or(cube + w[p][a], bit[p]);
  }
}

// V11/V12: the product's 8-pair body with a register budget for 3 / 4 CTAs per SM.
template <int MINB>
__global__ void __launch_bounds__(kThreads, MINB) kx_update_lb(const __grid_constant__ Geo G, const uint32_t* __restrict__ src,
                                                               const uint32_t* __restrict__ dst, uint64_t n8,
                                                               uint32_t* __restrict__ cube, uint32_t lo, uint32_t span) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t skip = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += stride) {
    uint4 sa = ld_stream4(src + 8 * i), sb = ld_stream4(src + 8 * i + 4);
    uint4 da = ld_stream4(dst + 8 * i), db = ld_stream4(dst + 8 * i + 4);
    uint32_t ss[4] = {sa.x, sa.y, sa.z, sa.w}, dd[4] = {da.x, da.y, da.z, da.w};
    uint32_t ss2[4] = {sb.x, sb.y, sb.z, sb.w}, dd2[4] = {db.x, db.y, db.z, db.w};
    set_quad<3, 1, CBAA_UPDATE_TEST_SET, false>(G, ss, dd, cube, lo, span, skip);
    set_quad<3, 1, CBAA_UPDATE_TEST_SET, false>(G, ss2, dd2, cube, lo, span, skip);
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
      case 8: kx_update_tma<<<grid, kThreads, 0, s>>>(h->G, src, dst, n, h->cube, lo, hi - lo); break;
      case 11: kx_update_lb<3><<<grid, kThreads, 0, s>>>(h->G, src, dst, n / 8, h->cube, lo, hi - lo); break;
      case 12: kx_update_lb<4><<<grid, kThreads, 0, s>>>(h->G, src, dst, n / 8, h->cube, lo, hi - lo); break;
      case 9: kx_update_na<0><<<grid, kThreads, 0, s>>>(h->G, src, dst, n / 8, h->cube, lo, hi - lo); break;
      case 10: kx_update_na<1><<<grid, kThreads, 0, s>>>(h->G, src, dst, n / 8, h->cube, lo, hi - lo); break;
      case 13: kx_update_na<2><<<grid, kThreads, 0, s>>>(h->G, src, dst, n / 8, h->cube, lo, hi - lo); break;
      case 14: kx_update_na<3><<<grid, kThreads, 0, s>>>(h->G, src, dst, n / 8, h->cube, lo, hi - lo); break;
      case 15: kx_update_na<4><<<grid, kThreads, 0, s>>>(h->G, src, dst, n / 8, h->cube, lo, hi - lo); break;
      case 16: kx_update_na<5><<<grid, kThreads, 0, s>>>(h->G, src, dst, n / 8, h->cube, lo, hi - lo); break;
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
