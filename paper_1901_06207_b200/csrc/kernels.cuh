// sm_100a kernels of the CBAA window path (DESIGN.md §6 lists each with its roofline).
//   k_update      Alg. 1: 128-bit streaming loads of SoA pairs, 4 REDs per pair
//   k_zero        window reset
//   k_or_merge    global OR merge (Q1)
//   k_zero_counts zero counts of the RA columns (Alg. 2 input) and Ztot per CS
//   k_hot         per-CS η/ε/θ_bn + ordered hot-column compaction (Alg. 2) + work prefix
//   k_join3       Alg. 3 first half for |RA| = 3: CP chains by sorted-run join
//   k_union       Alg. 3 second half: warp-cooperative union-column AND/popcount, output with the
//                 Thm. 2 estimate
//   k_tuples      Alg. 3 for any |RA|: Cartesian enumeration with the union check inline
//   k_debug_map   Alg. 1 mapping only (test hook)
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "geometry.cuh"

namespace cbaa {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
// Window-end kernels run 128-thread CTAs so that, when windows are pipelined, a detect CTA fits in the
// registers the two persistent update CTAs leave free on every SM (2 × 8 warps × 112 regs of 64 K).
constexpr int kDetThreads = 128;
constexpr int kDetWarps = kDetThreads / 32;

// ---------------------------------------------------------------- primitives
__device__ __forceinline__ void red_or(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void red_or64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.or.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint4 ld_stream4(const uint32_t* p) {
  // input pairs are read exactly once: evict-first so they do not displace the cube in L2
  return __ldcs(reinterpret_cast<const uint4*>(p));
}

// one bulk prefetch of [p, p + bytes) into L2 (16-B aligned address and size; no registers, no shared memory)
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ uint32_t warp_sum(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// a0 membership test: one L1-resident bitmap probe by the top 16 bits; only addresses in a /16 that holds
// a longer prefix fall through to the exact comparison against the prefix list.
__device__ __forceinline__ bool is_inner(const Geo& G, uint32_t ip) {
  const uint32_t t = ip >> 16;
  if ((__ldg(G.full_bits + (t >> 5)) >> (t & 31)) & 1u) return true;
  if (!((__ldg(G.part_bits + (t >> 5)) >> (t & 31)) & 1u)) return false;
  bool in = false;
  for (uint32_t k = 0; k < G.n_prefix; ++k) in |= (ip & G.pmask[k]) == G.prefix[k];
  return in;
}

// a0 (Q25): returns false if the pair has zero or two inner endpoints.
template <bool PREFIX>
__device__ __forceinline__ bool normalize(const Geo& G, uint32_t& s, uint32_t& d) {
  if (!PREFIX) return true;
  bool si = is_inner(G, s), di = is_inner(G, d);
  if (si == di) return false;
  if (di) {
    uint32_t t = s;
    s = d;
    d = t;
  }
  return true;
}

// Word index of every bit Alg. 1 sets for one normalised pair, and the bit mask.
// Arrays: RA(0..nra−1) then VA(0..nva−1).  Words outside [lo, lo+span) become kNoWord.
constexpr uint32_t kNoWord = 0xffffffffu;

template <int NRA, int NVA>
__device__ __forceinline__ uint32_t pair_targets(const Geo& G, uint32_t iip, uint32_t oip, uint32_t lo, uint32_t span,
                                                 uint32_t* w) {
  uint32_t mi = G.mangle_a * iip + G.mangle_b;        // mangle (Q3)
  uint32_t mo = G.mangle_a * oip + G.mangle_b;        // oip mangled too (Q2)
  uint32_t cs = mi & G.rmask;                          // RP selects the CS
  uint32_t lp = mi >> G.r;                             // LP
  uint32_t row = mix32(mo ^ G.bv_seed) & (G.g - 1);    // bvIdx = H_bv(oip)
  uint32_t base = cs * G.cs_words + (row >> 5);
  uint64_t dbl = ((uint64_t)lp << G.L) | lp;           // LP twice: a rotate becomes one shift (Q6/Q7)
#pragma unroll
  for (int i = 0; i < NRA; ++i) {
    uint32_t col = (uint32_t)(dbl >> G.sh[i]) & G.colmask[i];     // CL(i)
    uint32_t x = base + G.arr_off[i] + (col << G.wpc_log2);
    w[i] = x - lo < span ? x : kNoWord;
  }
#pragma unroll
  for (int j = 0; j < NVA; ++j) {
    uint32_t col = mix32(lp ^ G.va_seeds[j]) & G.colmask[NRA + j];   // CL(j) = H_j(LP)
    uint32_t x = base + G.arr_off[NRA + j] + (col << G.wpc_log2);
    w[NRA + j] = x - lo < span ? x : kNoWord;
  }
  return 1u << (row & 31);
}

// Any shape with NA = |RA| + |VA| arrays known at compile time and the RA/VA split at run time
// (NVA < 0 in the templates below): the same word indices as pair_targets, array by array.
template <int NA>
__device__ __forceinline__ uint32_t pair_targets_rt(const Geo& G, uint32_t iip, uint32_t oip, uint32_t lo, uint32_t span,
                                                    uint32_t* w) {
  uint32_t mi = G.mangle_a * iip + G.mangle_b;
  uint32_t mo = G.mangle_a * oip + G.mangle_b;
  uint32_t cs = mi & G.rmask;
  uint32_t lp = mi >> G.r;
  uint32_t row = mix32(mo ^ G.bv_seed) & (G.g - 1);
  uint32_t base = cs * G.cs_words + (row >> 5);
  uint64_t dbl = ((uint64_t)lp << G.L) | lp;
#pragma unroll
  for (int a = 0; a < NA; ++a) {
    const bool ra = a < (int)G.num_ra;
    uint32_t col = ra ? (uint32_t)(dbl >> G.sh[a < CBAA_MAX_RA ? a : 0]) & G.colmask[a]   // CL(i)
                      : mix32(lp ^ G.va_seeds[(a - G.num_ra) & (CBAA_MAX_VA - 1)]) & G.colmask[a];   // H_j
    uint32_t x = base + G.arr_off[a] + (col << G.wpc_log2);
    w[a] = x - lo < span ? x : kNoWord;
  }
  return 1u << (row & 31);
}

// Generic geometry (runtime |RA|, |VA|): one pair at a time.
template <int MODE>
__device__ __forceinline__ void set_pair_generic(const Geo& G, uint32_t iip, uint32_t oip, uint32_t* __restrict__ cube,
                                                 uint32_t lo, uint32_t span) {
  uint32_t mi = G.mangle_a * iip + G.mangle_b;
  uint32_t mo = G.mangle_a * oip + G.mangle_b;
  uint32_t cs = mi & G.rmask;
  uint32_t lp = mi >> G.r;
  uint32_t row = mix32(mo ^ G.bv_seed) & (G.g - 1);
  uint32_t bit = 1u << (row & 31);
  uint32_t base = cs * G.cs_words + (row >> 5);
  uint64_t dbl = ((uint64_t)lp << G.L) | lp;
  for (uint32_t a = 0; a < G.narr; ++a) {
    uint32_t col = a < G.num_ra ? (uint32_t)(dbl >> G.sh[a]) & G.colmask[a]
                                : mix32(lp ^ G.va_seeds[a - G.num_ra]) & G.colmask[a];
    uint32_t x = base + G.arr_off[a] + (col << G.wpc_log2);
    if (x - lo >= span) continue;
    if (MODE == CBAA_UPDATE_TEST_SET && (__ldca(cube + x) & bit)) continue;
    red_or(cube + x, bit);
  }
}

// Four pairs of the fixed paper-shaped geometry (NRA RAs + NVA VAs): all 4·(NRA+NVA) word indices
// first, then (TEST_SET) all the L1-cached loads back to back, then the REDs still needed.
// Skipping a RED whose bit is already 1 leaves the cube unchanged: bits only go 0 → 1 inside a
// window and L1 is invalidated at every kernel boundary, so a stale 0 only costs a redundant RED.
template <int NRA, int NVA, int MODE, bool PREFIX>
__device__ __forceinline__ void set_quad(const Geo& G, uint32_t* ss, uint32_t* dd, uint32_t* __restrict__ cube,
                                         uint32_t lo, uint32_t span, uint32_t& skip) {
  constexpr int NA = NVA < 0 ? NRA : NRA + NVA;
  uint32_t w[4][NA], bit[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    bool ok = normalize<PREFIX>(G, ss[p], dd[p]);
    skip += ok ? 0u : 1u;
    if constexpr (NVA < 0) bit[p] = pair_targets_rt<NA>(G, ss[p], dd[p], lo, ok ? span : 0u, w[p]);
    else bit[p] = pair_targets<NRA, NVA>(G, ss[p], dd[p], lo, ok ? span : 0u, w[p]);
  }
  if (MODE == CBAA_UPDATE_TEST_SET) {
    uint32_t v[4][NA];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int a = 0; a < NA; ++a) v[p][a] = w[p][a] != kNoWord ? __ldca(cube + w[p][a]) : bit[p];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int a = 0; a < NA; ++a)
        if (!(v[p][a] & bit[p])) red_or(cube + w[p][a], bit[p]);
  } else {
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int a = 0; a < NA; ++a)
        if (w[p][a] != kNoWord) red_or(cube + w[p][a], bit[p]);
  }
}

// Persistent grid-stride update.  Pairs [0, head) and [head + 4·n4, n) go one per thread;
// [head, head + 4·n4) is 16-B aligned in both arrays and goes four per thread per step.
// <3, 1>: the paper shape; <NA, -1>: NA arrays, RA/VA split at run time; <0, 0>: any geometry, one
// pair at a time.
template <int NRA, int NVA, int MODE, bool PREFIX>
__global__ void __launch_bounds__(kThreads) k_update(const __grid_constant__ Geo G, const uint32_t* __restrict__ src,
                                                     const uint32_t* __restrict__ dst, uint64_t head, uint64_t n4,
                                                     uint64_t n, uint32_t* __restrict__ cube, uint32_t lo,
                                                     uint32_t span, unsigned long long* __restrict__ skipped) {
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t skip = 0;
  const uint64_t tail0 = head + 4 * n4;
  // scalar head [0, head) and tail [tail0, n), grid-stride: with differently aligned arrays head = n, so
  // the whole window can take this path and may be far larger than the grid
  for (uint64_t k = gid; k < head; k += stride) {
    uint32_t s = src[k], d = dst[k];
    if (normalize<PREFIX>(G, s, d)) set_pair_generic<MODE>(G, s, d, cube, lo, span);
    else ++skip;
  }
  for (uint64_t k = tail0 + gid; k < n; k += stride) {
    uint32_t s = src[k], d = dst[k];
    if (normalize<PREFIX>(G, s, d)) set_pair_generic<MODE>(G, s, d, cube, lo, span);
    else ++skip;
  }
  const uint32_t* s4 = src + head;
  const uint32_t* d4 = dst + head;
  if (NRA) {
    // fixed geometry: eight pairs per thread per step (two quads) — twice the random loads in flight
    // per thread (tools/variants.py: 1.58 -> 1.49 ms on C2); an odd last quad goes to thread 0
    const uint64_t n8 = n4 / 2;
    for (uint64_t i = gid; i < n8; i += stride) {
      uint4 sa = ld_stream4(s4 + 8 * i), sb = ld_stream4(s4 + 8 * i + 4);
      uint4 da = ld_stream4(d4 + 8 * i), db = ld_stream4(d4 + 8 * i + 4);
      uint32_t ss[4] = {sa.x, sa.y, sa.z, sa.w}, dd[4] = {da.x, da.y, da.z, da.w};
      uint32_t ss2[4] = {sb.x, sb.y, sb.z, sb.w}, dd2[4] = {db.x, db.y, db.z, db.w};
      set_quad<(NRA ? NRA : 1), NVA, MODE, PREFIX>(G, ss, dd, cube, lo, span, skip);
      set_quad<(NRA ? NRA : 1), NVA, MODE, PREFIX>(G, ss2, dd2, cube, lo, span, skip);
    }
    if ((n4 & 1) && gid == 0) {
      uint4 s = ld_stream4(s4 + 4 * (n4 - 1)), d = ld_stream4(d4 + 4 * (n4 - 1));
      uint32_t ss[4] = {s.x, s.y, s.z, s.w}, dd[4] = {d.x, d.y, d.z, d.w};
      set_quad<(NRA ? NRA : 1), NVA, MODE, PREFIX>(G, ss, dd, cube, lo, span, skip);
    }
  } else {
    for (uint64_t i = gid; i < n4; i += stride) {
      uint4 s = ld_stream4(s4 + 4 * i);
      uint4 d = ld_stream4(d4 + 4 * i);
      uint32_t ss[4] = {s.x, s.y, s.z, s.w};
      uint32_t dd[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        if (normalize<PREFIX>(G, ss[p], dd[p])) set_pair_generic<MODE>(G, ss[p], dd[p], cube, lo, span);
        else ++skip;
      }
    }
  }
  if (PREFIX && skipped) {
    skip = warp_sum(skip);
    if ((threadIdx.x & 31) == 0 && skip) atomicAdd(skipped, (unsigned long long)skip);
  }
}

// Interleaved ("packed") pairs: pairs[2k] = src, pairs[2k+1] = dst, e.g. straight out of a capture
// buffer.  One 16-B load carries two pairs; eight pairs per thread per step.  Pairs [0, head) and
// [head + 8·n8, n) go one per thread; [head, head + 8·n8) is 16-B aligned.
template <int NRA, int NVA, int MODE, bool PREFIX>
__global__ void __launch_bounds__(kThreads) k_update_aos(const __grid_constant__ Geo G, const uint2* __restrict__ pairs,
                                                         uint64_t head, uint64_t n8, uint64_t n,
                                                         uint32_t* __restrict__ cube, uint32_t lo, uint32_t span,
                                                         unsigned long long* __restrict__ skipped) {
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t skip = 0;
  const uint64_t tail0 = head + 8 * n8;
  for (int t = 0; t < 2; ++t) {
    const uint64_t k = t == 0 ? gid : tail0 + gid;
    if ((t == 0 && k < head) || (t == 1 && k < n)) {
      uint2 pr = pairs[k];
      uint32_t s = pr.x, d = pr.y;
      if (normalize<PREFIX>(G, s, d)) set_pair_generic<MODE>(G, s, d, cube, lo, span);
      else ++skip;
    }
  }
  const uint4* p4 = reinterpret_cast<const uint4*>(pairs + head);
  for (uint64_t i = gid; i < n8; i += stride) {
    uint4 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = __ldcs(p4 + 4 * i + q);
    uint32_t ss[8] = {v[0].x, v[0].z, v[1].x, v[1].z, v[2].x, v[2].z, v[3].x, v[3].z};
    uint32_t dd[8] = {v[0].y, v[0].w, v[1].y, v[1].w, v[2].y, v[2].w, v[3].y, v[3].w};
    if (NRA) {
      set_quad<(NRA ? NRA : 1), NVA, MODE, PREFIX>(G, ss, dd, cube, lo, span, skip);
      set_quad<(NRA ? NRA : 1), NVA, MODE, PREFIX>(G, ss + 4, dd + 4, cube, lo, span, skip);
    } else {
      for (int p = 0; p < 8; ++p) {
        if (normalize<PREFIX>(G, ss[p], dd[p])) set_pair_generic<MODE>(G, ss[p], dd[p], cube, lo, span);
        else ++skip;
      }
    }
  }
  if (PREFIX && skipped) {
    skip = warp_sum(skip);
    if ((threadIdx.x & 31) == 0 && skip) atomicAdd(skipped, (unsigned long long)skip);
  }
}

// ---------------------------------------------------------------- reset / merge
__global__ void __launch_bounds__(kThreads) k_zero(uint4* __restrict__ p, uint64_t n16) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride)
    p[i] = make_uint4(0, 0, 0, 0);
}

struct MergeSrcs {
  const uint4* p[16];
  int k;
};

// dst |= src[0] | … | src[k−1] over n16 16-byte words ("bits OR").
__global__ void __launch_bounds__(kThreads) k_or_merge(uint4* __restrict__ dst, const __grid_constant__ MergeSrcs S,
                                                       uint64_t n16) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
    uint4 a = dst[i];
    for (int j = 0; j < S.k; ++j) {
      uint4 b = __ldcs(S.p[j] + i);
      a.x |= b.x;
      a.y |= b.y;
      a.z |= b.z;
      a.w |= b.w;
    }
    dst[i] = a;
  }
}

// ---------------------------------------------------------------- window-end detect
// Per-CS window math in fp64 (Q12, Thm. 1, θ_bn P:261 / Q15, Q16).
__device__ void cs_math(const Geo& G, uint64_t ztot, uint32_t theta, cbaa_cs_stats* rec) {
  const double g = (double)G.g;
  const double bits0 = (double)G.ncols[0] * g;
  double eta = ztot == 0 ? (double)INFINITY : -bits0 * log((double)ztot / bits0);
  double eps = 1.0;
  for (uint32_t i = 0; i < G.narr; ++i) eps *= 1.0 - exp(-eta / ((double)G.ncols[i] * g));
  const double cap = 1.0 - 9.5367431640625e-07;   // 1 − 2^−20
  if (eps > cap) eps = cap;
  double tbn = G.theta_formula == CBAA_THETA_PAPER ? g * (1.0 + eps) * exp(-(double)theta / g) - g * eps
                                                   : g * (1.0 - eps) * exp(-(double)theta / g);
  if (tbn < 0.0) tbn = 0.0;
  // Alg. 3's union-column threshold (Q20): θ_bn as written, or θ_uc = g(1−ε)e^{−θ/g}, the Thm. 2
  // estimate solved for Z so that a candidate is accepted iff its estimate reaches θ (Def. 1)
  double tuc = G.union_threshold == CBAA_UNION_THM2 ? g * (1.0 - eps) * exp(-(double)theta / g) : tbn;
  if (tuc < 0.0) tuc = 0.0;
  auto zfloor = [&](double t) {
    const double f = floor(t);
    return f < 0.0 ? 0u : (f > g ? G.g : (uint32_t)f);
  };
  rec->ztot = ztot;
  rec->eta = eta;
  rec->eps = eps;
  rec->theta_bn = tbn;
  rec->zmax = zfloor(tbn);
  rec->theta_uc = tuc;
  rec->zmax_uc = zfloor(tuc);
}

struct DetectScratch {
  uint32_t* zc;                 // [n_cs][ra_cols]
  uint32_t* hc;                 // [n_cs][ra_cols], first n_hot[i] of each RA(i) block valid
  cbaa_cs_stats* rec;           // [n_cs]
  unsigned int* done;           // [n_cs] CTA arrival counters
  unsigned int* done_all;       // [1]
  unsigned long long* prefix;   // [n_range + 1] prefix of the work units of k_tuples (0 for overflowed CSs)
  unsigned long long* units;    // [n_cs] work units per CS: tuples (Cartesian) or |HC(0)|·|HC(1)| (join)
  unsigned long long* n_hits;   // [1]
  cbaa_host* hits;              // [hit_cap]
  uint32_t hit_cap;
  unsigned long long* n_cand;   // [1]   candidate recording (debug)
  unsigned long long* cand;     // [cand_cap]
  uint64_t cand_cap;
  unsigned long long* n_join;   // [1]   CP-consistent chains found by k_join3 (may exceed join_cap)
  unsigned long long* join;     // [join_cap] (cs << 32 | lp) of each chain, consumed by k_union
  uint64_t join_cap;
};

// Block-wide exclusive prefix sum of one value per thread; returns the block total in *total.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* s_warp, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  uint32_t before = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kDetWarps; ++w) {
    uint32_t c = s_warp[w];
    before += w < warp ? c : 0u;
    tot += c;
  }
  __syncthreads();
  *total = tot;
  return before + incl - v;
}

// Per-detect counters, zeroed by CTA 0 of the zero-count kernel (everything that uses them runs in later
// graph nodes): the k_hot arrival counters, the chain/candidate counters and the result-block head.
__device__ __forceinline__ void zero_detect_counters(const DetectScratch& D, uint32_t cs_lo, uint32_t n_range) {
  for (uint32_t k = threadIdx.x; k < n_range; k += blockDim.x) D.done[cs_lo + k] = 0;
  if (threadIdx.x == 0) {
    *D.done_all = 0;
    *D.n_cand = 0;
    *D.n_join = 0;
    D.n_hits[0] = 0;
    D.n_hits[1] = 0;   // result-block slot for the chain count (written by k_union)
  }
}

// ---------------------------------------------------------------- TMA bulk-copy helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_addr(b)), "r"(parity) : "memory");
  }
}
// 1-D bulk copy global → shared (TMA engine), completion counted on the mbarrier; bytes % 16 == 0.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(b)), "l"(0x12F0000000000000ull)   // evict_first
               : "memory");
}

// Zero counts for g = 4096 (a column = 512 B) streamed by the TMA engine: the RA block of a CS is
// contiguous, so it is cut into 8 KiB tiles of 16 columns; persistent CTAs run a kStages-deep
// cp.async.bulk + mbarrier pipeline and each warp popcounts 4 columns of a tile out of shared memory.
// The copies need no registers, so far more bytes are in flight than with register loads.
constexpr int kZcStages = 4;
constexpr uint32_t kZcTileCols = 16;
__global__ void __launch_bounds__(kDetThreads) k_zero_counts_tma(const __grid_constant__ Geo G,
                                                                 const uint32_t* __restrict__ cube,
                                                                 const __grid_constant__ DetectScratch D,
                                                                 uint32_t cs_lo, uint32_t n_range, int finish) {
  __shared__ __align__(128) uint4 tile[kZcStages][kZcTileCols * 32];   // 16 columns × 512 B per stage
  __shared__ __align__(8) uint64_t bar[kZcStages];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t tiles_per_cs = G.ra_cols / kZcTileCols;
  const uint64_t n_tiles = (uint64_t)n_range * tiles_per_cs;
  if (finish && blockIdx.x == 0) zero_detect_counters(D, cs_lo, n_range);
  if (threadIdx.x == 0) {
    for (int k = 0; k < kZcStages; ++k) mbar_init(&bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](uint64_t t, int st) {
    const uint32_t cs = cs_lo + (uint32_t)(t / tiles_per_cs);
    const uint32_t col0 = (uint32_t)(t % tiles_per_cs) * kZcTileCols;   // column index within the RA block
    const uint32_t* src = cube + (size_t)cs * G.cs_words + ((size_t)col0 << G.wpc_log2);
    mbar_expect_tx(&bar[st], kZcTileCols * 512);
    bulk_load(tile[st], src, kZcTileCols * 512, &bar[st]);
  };
  uint64_t t = blockIdx.x;
  if (threadIdx.x == 0)
    for (int k = 0; k < kZcStages; ++k)
      if (t + (uint64_t)k * gridDim.x < n_tiles) issue(t + (uint64_t)k * gridDim.x, k);
  for (uint32_t it = 0; t < n_tiles; t += gridDim.x, ++it) {
    const int st = it % kZcStages;
    mbar_wait(&bar[st], (it / kZcStages) & 1);
    const uint32_t cs = cs_lo + (uint32_t)(t / tiles_per_cs);
    const uint32_t col0 = (uint32_t)(t % tiles_per_cs) * kZcTileCols;
#pragma unroll
    for (int k = 0; k < (int)kZcTileCols / kDetWarps; ++k) {
      const uint32_t c = warp * (kZcTileCols / kDetWarps) + k;
      const uint4 v = tile[st][c * 32 + lane];
      const uint32_t pop = warp_sum(__popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w));
      if (lane == 0) D.zc[(size_t)cs * G.ra_cols + col0 + c] = G.g - pop;   // zero bits
    }
    __syncthreads();   // the whole tile has been read: refill this stage
    if (threadIdx.x == 0 && t + (uint64_t)kZcStages * gridDim.x < n_tiles) issue(t + (uint64_t)kZcStages * gridDim.x, st);
  }
}

// Zero counts of every RA column of CSs [cs_lo, cs_lo + n_range) (Alg. 2 input) and the per-CS
// RA(0) totals Ztot (η source, Q12).  Persistent grid; a warp takes 16 columns of one (cs, RA i) at a
// time and keeps all 16 column loads in flight (VEC: one 16-B load per lane per column, g = 4096).
template <bool VEC>
__global__ void __launch_bounds__(kDetThreads) k_zero_counts(const __grid_constant__ Geo G,
                                                          const uint32_t* __restrict__ cube,
                                                          const __grid_constant__ DetectScratch D, uint32_t cs_lo,
                                                          uint32_t n_range, int finish) {
  constexpr uint32_t kGroup = 16;
  const int lane = threadIdx.x & 31;
  uint32_t gpc = 0;   // column groups per CS
  for (uint32_t i = 0; i < G.num_ra; ++i) gpc += (G.ncols[i] + kGroup - 1) / kGroup;
  const uint64_t total = (uint64_t)n_range * gpc;
  if (finish && blockIdx.x == 0) zero_detect_counters(D, cs_lo, n_range);
  const uint64_t n_warps = ((uint64_t)gridDim.x * kDetThreads) >> 5;
  for (uint64_t gi = ((uint64_t)blockIdx.x * kDetThreads + threadIdx.x) >> 5; gi < total; gi += n_warps) {
    const uint32_t cs = cs_lo + (uint32_t)(gi / gpc);
    uint32_t rem = (uint32_t)(gi % gpc), i = 0;
    for (;; ++i) {
      const uint32_t gi_i = (G.ncols[i] + kGroup - 1) / kGroup;
      if (rem < gi_i) break;
      rem -= gi_i;
    }
    const uint32_t c0 = rem * kGroup, c1 = min(c0 + kGroup, G.ncols[i]);
    const uint32_t* arr = cube + (size_t)cs * G.cs_words + G.arr_off[i];
    uint32_t pop[kGroup];
    if (VEC) {
      uint4 v[kGroup];
#pragma unroll
      for (uint32_t k = 0; k < kGroup; ++k)
        v[k] = c0 + k < c1 ? __ldcs(reinterpret_cast<const uint4*>(arr + ((size_t)(c0 + k) << G.wpc_log2)) + lane)
                           : make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
#pragma unroll
      for (uint32_t k = 0; k < kGroup; ++k) pop[k] = __popc(v[k].x) + __popc(v[k].y) + __popc(v[k].z) + __popc(v[k].w);
    } else {
#pragma unroll
      for (uint32_t k = 0; k < kGroup; ++k) {
        pop[k] = 0;
        if (c0 + k < c1)
          for (uint32_t w = lane; w < G.wpc; w += 32) pop[k] += __popc(__ldcs(arr + ((size_t)(c0 + k) << G.wpc_log2) + w));
      }
    }
    // lane k ends up holding the population of column c0 + k (transpose-reduce of 16 warp sums)
    uint32_t mine = 0;
#pragma unroll
    for (uint32_t k = 0; k < kGroup; ++k) {
      const uint32_t t = warp_sum(pop[k]);
      if (lane == (int)k) mine = t;
    }
    if (lane < (int)(c1 - c0)) D.zc[(size_t)cs * G.ra_cols + G.ra_off[i] + c0 + lane] = G.g - mine;
  }
}

// One CTA per (cs, RA i) of the range, after k_zero_counts: the per-CS fp64 math (every CTA of the CS
// computes the same values; RA(0)'s CTA records them), the ordered Alg. 2 compaction of HC(i), and — in
// the last CTA of the CS — ∏|HC(i)|, the overflow flag and the work units of the Alg. 3 kernel; the last
// CS overall writes the prefix of those units.
__global__ void __launch_bounds__(kDetThreads) k_hot(const __grid_constant__ Geo G, const __grid_constant__ DetectScratch D,
                                                  uint32_t cs_lo, uint32_t n_range, uint32_t theta, int join) {
  __shared__ uint32_t s_warp[kDetWarps];
  __shared__ int s_last, s_last_all;
  __shared__ uint32_t s_zmax;
  const uint32_t cs = cs_lo + blockIdx.x / G.num_ra;
  const uint32_t a = blockIdx.x % G.num_ra;
  cbaa_cs_stats* rec = D.rec + cs;
  // Ztot = zero bits of RA(0) of this CS (η source, Q12): every CTA of the CS sums the same c(0) counts
  __shared__ unsigned long long s_zsum[kDetWarps];
  unsigned long long zpart = 0;
  const uint32_t* z0 = D.zc + (size_t)cs * G.ra_cols;   // RA(0) block
  for (uint32_t c = threadIdx.x; c < G.ncols[0]; c += kDetThreads) zpart += __ldcg(z0 + c);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) zpart += __shfl_xor_sync(0xffffffffu, zpart, o);
  if ((threadIdx.x & 31) == 0) s_zsum[threadIdx.x >> 5] = zpart;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long ztot = 0;
    for (int w = 0; w < kDetWarps; ++w) ztot += s_zsum[w];
    cbaa_cs_stats st;
    cs_math(G, ztot, theta, &st);
    if (a == 0) {
      rec->ztot = st.ztot;
      rec->eta = st.eta;
      rec->eps = st.eps;
      rec->theta_bn = st.theta_bn;
      rec->zmax = st.zmax;
      rec->theta_uc = st.theta_uc;
      rec->zmax_uc = st.zmax_uc;
      rec->candidates = 0;   // accumulated by the Alg. 3 kernels, which run after this grid
      rec->hits = 0;
    }
    s_zmax = st.zmax;
  }
  __syncthreads();
  const uint32_t zmax = s_zmax;
  const uint32_t* za = D.zc + (size_t)cs * G.ra_cols + G.ra_off[a];
  uint32_t* ha = D.hc + (size_t)cs * G.ra_cols + G.ra_off[a];
  constexpr uint32_t kPer = 16;                        // columns per thread per tile, held in registers
  uint32_t written = 0;
  for (uint32_t t0 = 0; t0 < G.ncols[a]; t0 += kDetThreads * kPer) {
    const uint32_t my0 = t0 + threadIdx.x * kPer;
    uint32_t z[kPer];
#pragma unroll
    for (uint32_t k = 0; k < kPer; ++k) z[k] = my0 + k < G.ncols[a] ? __ldcg(za + my0 + k) : 0xffffffffu;
    uint32_t flags = 0;
#pragma unroll
    for (uint32_t k = 0; k < kPer; ++k) flags |= (z[k] <= zmax ? 1u : 0u) << k;   // P:272, Q16
    uint32_t tot;
    uint32_t off = written + block_exclusive_scan(__popc(flags), s_warp, &tot);
    while (flags) {
      int k = __ffs(flags) - 1;
      flags &= flags - 1;
      ha[off++] = my0 + k;
    }
    written += tot;
  }
  if (threadIdx.x == 0) {
    rec->n_hot[a] = written;
    __threadfence();
    unsigned int old = atomicAdd(D.done + cs, 1u);
    s_last = old == G.num_ra - 1;
  }
  __syncthreads();
  if (!s_last) return;
  // ---- last CTA of this CS: tuple space and work units
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned long long prod = 1;
    for (uint32_t i = 0; i < G.num_ra; ++i) {
      const uint32_t n = __ldcg(&rec->n_hot[i]);
      prod = (n != 0 && prod > ~0ull / n) ? ~0ull : prod * n;   // saturating ∏|HC(i)|
    }
    rec->tuples = prod;
    rec->overflow = prod > G.tuple_cap ? 1 : 0;
    // work units of the Alg. 3 kernel: every tuple (Cartesian) or every (hc0, hc1) pair (join)
    // (an empty HC(i) makes the tuple space empty: no units, the join would only enumerate dead pairs)
    D.units[cs] = (rec->overflow || prod == 0)
                      ? 0ull
                      : (join ? (unsigned long long)__ldcg(&rec->n_hot[0]) * __ldcg(&rec->n_hot[1]) : prod);
    __threadfence();
    unsigned int old = atomicAdd(D.done_all, 1u);
    s_last_all = old == n_range - 1;   // a second flag: other warps may still be reading s_last
  }
  __syncthreads();
  if (!s_last_all) return;
  // ---- last CS overall: exclusive prefix of the work units over the range
  __threadfence();
  const uint32_t per = (n_range + kDetThreads - 1) / kDetThreads;
  const uint32_t b0 = min(threadIdx.x * per, n_range), b1 = min(b0 + per, n_range);
  unsigned long long loc = 0;
  for (uint32_t k = b0; k < b1; ++k) loc += __ldcg(D.units + cs_lo + k);
  __shared__ unsigned long long s_scan[kDetThreads];
  s_scan[threadIdx.x] = loc;
  __syncthreads();
  for (int o = 1; o < kDetThreads; o <<= 1) {   // Hillis-Steele inclusive scan
    unsigned long long v = threadIdx.x >= o ? s_scan[threadIdx.x - o] : 0ull;
    __syncthreads();
    s_scan[threadIdx.x] += v;
    __syncthreads();
  }
  unsigned long long run = s_scan[threadIdx.x] - loc;
  for (uint32_t k = b0; k < b1; ++k) {
    D.prefix[k] = run;
    run += __ldcg(D.units + cs_lo + k);
  }
  if (threadIdx.x == kDetThreads - 1) D.prefix[n_range] = s_scan[kDetThreads - 1];
}

// Union-column test of one candidate by the whole warp (Alg. 3) and its output.
// All lanes call it with the same (cs, lp, ra_cols); lane 0 records the result.
template <int NRA>
__device__ __forceinline__ void union_check(const Geo& G, const uint32_t* __restrict__ cube,
                                            const DetectScratch& D, uint32_t cs, uint32_t lp, const uint32_t* ra_cols,
                                            int record) {
  const int lane = threadIdx.x & 31;
  const int nra = NRA ? NRA : (int)G.num_ra;
  const uint32_t* csb = cube + (size_t)cs * G.cs_words;
  const uint32_t* colp[CBAA_MAX_ARRAYS];
#pragma unroll
  for (int i = 0; i < (NRA ? NRA : CBAA_MAX_RA); ++i)
    if (i < nra) colp[i] = csb + G.arr_off[i] + ((size_t)ra_cols[i] << G.wpc_log2);
  for (uint32_t j = 0; j < G.num_va; ++j) {
    uint32_t a = nra + j;
    uint32_t c = mix32(lp ^ G.va_seeds[j]) & G.colmask[a];                // H_j(LP)
    colp[a] = csb + G.arr_off[a] + ((size_t)c << G.wpc_log2);
  }
  uint32_t pop = 0;
  if (NRA == 3 && G.num_va == 1) {   // paper shape: four columns held in registers
    const uint32_t *p0 = colp[0], *p1 = colp[1], *p2 = colp[2], *p3 = colp[3];
    for (uint32_t w = lane; w < G.wpc; w += 32)
      pop += __popc(__ldcg(p0 + w) & __ldcg(p1 + w) & __ldcg(p2 + w) & __ldcg(p3 + w));   // UCol
  } else {
    for (uint32_t w = lane; w < G.wpc; w += 32) {
      uint32_t v = 0xffffffffu;
      for (uint32_t a = 0; a < G.narr; ++a) v &= __ldcg(colp[a] + w);     // UCol AND
      pop += __popc(v);
    }
  }
  pop = warp_sum(pop);
  if (lane == 0) {
    cbaa_cs_stats* rec = D.rec + cs;
    const uint32_t z = G.g - pop;
    atomicAdd(reinterpret_cast<unsigned long long*>(&rec->candidates), 1ull);
    if (record) {
      unsigned long long k = atomicAdd(D.n_cand, 1ull);
      if (k < D.cand_cap) D.cand[k] = ((unsigned long long)cs << 32) | lp;
    }
    if (z <= rec->zmax_uc) {   // reject iff zero bits > θ_bn (Q16), or > θ_uc (Q20 option)
      atomicAdd(reinterpret_cast<unsigned long long*>(&rec->hits), 1ull);
      unsigned long long k = atomicAdd(D.n_hits, 1ull);
      if (k < D.hit_cap) {
        const double g = (double)G.g;
        double est = z == 0 ? (double)INFINITY : -g * log((double)z / (g - g * rec->eps));   // Thm. 2
        if (est < 0.0) est = 0.0;
        cbaa_host h;
        h.ip = G.inv_a * (((lp << G.r) | cs) - G.mangle_b);      // unmangle
        h.cs = cs;
        h.lp = lp;
        h.z = z;
        h.estimate = est;
        D.hits[k] = h;
      }
    }
  }
}

// Alg. 3 over the whole tuple space of the range.  One lane per tuple for the CP check
// and LP assembly; passing tuples are then checked one at a time by the
// whole warp: AND of the |RA|+|VA| columns, popcount, Z ≤ zmax.
template <int NRA>
__global__ void __launch_bounds__(kDetThreads) k_tuples(const __grid_constant__ Geo G, const uint32_t* __restrict__ cube,
                                                     const __grid_constant__ DetectScratch D, uint32_t cs_lo,
                                                     uint32_t n_range, int record) {
  const int lane = threadIdx.x & 31;
  const int nra = NRA ? NRA : (int)G.num_ra;
  const unsigned long long total = __ldcg(D.prefix + n_range);
  const uint64_t warp_id = ((uint64_t)blockIdx.x * kDetThreads + threadIdx.x) >> 5;
  const uint64_t n_warps = ((uint64_t)gridDim.x * kDetThreads) >> 5;
  const uint32_t Lmask = G.L == 32 ? 0xffffffffu : ((1u << G.L) - 1u);
  for (uint64_t t0 = warp_id * 32; t0 < total; t0 += n_warps * 32) {
    const uint64_t t = t0 + lane;
    bool pass = false;
    uint32_t cs_rel = 0, lp = 0;
    uint32_t cols[NRA ? NRA : CBAA_MAX_RA];
    if (t < total) {
      // CS of tuple t: last k with prefix[k] ≤ t (binary search; empty CSs have equal prefixes)
      uint32_t lo = 0, hi = n_range;
      while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (__ldg(D.prefix + mid) <= t) lo = mid;
        else hi = mid;
      }
      cs_rel = lo;
      const uint32_t cs = cs_lo + cs_rel;
      const cbaa_cs_stats* rec = D.rec + cs;
      uint64_t u = t - __ldg(D.prefix + cs_rel);
      const uint32_t* hcs = D.hc + (size_t)cs * G.ra_cols;
      if (total <= 0xffffffffull) {   // 32-bit mixed radix (the common case: tuple_cap ≤ 2^32)
        uint32_t u32 = (uint32_t)u;
#pragma unroll
        for (int i = (NRA ? NRA : CBAA_MAX_RA) - 1; i >= 0; --i) {   // last index fastest
          if (i < nra) {
            uint32_t nh = __ldg(&rec->n_hot[i]);
            uint32_t q = u32 / nh;
            cols[i] = __ldg(hcs + G.ra_off[i] + (u32 - q * nh));
            u32 = q;
          }
        }
      } else {
#pragma unroll
        for (int i = (NRA ? NRA : CBAA_MAX_RA) - 1; i >= 0; --i) {
          if (i < nra) {
            uint32_t nh = __ldg(&rec->n_hot[i]);
            uint64_t q = u / nh;
            cols[i] = __ldg(hcs + G.ra_off[i] + (uint32_t)(u - q * nh));
            u = q;
          }
        }
      }
      pass = true;
#pragma unroll
      for (int i = 0; i < (NRA ? NRA : CBAA_MAX_RA); ++i) {
        if (i < nra) {
          const int nx = (i + 1 == nra) ? 0 : i + 1;
          uint32_t low = cols[i] & ((1u << G.cp[i]) - 1u);                 // CP of hc_i
          uint32_t top = cols[nx] >> (G.cbn[nx] - G.cp[i]);               // first |CP(i)| bits of hc_{i+1}
          pass &= low == top;
          // EP(i) = high |EP(i)| bits of hc_i, at LP offsets clbs(i).. (mod L), MSB-first
          uint64_t x = (uint64_t)(cols[i] >> G.cp[i]) << (2 * G.L - G.clbs[i] - G.ep[i]);
          lp |= (uint32_t)((x >> G.L) | x) & Lmask;
        }
      }
    }
    unsigned int m = __ballot_sync(0xffffffffu, pass);
    while (m) {
      const int srcl = __ffs(m) - 1;
      m &= m - 1;
      const uint32_t c_cs = cs_lo + __shfl_sync(0xffffffffu, cs_rel, srcl);
      const uint32_t c_lp = __shfl_sync(0xffffffffu, lp, srcl);
      uint32_t c_cols[NRA ? NRA : CBAA_MAX_RA];
#pragma unroll
      for (int i = 0; i < (NRA ? NRA : CBAA_MAX_RA); ++i)
        c_cols[i] = __shfl_sync(0xffffffffu, i < nra ? cols[i] : 0u, srcl);
      union_check<NRA>(G, cube, D, c_cs, c_lp, c_cols, record);
    }
  }
}

// First index in the ascending list a[0..n) whose value is ≥ key.
__device__ __forceinline__ uint32_t lower_bound(const uint32_t* __restrict__ a, uint32_t n, uint32_t key) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Alg. 3 for |RA| = 3, first half, as a range join.  HC(i) lists are ascending, so the hc_{i+1} whose
// first |CP(i)| bits equal the last |CP(i)| bits of hc_i (Q19) form one contiguous run, found by
// binary search.  One lane per (hc0, hc1) pair: CP(0) check, then the run of HC(2) matching CP(1), each
// checked against the wrap condition CP(2) with hc0; every passing chain's LP is appended to
// D.join.  The chain set is exactly the CP-passing tuples of the Cartesian product the oracle
// enumerates, but only CP-consistent chains are visited (~n² instead of n³ work).
__global__ void __launch_bounds__(kDetThreads) k_join3(const __grid_constant__ Geo G, const __grid_constant__ DetectScratch D,
                                                    uint32_t cs_lo, uint32_t n_range) {
  const int lane = threadIdx.x & 31;
  const unsigned long long total = __ldcg(D.prefix + n_range);
  const uint64_t stride = (uint64_t)gridDim.x * kDetThreads;
  const uint32_t Lmask = G.L == 32 ? 0xffffffffu : ((1u << G.L) - 1u);
  for (uint64_t base = (uint64_t)blockIdx.x * kDetThreads + (threadIdx.x & ~31u); base < total; base += stride) {
    const uint64_t t = base + lane;
    bool active = false;
    uint32_t cs = 0, hc0 = 0, hc1 = 0, j = 0, jend = 0;
    const uint32_t* hc2list = nullptr;
    if (t < total) {
      uint32_t lo = 0, hi = n_range;   // CS of pair t: last k with prefix[k] ≤ t
      while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (__ldg(D.prefix + mid) <= t) lo = mid;
        else hi = mid;
      }
      cs = cs_lo + lo;
      const cbaa_cs_stats* rec = D.rec + cs;
      const uint32_t n1 = __ldg(&rec->n_hot[1]);
      const uint32_t n2 = __ldg(&rec->n_hot[2]);
      const uint64_t u = t - __ldg(D.prefix + lo);   // < |HC(0)|·|HC(1)|, which can pass 2^32
      const uint32_t* hcs = D.hc + (size_t)cs * G.ra_cols;
      const uint64_t q = u / n1;
      hc0 = __ldg(hcs + G.ra_off[0] + (uint32_t)q);
      hc1 = __ldg(hcs + G.ra_off[1] + (uint32_t)(u - q * n1));
      hc2list = hcs + G.ra_off[2];
      // CP(0): low cp0 bits of hc0 == top cp0 bits of hc1
      if ((hc0 & ((1u << G.cp[0]) - 1u)) == (hc1 >> (G.cbn[1] - G.cp[0]))) {
        const uint32_t v = hc1 & ((1u << G.cp[1]) - 1u);     // CP(1) selects the run of HC(2)
        const uint32_t sh = G.cbn[2] - G.cp[1];
        j = lower_bound(hc2list, n2, v << sh);
        jend = G.cp[1] == 0 ? n2 : lower_bound(hc2list, n2, (v + 1) << sh);
        active = j < jend;
      }
    }
    // LP bits contributed by hc0 and hc1; hc2 adds its EP per chain
    uint32_t lp01 = 0;
    {
      const uint32_t c01[2] = {hc0, hc1};
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        uint64_t x = (uint64_t)(c01[i] >> G.cp[i]) << (2 * G.L - G.clbs[i] - G.ep[i]);
        lp01 |= (uint32_t)((x >> G.L) | x) & Lmask;
      }
    }
    const uint32_t top0 = hc0 >> (G.cbn[0] - G.cp[2]);
    for (; active; ++j) {
      active = j + 1 < jend;
      const uint32_t hc2 = __ldg(hc2list + j);
      if ((hc2 & ((1u << G.cp[2]) - 1u)) == top0) {                  // CP(2), the wrap
        uint64_t x = (uint64_t)(hc2 >> G.cp[2]) << (2 * G.L - G.clbs[2] - G.ep[2]);
        const uint32_t lp = lp01 | ((uint32_t)((x >> G.L) | x) & Lmask);
        unsigned long long k = atomicAdd(D.n_join, 1ull);
        if (k < D.join_cap) D.join[k] = ((unsigned long long)cs << 32) | lp;
      }
    }
  }
}

// Alg. 3, second half: one warp per chain of D.join — the RA columns are the LP's own extraction
// (Alg. 1, the round trip lpFromTuple ∘ raColumnIndex = id), the VA columns H_j(LP).
__global__ void __launch_bounds__(kDetThreads) k_union(const __grid_constant__ Geo G, const uint32_t* __restrict__ cube,
                                                    const __grid_constant__ DetectScratch D, int record) {
  const unsigned long long n_all = __ldcg(D.n_join);
  const unsigned long long n = min(n_all, (unsigned long long)D.join_cap);
  if (blockIdx.x == 0 && threadIdx.x == 0) D.n_hits[1] = n_all;   // lets the host see a join-buffer overflow
  const uint64_t warp_id = ((uint64_t)blockIdx.x * kDetThreads + threadIdx.x) >> 5;
  const uint64_t n_warps = ((uint64_t)gridDim.x * kDetThreads) >> 5;
  for (uint64_t k = warp_id; k < n; k += n_warps) {
    const unsigned long long e = __ldcg(D.join + k);
    const uint32_t cs = (uint32_t)(e >> 32), lp = (uint32_t)e;
    const uint64_t dbl = ((uint64_t)lp << G.L) | lp;
    uint32_t cols[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) cols[i] = (uint32_t)(dbl >> G.sh[i]) & G.colmask[i];
    union_check<3>(G, cube, D, cs, lp, cols, record);
  }
}

// Output order of S:418 (estimate descending, then ip ascending) on the device: one CTA bitonic-sorts up to
// kSortMax hits in shared memory, so the host copies them out already ordered.  More hits: left to the
// host (the library sorts there).
constexpr int kSortMax = 2048;
__global__ void __launch_bounds__(1024) k_sort_hits(const __grid_constant__ DetectScratch D) {
  __shared__ unsigned long long s_est[kSortMax];
  __shared__ uint32_t s_ip[kSortMax];
  __shared__ uint16_t s_idx[kSortMax];
  const unsigned long long n = min(*D.n_hits, (unsigned long long)D.hit_cap);
  if (n <= 1 || n > (unsigned long long)kSortMax) return;
  uint32_t m = 1;
  while (m < n) m <<= 1;
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
    const bool v = i < n;
    // estimates are ≥ 0 (or +inf): their IEEE bits order like the values
    s_est[i] = v ? (unsigned long long)__double_as_longlong(D.hits[i].estimate) : 0ull;
    s_ip[i] = v ? D.hits[i].ip : 0xffffffffu;
    s_idx[i] = (uint16_t)i;
  }
  __syncthreads();
  // "before(a, b)": a comes first in the output; padding (index ≥ n) always last
  auto before = [&](uint32_t a, uint32_t b) {
    const bool va = s_idx[a] < n, vb = s_idx[b] < n;
    if (va != vb) return va;
    return s_est[a] != s_est[b] ? s_est[a] > s_est[b] : s_ip[a] < s_ip[b];
  };
  for (uint32_t k = 2; k <= m; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          if (up ? before(l, i) : before(i, l)) {
            unsigned long long te = s_est[i]; s_est[i] = s_est[l]; s_est[l] = te;
            uint32_t ti = s_ip[i]; s_ip[i] = s_ip[l]; s_ip[l] = ti;
            uint16_t tx = s_idx[i]; s_idx[i] = s_idx[l]; s_idx[l] = tx;
          }
        }
      }
      __syncthreads();
    }
  }
  // gather through registers: read every hit first, then write the permuted order
  cbaa_host tmp[2];
  uint32_t cnt = 0;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) tmp[cnt++] = D.hits[s_idx[i]];
  __syncthreads();
  cnt = 0;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) D.hits[i] = tmp[cnt++];
}

// Alg. 1 mapping for the unit parity tests (no cube access).
__global__ void k_debug_map(const __grid_constant__ Geo G, const uint32_t* __restrict__ iip,
                            const uint32_t* __restrict__ oip, uint64_t n, uint32_t* __restrict__ cs_out,
                            uint32_t* __restrict__ cols_out, uint32_t* __restrict__ row_out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    uint32_t mi = G.mangle_a * iip[k] + G.mangle_b;
    uint32_t mo = G.mangle_a * oip[k] + G.mangle_b;
    uint32_t lp = mi >> G.r;
    uint64_t dbl = ((uint64_t)lp << G.L) | lp;
    cs_out[k] = mi & G.rmask;
    row_out[k] = mix32(mo ^ G.bv_seed) & (G.g - 1);
    for (uint32_t i = 0; i < G.num_ra; ++i) cols_out[k * G.narr + i] = (uint32_t)(dbl >> G.sh[i]) & G.colmask[i];
    for (uint32_t j = 0; j < G.num_va; ++j)
      cols_out[k * G.narr + G.num_ra + j] = mix32(lp ^ G.va_seeds[j]) & G.colmask[G.num_ra + j];
  }
}

}  // namespace cbaa

namespace cbaa {
// ---------------------------------------------------------------- window-end exchange across GPUs
// Signal area of a cube allocation (after the cube, 256-B aligned): u64 epoch[kMaxRanks] written by the
// peers (slot k by rank k) + u32 status (non-zero: a barrier timed out).
constexpr int kMaxRanks = 64;
constexpr uint64_t kSigBytes = 4096;

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct PeerSigs {
  unsigned long long* sig[kMaxRanks];   // rank k's signal area as mapped here (NVLink P2P / IPC)
};

// Device-side barrier of the routers' streams: every prior kernel on this stream has finished (stream
// order) and its cube writes are made visible system-wide, then rank `rank` writes `epoch` into slot
// `rank` of every peer's signal area and waits until every peer has written it into its own.  One CTA;
// gives up after timeout_ns (status := 1) instead of spinning forever.
__global__ void k_peer_barrier(const __grid_constant__ PeerSigs P, int world, int rank, unsigned long long epoch,
                               unsigned long long timeout_ns, uint32_t* status) {
  __threadfence_system();
  __syncthreads();
  const int t = threadIdx.x;
  if (t < world) st_release_sys(P.sig[t] + rank, epoch);
  if (t < world) {
    const unsigned long long* mine = P.sig[rank] + t;
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_sys(mine) < epoch) {
      if (globaltimer() - t0 > timeout_ns) {
        atomicExch(status, 1u);
        break;
      }
      __nanosleep(256);
    }
  }
  __syncthreads();
}

// Pull-OR of the owner's CS range fused with the window-end zero counts (a8 + a9): one warp per column,
// g = 4096 (a column = 512 B = one 16-B load per lane): own | peer_0 | … | peer_{k−1} is stored back and,
// for RA columns, g − popcount is written to zc — the detect that follows skips its zero-count pass.
// Block 0 also zeroes the per-detect counters (as k_zero_counts does).
__global__ void __launch_bounds__(kDetThreads) k_or_merge_zc(const __grid_constant__ Geo G, uint32_t* __restrict__ cube,
                                                          const __grid_constant__ MergeSrcs S, uint32_t cs_lo,
                                                          uint32_t n_range, const __grid_constant__ DetectScratch D) {
  const int lane = threadIdx.x & 31;
  const uint32_t cols_per_cs = G.cs_words >> G.wpc_log2;
  const uint64_t total = (uint64_t)n_range * cols_per_cs;
  if (blockIdx.x == 0) zero_detect_counters(D, cs_lo, n_range);
  const uint64_t n_warps = ((uint64_t)gridDim.x * kDetThreads) >> 5;
  for (uint64_t c = ((uint64_t)blockIdx.x * kDetThreads + threadIdx.x) >> 5; c < total; c += n_warps) {
    const uint32_t cs = cs_lo + (uint32_t)(c / cols_per_cs), col = (uint32_t)(c % cols_per_cs);
    const uint64_t w0 = (uint64_t)cs * G.cs_words + ((uint64_t)col << G.wpc_log2);
    uint4* dst = reinterpret_cast<uint4*>(cube + w0) + lane;
    uint4 a = *dst;
    const uint64_t off16 = (w0 - (uint64_t)cs_lo * G.cs_words) / 4 + lane;   // slices start at cs_lo
#pragma unroll 4
    for (int j = 0; j < S.k; ++j) {
      const uint4 b = __ldcs(S.p[j] + off16);
      a.x |= b.x, a.y |= b.y, a.z |= b.z, a.w |= b.w;
    }
    *dst = a;
    const uint32_t pop = warp_sum(__popc(a.x) + __popc(a.y) + __popc(a.z) + __popc(a.w));
    if (lane == 0 && col < G.ra_cols) D.zc[(size_t)cs * G.ra_cols + col] = G.g - pop;   // RA blocks come first
  }
}

// NVLS: the switch ORs the same 8 bytes of every rank's buffer (multimem.ld_reduce on a multicast
// address, NVLink SHARP); the owner stores the result into its own cube slice.
__device__ __forceinline__ unsigned long long mc_or(const uint64_t* p) {
  unsigned long long v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.or.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__global__ void k_or_multicast(uint64_t* __restrict__ dst, const uint64_t* __restrict__ mc, uint64_t n8) {
  constexpr int kU = 4;   // independent switch reductions in flight per thread
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (kU - 1) * stride < n8; i += kU * stride) {
    unsigned long long v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) v[u] = mc_or(mc + i + u * stride);
#pragma unroll
    for (int u = 0; u < kU; ++u) dst[i + u * stride] = v[u];
  }
  for (; i < n8; i += stride) dst[i] = mc_or(mc + i);
}
}  // namespace cbaa

namespace cbaa {
// ---------------------------------------------------------------- sparse SketchFile "CBA2"
// Blocks of 2^15 cube bits = 1024 words; one warp per block, lane l owns words [32l, 32l + 32).  A block's
// stream is the LEB128 gaps between its ascending set-bit positions.  The first gap of a lane's segment
// depends on the last set bit of the lanes before it: a warp max-scan of "last set position".
constexpr uint32_t kSparseBlockWords = 1024;
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint32_t leb128_len(uint32_t v) { return 1u + (v >= 128u) + (v >= (1u << 14)) + (v >= (1u << 21)) + (v >= (1u << 28)); }

// Per lane: first/last set position in its segment (−1 if none) and the bytes of the gaps inside it.
struct SparseSeg {
  int32_t first, last;
  uint32_t inner_bytes;
};
__device__ __forceinline__ SparseSeg sparse_seg(const uint32_t* __restrict__ blk, uint32_t nwords, uint32_t lane) {
  SparseSeg s{-1, -1, 0};
  for (uint32_t j = 0; j < 32; ++j) {
    const uint32_t wi = lane * 32 + j;
    uint32_t w = wi < nwords ? blk[wi] : 0u;
    while (w) {
      const int32_t pos = (int32_t)(wi * 32 + (__ffs(w) - 1));
      w &= w - 1;
      if (s.last >= 0) s.inner_bytes += leb128_len((uint32_t)(pos - s.last - 1));
      else s.first = pos;
      s.last = pos;
    }
  }
  return s;
}
// Last set position of the lanes before this one (−1 if none): exclusive max-scan over the warp.
__device__ __forceinline__ int32_t prev_last(int32_t last, uint32_t lane) {
  int32_t v = last;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, v, o);
    if ((int)lane >= o) v = max(v, y);
  }
  const int32_t ex = __shfl_up_sync(0xffffffffu, v, 1);
  return lane == 0 ? -1 : ex;
}

// Pass 1: bytes of each block's stream.
__global__ void k_sparse_size(const uint32_t* __restrict__ cube, uint64_t nwords, uint64_t nblocks,
                              uint32_t* __restrict__ bytes) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t b = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nblocks; b += nw) {
    const uint64_t w0 = b * kSparseBlockWords;
    const uint32_t n = (uint32_t)umin64(kSparseBlockWords, nwords - w0);
    const SparseSeg s = sparse_seg(cube + w0, n, lane);
    const int32_t pl = prev_last(s.last, lane);
    uint32_t my = s.inner_bytes + (s.first >= 0 ? leb128_len((uint32_t)(s.first - pl - 1)) : 0u);
    my = warp_sum(my);
    if (lane == 0) bytes[b] = my;
  }
}

// Exclusive prefix of the block sizes (one CTA of 1024 threads): off[b], off[nblocks] = total.
__global__ void __launch_bounds__(1024) k_sparse_offsets(const uint32_t* __restrict__ bytes, uint64_t nblocks,
                                                         unsigned long long* __restrict__ off) {
  __shared__ unsigned long long s_w[32];
  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint64_t per = (nblocks + 1023) / 1024, b0 = umin64(t * per, nblocks), b1 = umin64(b0 + per, nblocks);
  unsigned long long loc = 0;
  for (uint64_t b = b0; b < b1; ++b) loc += bytes[b];
  unsigned long long incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if ((int)lane >= o) incl += y;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  unsigned long long run = incl - loc, tot = 0;
  for (int w = 0; w < 32; ++w) {
    run += w < (int)warp ? s_w[w] : 0ull;
    tot += s_w[w];
  }
  for (uint64_t b = b0; b < b1; ++b) {
    off[b] = run;
    run += bytes[b];
  }
  if (t == 0) off[nblocks] = tot;
}

// Pass 2: the streams, at off[b] + (bytes of the lanes before) in out.
__global__ void k_sparse_write(const uint32_t* __restrict__ cube, uint64_t nwords, uint64_t nblocks,
                               const unsigned long long* __restrict__ off, uint8_t* __restrict__ out) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t b = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nblocks; b += nw) {
    const uint64_t w0 = b * kSparseBlockWords;
    const uint32_t n = (uint32_t)umin64(kSparseBlockWords, nwords - w0);
    const uint32_t* blk = cube + w0;
    const SparseSeg s = sparse_seg(blk, n, lane);
    int32_t prev = prev_last(s.last, lane);
    const uint32_t my = s.inner_bytes + (s.first >= 0 ? leb128_len((uint32_t)(s.first - prev - 1)) : 0u);
    uint32_t incl = my;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if ((int)lane >= o) incl += y;
    }
    uint8_t* p = out + off[b] + (incl - my);
    for (uint32_t j = 0; j < 32; ++j) {
      const uint32_t wi = lane * 32 + j;
      uint32_t w = wi < n ? blk[wi] : 0u;
      while (w) {
        const int32_t pos = (int32_t)(wi * 32 + (__ffs(w) - 1));
        w &= w - 1;
        uint32_t gap = (uint32_t)(pos - prev - 1);
        while (gap >= 128u) {
          *p++ = (uint8_t)(0x80u | (gap & 0x7Fu));
          gap >>= 7;
        }
        *p++ = (uint8_t)gap;
        prev = pos;
      }
    }
  }
}

// Decode (one thread per block): OR the block's set bits into the cube; a malformed stream (a varint
// past its end, a position past the block) sets *bad.
__global__ void k_sparse_decode(const uint8_t* __restrict__ in, const unsigned long long* __restrict__ off,
                                uint64_t nblocks, uint64_t nwords, uint32_t* __restrict__ cube, uint32_t* bad) {
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nblocks; b += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e = off[b + 1], w0 = b * kSparseBlockWords;
    const uint64_t nbits = umin64(kSparseBlockWords, nwords - w0) * 32;
    uint64_t k = off[b];
    int64_t prev = -1;
    while (k < e) {
      uint64_t gap = 0;
      int shift = 0;
      bool okv = false;
      while (k < e && shift <= 28) {
        const uint8_t byte = in[k++];
        gap |= (uint64_t)(byte & 0x7Fu) << shift;
        shift += 7;
        if (!(byte & 0x80u)) {
          okv = true;
          break;
        }
      }
      const int64_t pos = prev + 1 + (int64_t)gap;
      if (!okv || pos >= (int64_t)nbits) {
        atomicExch(bad, 1u);
        break;
      }
      atomicOr(cube + w0 + (pos >> 5), 1u << (pos & 31));
      prev = pos;
    }
  }
}
}  // namespace cbaa
