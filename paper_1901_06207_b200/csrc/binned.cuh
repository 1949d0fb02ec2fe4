// Binned update (CBAA_UPDATE_BINNED): Alg. 1 with the random bit sets moved on chip.
//
// All |RA|+|VA| bits of one pair sit in the same CS (RP) and in the same row (H_bv(oip)),
// so a pair's bits all fall in one "word group" — word w = row/32 of every column of CS cs — a set of
// Σc(i) cube words (64 KiB at the paper geometry) that fits in shared memory.  The update then runs as
// streaming kernels instead of 4 random L2 accesses per pair:
//   k_bin_count    bin histogram, bins (cs, row >> s), added into global totals     reads 8 B/pair
//   k_bin_starts   exclusive scan of the totals → bin regions, write cursors
//   k_bin_scatter  tile-local counting sort; each bin's run of a tile is appended at that bin's global
//                  cursor (one atomic per tile and bin), so every bin region fills front to back and L2
//                  only ever holds one partial line per bin                     reads 8, writes 4 B/pair
//                  entry = LP << s | (row mod 2^s), s = min(5, r) (fits 32 bits since |LP| = 32 − r)
//                  (CBAA_BIN_SCATTER=wc: k_bin_wc, per-bin 32-B write-combining slots in shared memory instead)
//   k_bin_apply    one CTA per word group: the bits are set in a shared-memory image of the group
//                  (test-and-set, ATOMS.OR only when the bit is still 0), then OR-ed into the cube with
//                  one RED per non-zero word                                      reads 4 B/pair
// The order of entries inside a bin depends on scheduling; the cube does not: it is the same set of bits
// as the direct update's (OR is order-free), so parity is bit-exact.
#pragma once
#include "kernels.cuh"

namespace cbaa {

struct BinGeo {
  uint32_t s;          // row bits kept in an entry, min(5, r)
  uint32_t bpc_log2;   // log2(bins per CS) = log2(g) − s
  uint32_t nbins;      // 2^r · g / 2^s
  uint32_t nblk;       // CTAs of k_bin_scatter (two per SM); CTA j reads pairs [j·per, (j+1)·per)
  uint32_t ncols;      // Σc(i): words of one word group
};

#ifndef CBAA_BIN_THREADS
#define CBAA_BIN_THREADS 256
#endif
#ifndef CBAA_BIN_PPT
#define CBAA_BIN_PPT 32
#endif
#ifndef CBAA_BIN_MINB
#define CBAA_BIN_MINB 2
#endif
constexpr int kBinMinBlocks = CBAA_BIN_MINB;       // k_bin_scatter CTAs per SM (grid = SMs × this)
constexpr int kBinThreads = CBAA_BIN_THREADS;      // k_bin_scatter: two CTAs per SM (128 regs × 512 = the RF);
constexpr int kBinPPT = CBAA_BIN_PPT;              // one 512-thread CTA with 16K-pair tiles measured 9 % slower
constexpr int kBinTile = kBinThreads * kBinPPT;    // 8192 pairs per tile
constexpr int kBinRankBits = 14;                   // key = bin << 14 | rank within the tile
constexpr int kApplyThreads = 256;
constexpr int kApplyUnroll = 8;                    // entries per thread in flight
constexpr int kCountThreads = 1024;
#ifndef CBAA_CUR_STRIDE
#define CBAA_CUR_STRIDE 1
#endif
// bin b's write cursor is cursor[b · kCurStride]; adjacent cursors (stride 1) measured fastest — a warp's
// 32 reservation atomics then go to one L2 line (strides 8 / 32: profiles/r02_scatter_ab.md)
constexpr uint32_t kCurStride = CBAA_CUR_STRIDE;

template <bool PREFIX>
__device__ __forceinline__ bool pair_bin(const Geo& G, const BinGeo& B, uint32_t iip, uint32_t oip, uint32_t& bin,
                                         uint32_t& entry) {
  if (!normalize<PREFIX>(G, iip, oip)) return false;
  const uint32_t mi = G.mangle_a * iip + G.mangle_b;                    // P:175 (Q3)
  const uint32_t mo = G.mangle_a * oip + G.mangle_b;                    // Q2
  const uint32_t row = mix32(mo ^ G.bv_seed) & (G.g - 1);
  bin = ((mi & G.rmask) << B.bpc_log2) | (row >> B.s);                  // (cs, row >> s)
  entry = ((mi >> G.r) << B.s) | (row & ((1u << B.s) - 1u));            // LP and the low row bits
  return true;
}

__device__ __forceinline__ uint32_t vsum(uint4 v) { return v.x + v.y + v.z + v.w; }
// Shared-memory fetch-and-increment on a 32-bit shared address.
__device__ __forceinline__ uint32_t atoms_inc(uint32_t a) {
  uint32_t v;
  asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(v) : "r"(a));
  return v;
}
// Predicated fetch-and-increment (one instruction, no branch): returns 0 when pred == 0.
__device__ __forceinline__ uint32_t atoms_inc_if(uint32_t a, uint32_t pred) {
  uint32_t v = 0;
  asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p atom.shared.add.u32 %0, [%1], 1;\n}"
               : "+r"(v) : "r"(a), "r"(pred));
  return v;
}
// Opaque to the optimizer: keeps a loop-invariant in a register instead of re-reading the parameter bank.
__device__ __forceinline__ uint32_t pin(uint32_t x) {
  asm volatile("" : "+r"(x));
  return x;
}

// Loads the 4 pairs starting at k of a CTA chunk ending at c1 (vector load when the group is whole and
// both arrays are 16-B aligned at the chunk starts).
__device__ __forceinline__ void load_quad(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                                          uint64_t k, uint64_t c1, bool vec, uint32_t* ss, uint32_t* dd, bool* in) {
  if (vec && k + 4 <= c1) {
    const uint4 a = ld_stream4(src + k), b = ld_stream4(dst + k);
    ss[0] = a.x, ss[1] = a.y, ss[2] = a.z, ss[3] = a.w;
    dd[0] = b.x, dd[1] = b.y, dd[2] = b.z, dd[3] = b.w;
    in[0] = in[1] = in[2] = in[3] = true;
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      in[e] = k + e < c1;
      ss[e] = in[e] ? __ldcs(src + k + e) : 0u;
      dd[e] = in[e] ? __ldcs(dst + k + e) : 0u;
    }
  }
}

// Phase 1: bin histogram of each CTA's chunk, added into counts[bin] (zeroed by k_bin_starts).
template <bool PREFIX>
__global__ void __launch_bounds__(kCountThreads) k_bin_count(const __grid_constant__ Geo G, const __grid_constant__ BinGeo B,
                                                           const uint32_t* __restrict__ src,
                                                           const uint32_t* __restrict__ dst, uint64_t n, uint64_t per,
                                                           int vec, uint32_t* __restrict__ counts,
                                                           unsigned long long* __restrict__ skipped) {
  extern __shared__ uint32_t hist[];
  for (uint32_t b = threadIdx.x; b < B.nbins; b += kCountThreads) hist[b] = 0;
  __syncthreads();
  const uint64_t c0 = (uint64_t)blockIdx.x * per, c1 = min(n, c0 + per);
  uint32_t skip = 0;
  for (uint64_t k = c0 + 4ull * threadIdx.x; k < c1; k += 4ull * kCountThreads * 2) {
    uint32_t ss[8], dd[8];
    bool in[8];
    load_quad(src, dst, k, c1, vec, ss, dd, in);
    load_quad(src, dst, k + 4ull * kCountThreads, c1, vec, ss + 4, dd + 4, in + 4);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      uint32_t bin, ent;
      if (!in[e]) continue;
      if (pair_bin<PREFIX>(G, B, ss[e], dd[e], bin, ent)) atomicAdd(&hist[bin], 1u);
      else ++skip;
    }
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < B.nbins; b += kCountThreads)
    if (hist[b]) atomicAdd(counts + b, hist[b]);
  if (PREFIX && skipped) {
    skip = warp_sum(skip);
    if ((threadIdx.x & 31) == 0 && skip) atomicAdd(skipped, (unsigned long long)skip);
  }
}

// Phase 1, sampled (default for large normalised windows): the histogram of 8 consecutive pairs — one
// 32-B sector of each array — out of every 2^L pairs (L = 9: 1/64 of the pairs and of the input's DRAM
// sectors); k_bin_starts scales it up with a margin.  Units of 8 pairs, not large blocks, so a flow
// whose packets arrive in one burst is sampled in proportion to its length instead of all-or-nothing.
// A region that still turns out too small spills its excess entries to the overflow log (k_bin_log), so
// the cube is exact for any input — the sample only decides how much of the work takes the fast path.
constexpr uint32_t kSampleUnit = 8;                // pairs per sample unit (one sector per array)
constexpr int kSampleUnroll = 2;
template <bool PREFIX>
__global__ void __launch_bounds__(kCountThreads) k_bin_sample(const __grid_constant__ Geo G, const __grid_constant__ BinGeo B,
                                                            const uint32_t* __restrict__ src,
                                                            const uint32_t* __restrict__ dst, uint64_t n,
                                                            uint32_t stride_log2, int vec, uint32_t* __restrict__ counts) {
  extern __shared__ uint32_t hist[];
  for (uint32_t b = threadIdx.x; b < B.nbins; b += kCountThreads) hist[b] = 0;
  __syncthreads();
  const uint64_t nu = (n + (1ull << stride_log2) - 1) >> stride_log2;   // units: pairs [u·2^L, u·2^L + 8)
  const uint64_t step = (uint64_t)gridDim.x * kCountThreads;
  for (uint64_t u0 = (uint64_t)blockIdx.x * kCountThreads + threadIdx.x; u0 < nu; u0 += step * kSampleUnroll) {
    uint32_t ss[kSampleUnroll][kSampleUnit], dd[kSampleUnroll][kSampleUnit];
    uint32_t cnt[kSampleUnroll];
#pragma unroll
    for (int v = 0; v < kSampleUnroll; ++v) {
      const uint64_t k = (u0 + v * step) << stride_log2;
      cnt[v] = u0 + v * step < nu ? (n - k >= kSampleUnit ? kSampleUnit : (uint32_t)(n - k)) : 0u;
      if (vec && cnt[v] == kSampleUnit) {
        const uint4 a0 = ld_stream4(src + k), a1 = ld_stream4(src + k + 4), b0 = ld_stream4(dst + k), b1 = ld_stream4(dst + k + 4);
        ss[v][0] = a0.x, ss[v][1] = a0.y, ss[v][2] = a0.z, ss[v][3] = a0.w;
        ss[v][4] = a1.x, ss[v][5] = a1.y, ss[v][6] = a1.z, ss[v][7] = a1.w;
        dd[v][0] = b0.x, dd[v][1] = b0.y, dd[v][2] = b0.z, dd[v][3] = b0.w;
        dd[v][4] = b1.x, dd[v][5] = b1.y, dd[v][6] = b1.z, dd[v][7] = b1.w;
      } else {
#pragma unroll
        for (uint32_t e = 0; e < kSampleUnit; ++e) {
          ss[v][e] = e < cnt[v] ? __ldcs(src + k + e) : 0u;
          dd[v][e] = e < cnt[v] ? __ldcs(dst + k + e) : 0u;
        }
      }
    }
#pragma unroll
    for (int v = 0; v < kSampleUnroll; ++v)
#pragma unroll
      for (uint32_t e = 0; e < kSampleUnit; ++e) {
        uint32_t bin, ent;
        if (e < cnt[v] && pair_bin<PREFIX>(G, B, ss[v][e], dd[v][e], bin, ent)) atomicAdd(&hist[bin], 1u);
      }
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < B.nbins; b += kCountThreads)
    if (hist[b]) atomicAdd(counts + b, hist[b]);
}

// Phase 2: bin regions.  start[b] = Σ_{b' < b} cap(b') with cap(b) = align8(counts[b] + slack) for exact
// counts (sector-aligned; slack = the duplicate padding k_bin_wc may add, 8 entries per CTA), or, for a
// sample of 8 pairs per 2^L, the scaled count est = counts[b]·2^L/8 plus est/4 + 2·sqrt(2^L·est) + 64; start[nbins] = total, cursor :=
// start (the scatter's bump allocator; the apply reads [start[b], min(cursor[b], start[b + 1]))),
// counts := 0 for the next round, the overflow-log count := 0.  One CTA (nbins ≤ 16384).
constexpr int kStartThreads = 1024;
__device__ __forceinline__ uint32_t bin_cap(uint32_t c, uint32_t slack, uint32_t sample_log2) {
  if (!sample_log2) return (c + slack + 7u) & ~7u;
  // est = c·2^L/8; sampled in units of 8 pairs, its error is at most ~sqrt(2^L·est) (a bin's pairs
  // clustered in whole units): margin est/4 + 2·sqrt(2^L·est) + 64
  const uint32_t est = (c << sample_log2) / kSampleUnit;
  const uint32_t sd = (uint32_t)sqrtf((float)est * (float)(1u << sample_log2));
  return (est + est / 4u + 2u * sd + 64u + slack + 7u) & ~7u;
}
__global__ void __launch_bounds__(kStartThreads) k_bin_starts(uint32_t nbins, uint32_t slack, uint32_t sample_log2,
                                                              uint32_t* __restrict__ counts,
                                                              uint32_t* __restrict__ start,
                                                              uint32_t* __restrict__ cursor,
                                                              uint32_t* __restrict__ log_n) {
  __shared__ uint32_t s_w[kStartThreads / 32];
  const uint32_t per = (nbins + kStartThreads - 1) / kStartThreads;
  const uint32_t b0 = threadIdx.x * per, b1 = min(nbins, b0 + per);
  uint32_t loc = 0;
  for (uint32_t b = b0; b < b1; ++b) loc += bin_cap(counts[b], slack, sample_log2);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  uint32_t run = incl - loc, tot = 0;
  for (int w = 0; w < kStartThreads / 32; ++w) {
    run += w < warp ? s_w[w] : 0u;
    tot += s_w[w];
  }
  for (uint32_t b = b0; b < b1; ++b) {
    const uint32_t x = counts[b];
    start[b] = run;
    cursor[b * kCurStride] = run;
    counts[b] = 0;
    run += bin_cap(x, slack, sample_log2);
  }
  if (threadIdx.x == 0) {
    start[nbins] = tot;
    *log_n = 0;
  }
}

// Phase 3 (default): entries of CTA j's chunk, tile by tile: rank within the tile by ATOMS on
// the tile's bin counts, a block scan of those counts (which also reserves each run at its bin's global cursor), a
// shared-memory counting sort, then the runs written out.
template <bool PREFIX, int NB>   // NB: the bin count at compile time (4096; −1: the paper geometry), 0: run time
__global__ void __launch_bounds__(kBinThreads, kBinMinBlocks) k_bin_scatter(const __grid_constant__ Geo G,
                                                             const __grid_constant__ BinGeo B,
                                                             const uint32_t* __restrict__ src,
                                                             const uint32_t* __restrict__ dst, uint64_t n, uint64_t per,
                                                             int vec, uint32_t* __restrict__ cursor,
                                                             uint32_t* __restrict__ entries,
                                                             const uint32_t* __restrict__ start,
                                                             uint32_t* __restrict__ log_n, uint32_t* __restrict__ log_e,
                                                             uint16_t* __restrict__ log_b, uint32_t pf) {
  extern __shared__ uint32_t sm[];
  uint32_t* base = sm;                                   // [nbins] this tile's reserved slot of each bin
  uint32_t* toff = base + B.nbins;                       // [nbins + 1] tile counts → exclusive offsets
  uint32_t* stage = toff + B.nbins + 1;                  // [kBinTile] entries sorted by bin
  uint16_t* sbin = reinterpret_cast<uint16_t*>(stage + kBinTile);   // [kBinTile] their bins
  uint32_t* rend = reinterpret_cast<uint32_t*>(sbin + kBinTile);    // [nbins] region ends start[b + 1]
  __shared__ uint32_t s_w[kBinThreads / 32];
  __shared__ int s_ovf;                                  // some run of this tile passes its region's end
  const uint32_t tid = threadIdx.x;
  const uint32_t nbins = NB < 0 ? 4096u : NB ? (uint32_t)NB : B.nbins;
  for (uint32_t b = tid; b < nbins; b += kBinThreads) toff[b] = 0, rend[b] = start[b + 1];
  if (tid == 0) s_ovf = 0;
  const uint64_t c0 = (uint64_t)blockIdx.x * per, c1 = min(n, c0 + per);
  const uint32_t wchunk = (nbins + kBinThreads - 1) / kBinThreads * 32;   // bins per warp (multiple of 32)
  const uint32_t pa = pin(G.mangle_a), pb = pin(G.mangle_b), pbv = pin(G.bv_seed);
  // NB < 0: the paper geometry (r = 4, g = 4096, s = 4, 256 bins per CS) with its shifts and masks as
  // immediates; otherwise pinned in registers
  constexpr bool kPaper = NB < 0;
  const uint32_t pgm = kPaper ? 4095u : pin(G.g - 1u);
  const uint32_t prm = kPaper ? 15u : pin(G.rmask), pr = kPaper ? 4u : pin(G.r);
  const uint32_t pbl = kPaper ? 8u : pin(B.bpc_log2), pes = kPaper ? 4u : pin(B.s);
  const uint32_t psm = kPaper ? 15u : pin((1u << B.s) - 1u), toff_sa = pin(smem_addr(toff));
  // all kBinPPT pairs of the thread are loaded before any is hashed (one DRAM latency per tile), then
  // each pair's registers are reused for its key (bin, rank in the tile) and entry.  (Issuing the next
  // tile's loads right after the staging pass measured slower: profiles/r02_scatter_ab.md)
  uint32_t key[kBinPPT], ent[kBinPPT];
  auto load_whole = [&](uint64_t t) {
#pragma unroll
    for (int q = 0; q < kBinPPT / 4; ++q) {
      const uint64_t k = t + 4ull * ((uint64_t)q * kBinThreads + tid);
      const uint4 a = ld_stream4(src + k), b = ld_stream4(dst + k);
      key[4 * q] = a.x, key[4 * q + 1] = a.y, key[4 * q + 2] = a.z, key[4 * q + 3] = a.w;
      ent[4 * q] = b.x, ent[4 * q + 1] = b.y, ent[4 * q + 2] = b.z, ent[4 * q + 3] = b.w;
    }
  };
  __syncthreads();
  for (uint64_t t0 = c0; t0 < c1; t0 += kBinTile) {
    if (!PREFIX && vec && t0 + kBinTile <= c1) {
      // whole tile, normalised input: no per-pair checks; parameters pinned in registers
      load_whole(t0);
#pragma unroll
      for (int i = 0; i < kBinPPT; ++i) {
        const uint32_t mi = pa * key[i] + pb, mo = pa * ent[i] + pb;           // P:175, Q2
        const uint32_t row = mix32(mo ^ pbv) & pgm;
        const uint32_t bin = ((mi & prm) << pbl) | (row >> pes);              // (cs, row >> s)
        ent[i] = ((mi >> pr) << pes) | (row & psm);                           // LP, low row bits
        key[i] = (bin << kBinRankBits) | atoms_inc(toff_sa + 4u * bin);
      }
    } else {
      bool in[kBinPPT];
#pragma unroll
      for (int q = 0; q < kBinPPT / 4; ++q)
        load_quad(src, dst, t0 + 4ull * ((uint64_t)q * kBinThreads + tid), c1, vec, key + 4 * q, ent + 4 * q, in + 4 * q);
#pragma unroll
      for (int i = 0; i < kBinPPT; ++i) {
        uint32_t bin = 0, en = 0;
        const bool ok = in[i] && pair_bin<PREFIX>(G, B, key[i], ent[i], bin, en);
        key[i] = ok ? (bin << kBinRankBits) | atomicAdd(&toff[bin], 1u) : 0xffffffffu;
        ent[i] = en;
      }
    }
    __syncthreads();
    // L2 prefetch of the next tile after the rank barrier (as in k_bin_scatter_w; pf: distance in tiles)
    if ((pf & 255u) && vec && tid == 0) {
      const uint64_t tp = t0 + (uint64_t)(pf & 255u) * kBinTile;
      if (tp + kBinTile <= c1) prefetch_l2(src + tp, kBinTile * 4), prefetch_l2(dst + tp, kBinTile * 4);
    }
    // Warp w owns bins [w·wchunk, (w+1)·wchunk): in row j (32 consecutive bins) lane l owns bin
    // 32j + ((l + j) mod 32), so a warp touches 32 consecutive words per row (conflict-free, and its 32
    // reservation atomics hit one line of the cursors; 16 in flight per thread).  Then each bin gets its
    // run in the staging array: the staging order only has to keep a bin's entries together, so it is
    // thread-major — thread t's bins follow each other — and one scan of the per-thread totals places
    // every run.  The (l + j) rotation puts a thread's consecutive runs in different banks: the write-out's
    // base[bin] loads of 32 consecutive staging positions (~16 runs of one thread) are then conflict-free
    // instead of 16-way (lane-strided ownership without it: bins 32 apart, one bank).
    {
      const int lane = tid & 31, warp = tid >> 5;
      const uint32_t w0 = warp * wchunk;
      uint32_t loc = 0;
      for (uint32_t i0 = 0; i0 < wchunk; i0 += 32 * 16) {
        uint32_t x[16], r[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t b = w0 + i0 + 32 * j + ((lane + j) & 31);
          x[j] = (i0 + 32 * j < wchunk && b < nbins) ? toff[b] : 0u;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j)
          r[j] = x[j] ? atomicAdd(cursor + (w0 + i0 + 32 * j + ((lane + j) & 31)) * kCurStride, x[j]) : 0u;
        bool over = false;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (x[j]) {
            const uint32_t b = w0 + i0 + 32 * j + ((lane + j) & 31);
            base[b] = r[j];
            over |= r[j] + x[j] > rend[b];
          }
          loc += x[j];
        }
        if (over) s_ovf = 1;
      }
      uint32_t incl = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) s_w[warp] = incl;
      __syncthreads();
      uint32_t run = incl - loc, tot = 0;
#pragma unroll
      for (int w = 0; w < kBinThreads / 32; ++w) {
        run += w < warp ? s_w[w] : 0u;
        tot += s_w[w];
      }
      for (uint32_t i0 = 0; i0 < wchunk; i0 += 32 * 16) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t b = w0 + i0 + 32 * j + ((lane + j) & 31);
          if (i0 + 32 * j < wchunk && b < nbins) {
            const uint32_t x = toff[b];
            toff[b] = run;
            if (x) base[b] -= run;   // base[b] + p is the slot of staging position p
            run += x;
          }
        }
      }
      if (tid == 0) toff[nbins] = tot;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kBinPPT; ++i) {
      if (key[i] == 0xffffffffu) continue;
      const uint32_t bin = key[i] >> kBinRankBits;
      const uint32_t pos = toff[bin] + (key[i] & ((1u << kBinRankBits) - 1u));
      stage[pos] = ent[i];
      sbin[pos] = (uint16_t)bin;
    }
    __syncthreads();
    const uint32_t total = toff[nbins];
    if (!s_ovf) {
#pragma unroll 4
      for (uint32_t p = tid; p < total; p += kBinThreads) entries[base[sbin[p]] + p] = stage[p];
    } else {   // entries past their region's end (a sampled capacity fell short) go to the overflow log
      for (uint32_t p = tid; p < total; p += kBinThreads) {
        const uint32_t bin = sbin[p], g = base[bin] + p;
        if (g < rend[bin]) {
          entries[g] = stage[p];
        } else {
          const uint32_t k = atomicAdd(log_n, 1u);
          log_e[k] = stage[p];
          log_b[k] = (uint16_t)bin;
        }
      }
    }
    __syncthreads();
    for (uint32_t b = tid; b < nbins; b += kBinThreads) toff[b] = 0;
    if (tid == 0) s_ovf = 0;
    __syncthreads();
  }
}

// Column of array a for LP (P:235 RA: CL_bs window of LP; P:239 VA: H_j(LP)).
__device__ __forceinline__ uint32_t lp_col(const Geo& G, uint64_t dbl, uint32_t lp, uint32_t a) {
  return a < G.num_ra ? (uint32_t)(dbl >> G.sh[a]) & G.colmask[a]
                      : mix32(lp ^ G.va_seeds[a - G.num_ra]) & G.colmask[a];
}

// Phase 3 (CBAA_BIN_SCATTER=wc): write-combining scatter.  One 1024-thread CTA per SM streams its chunk in rounds of
// kWcRound pairs.  Every bin owns a kWcSlot-entry slot in shared memory; a pair is appended to its bin's
// slot (rank by ATOMS on the bin's fill count).  After a barrier, thread t owns bins 4t..4t+3: a slot
// holding ≥ 8 entries stores its first 8 to the bin's region as one 32-B sector, at a position reserved
// by a global atomic issued when the bin's previous sector was stored (so the reservation's latency
// overlaps a round of appends), and moves its tail to the front.  The 4 spare entries per slot make an
// append that finds its slot full rare (≥ 5 more appends to one bin in a round than the slot has room
// for); such appends go to an overflow log that k_bin_log applies with the direct update's test-and-set.
// When the CTA ends, each bin's pending reservation (or a fresh one) takes its partial slot, padded with
// duplicates of one of the bin's entries: OR is idempotent, so duplicates change nothing in the cube.  A
// region therefore needs counts[b] + 8 slots per CTA (k_bin_starts); the apply reads [start[b], cursor[b]).
constexpr int kWcThreads = 1024;
constexpr int kWcPPT = 4;                          // pairs per thread per round (one 16-B load per array)
constexpr int kWcRound = kWcThreads * kWcPPT;      // 4096 pairs per round
constexpr uint32_t kWcSlot = 12;                   // entries per slot (a sector + 4 spare)
__host__ __device__ constexpr size_t wc_smem_bytes(uint32_t nbins) { return (size_t)nbins * (4 * kWcSlot + 4); }
__device__ __forceinline__ uint4 lds4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts4(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
}
__device__ __forceinline__ void sts(uint32_t a, uint32_t v) { asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v)); }
__device__ __forceinline__ void st_sector(uint32_t* p, uint4 a, uint4 b) {
  reinterpret_cast<uint4*>(p)[0] = a;
  reinterpret_cast<uint4*>(p)[1] = b;
}
__device__ __forceinline__ uint32_t get4(const uint4& v, int k) { return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w; }

template <bool PREFIX>
__global__ void __launch_bounds__(kWcThreads, 1) k_bin_wc(const __grid_constant__ Geo G, const __grid_constant__ BinGeo B,
                                                          const uint32_t* __restrict__ src,
                                                          const uint32_t* __restrict__ dst, uint64_t n, uint64_t per,
                                                          int vec, uint32_t* __restrict__ cursor,
                                                          uint32_t* __restrict__ entries, uint32_t* __restrict__ log_n,
                                                          uint32_t* __restrict__ log_e, uint16_t* __restrict__ log_b) {
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* occ = sm + kWcSlot * B.nbins;                           // [nbins] fill counts; slot of bin b: sm[12·b ..]
  const uint32_t tid = threadIdx.x;
  for (uint32_t b = tid; b < B.nbins; b += kWcThreads) occ[b] = 0;
  const uint32_t slot_sa = pin(smem_addr(sm)), occ_sa = pin(smem_addr(occ));
  const uint32_t pa = pin(G.mangle_a), pb = pin(G.mangle_b), pbv = pin(G.bv_seed), pgm = pin(G.g - 1u);
  const uint32_t prm = pin(G.rmask), pr = pin(G.r), pbl = pin(B.bpc_log2), pes = pin(B.s);
  const uint32_t psm = pin((1u << B.s) - 1u);
  const uint64_t c0 = (uint64_t)blockIdx.x * per, c1 = min(n, c0 + per);
  const uint32_t b0 = 4u * tid;                                     // owned bins b0..b0+3
  const bool owner = b0 < B.nbins;
  uint32_t res[4] = {0u, 0u, 0u, 0u}, rep[4] = {0u, 0u, 0u, 0u}, hasres = 0;
  uint32_t ca[kWcPPT], cb[kWcPPT];
  bool cin[kWcPPT];
  load_quad(src, dst, c0 + 4ull * tid, c1, vec, ca, cb, cin);
  __syncthreads();
  for (uint64_t t0 = c0; t0 < c1; t0 += kWcRound) {
    const uint64_t t1 = t0 + kWcRound;
    uint32_t ab[kWcPPT], ae[kWcPPT], r[kWcPPT];
    bool av[kWcPPT];
#pragma unroll
    for (int i = 0; i < kWcPPT; ++i) {
      uint32_t bin = 0, e = 0;
      bool ok = cin[i];
      if (PREFIX) {
        ok = ok && pair_bin<true>(G, B, ca[i], cb[i], bin, e);
      } else {
        const uint32_t mi = pa * ca[i] + pb, mo = pa * cb[i] + pb;           // P:175, Q2
        const uint32_t row = mix32(mo ^ pbv) & pgm;
        bin = ((mi & prm) << pbl) | (row >> pes);                           // (cs, row >> s)
        e = ((mi >> pr) << pes) | (row & psm);                              // LP, low row bits
      }
      ab[i] = bin, ae[i] = e, av[i] = ok;
    }
#pragma unroll
    for (int i = 0; i < kWcPPT; ++i) r[i] = av[i] ? atoms_inc(occ_sa + 4u * ab[i]) : kWcSlot;
#pragma unroll
    for (int i = 0; i < kWcPPT; ++i) {
      if (r[i] < kWcSlot) {
        sts(slot_sa + 4u * (kWcSlot * ab[i] + r[i]), ae[i]);
      } else if (av[i]) {
        const uint32_t k = atomicAdd(log_n, 1u);
        log_e[k] = ae[i];
        log_b[k] = (uint16_t)ab[i];
      }
    }
    __syncthreads();
    // flush the owned slots holding a sector
    if (owner) {
      uint4 o = lds4(occ_sa + 4u * b0);
      const uint32_t had = hasres;
      bool any = false;
#pragma unroll
      for (int k = 0; k < 4; ++k) {   // unrolled: res[k] is written by its atomic directly, never waited on
        const uint32_t m = get4(o, k), b = b0 + k;
        if (m >= 8u) {
          const uint32_t sa = slot_sa + 4u * kWcSlot * b;
          const uint4 v0 = lds4(sa), v1 = lds4(sa + 16u), v2 = lds4(sa + 32u);
          const uint32_t pos = (had >> k) & 1u ? res[k] : atomicAdd(cursor + b * kCurStride, 8u);
          st_sector(entries + pos, v0, v1);
          sts4(sa, v2);                         // tail (entries 8..11) to the front
          rep[k] = v0.x;
          any = true;
        }
        // the next sector's position, used a round or more later: reserved after every stored sector, and
        // first when the slot is half full, so no flush waits on its atomic; a predicated atomic into res[k]
        // itself (a pending reservation always meets ≥ 4 entries or a stored sector at the end, so it can
        // always be filled)
        const uint32_t want = (m >= 8u || (m >= 4u && !((had >> k) & 1u))) ? 1u : 0u;
        asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p atom.global.add.u32 %0, [%1], %3;\n}"
                     : "+r"(res[k]) : "l"(cursor + b * kCurStride), "r"(want), "r"(8u) : "memory");
        hasres |= want << k;
      }
      if (any) {
        o.x = o.x >= 8u ? min(o.x, kWcSlot) - 8u : o.x, o.y = o.y >= 8u ? min(o.y, kWcSlot) - 8u : o.y;
        o.z = o.z >= 8u ? min(o.z, kWcSlot) - 8u : o.z, o.w = o.w >= 8u ? min(o.w, kWcSlot) - 8u : o.w;
        sts4(occ_sa + 4u * b0, o);
      }
    }
    load_quad(src, dst, t1 + 4ull * tid, c1, vec, ca, cb, cin);   // next round's pairs (after the flush)
    __syncthreads();
  }
  // partial slots: into the pending reservation (or a fresh sector), padded with duplicates
  if (owner) {
    const uint4 o = lds4(occ_sa + 4u * b0);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t m = get4(o, k), b = b0 + k, has = (hasres >> k) & 1u;
      if (!m && !has) continue;
      const uint32_t pos = has ? res[k] : atomicAdd(cursor + b * kCurStride, 8u);
      uint32_t v[8];
      const uint32_t fill = m ? sm[kWcSlot * b] : rep[k];
#pragma unroll
      for (uint32_t i = 0; i < 8; ++i) v[i] = i < m ? sm[kWcSlot * b + i] : fill;
      st_sector(entries + pos, make_uint4(v[0], v[1], v[2], v[3]), make_uint4(v[4], v[5], v[6], v[7]));
    }
  }
}

// Overflow log of k_bin_wc (appends that found their bin's slot full): each record sets its pair's bits in
// the cube with the direct update's test-and-set (L1-cached load, RED only for a clear bit; §6), so
// the repeated records of a heavy flow cost loads, not atomics.
__global__ void k_bin_log(const __grid_constant__ Geo G, const __grid_constant__ BinGeo B,
                          const uint32_t* __restrict__ log_n, const uint32_t* __restrict__ log_e,
                          const uint16_t* __restrict__ log_b, uint32_t* __restrict__ cube) {
  const uint32_t nrec = *log_n;
  const uint32_t smask = (1u << B.s) - 1u;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nrec; i += gridDim.x * blockDim.x) {
    const uint32_t bin = log_b[i], e = log_e[i];
    const uint32_t cs = bin >> B.bpc_log2, row = ((bin & ((1u << B.bpc_log2) - 1u)) << B.s) | (e & smask);
    const uint32_t lp = e >> B.s, bit = 1u << (row & 31u);
    const uint64_t dbl = ((uint64_t)lp << G.L) | lp;
    for (uint32_t a = 0; a < G.narr; ++a) {
      uint32_t* w = cube + (uint64_t)cs * G.cs_words + G.arr_off[a] + (uint64_t)lp_col(G, dbl, lp, a) * G.wpc + (row >> 5);
      if (!(__ldca(w) & bit)) red_or(w, bit);
    }
  }
}

// Shared-memory test-and-set pieces of k_bin_apply, on 32-bit shared addresses.  A load may see a stale
// 0 (the bit set by another thread meanwhile): that only costs a redundant RED, never a lost bit.
__device__ __forceinline__ uint32_t lds(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void reds_or(uint32_t a, uint32_t bit) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(bit));
}

// ---------------------------------------------------------------- wide entries (the paper configuration)
// With r = 4 a 32-bit entry holds LP (28 bits) and only s = 4 row bits, so a word group (32 rows) is
// split over two bins and an 8192-pair tile meets 4096 bins: runs of ~2 entries, and the write-out
// of a warp touches ~16 lines per store (profiles/r02_scatter_ab.md: that write-out is 0.24 of the
// scatter's 0.66 ms; with perfectly coalesced stores the scatter takes 0.46 ms).  Wide entries are
// 64-bit — LP << 6 | row mod 64 — so a bin is (cs, row >> 6), two word groups: 1024 bins, runs of ~8
// entries (64 B), 4× fewer reservation atomics, and the bin rides in the staged entry's top bits
// (no separate bin array).  The apply gives each bin one CTA with a 128 KiB image of its two word groups.
// DRAM: 8 instead of 4 B written and read back per pair.
constexpr int kWBins = 1024;                   // 2^4 CSs × 4096 / 64 rows
// CBAA_SCW_EARLY_LOAD: a tile's register loads are issued before the previous tile's write-out, whose
// stores do not need the key/ent registers (with the L2 prefetch they hit L2): scatter 0.509 → 0.488 ms
#ifndef CBAA_SCW_EARLY_LOAD
#define CBAA_SCW_EARLY_LOAD 1
#endif
// rank key of a pair: cs << 28 | row << 16 | rank in the tile (< 2^13), so key >> 22 is the bin
// (cs << 6 | row >> 6) and (key >> 16) mod 64 the row bits kept in the entry; 0xffffffff = no pair
#ifndef CBAA_WAPPLY_THREADS
#define CBAA_WAPPLY_THREADS 1024
#endif
constexpr int kWApplyThreads = CBAA_WAPPLY_THREADS;
constexpr uint64_t kWEntMask = (1ull << 48) - 1;   // staged entry: bin << 48 | LP << 6 | row mod 64
__host__ __device__ constexpr uint32_t ilog2c(uint32_t v) { return v <= 1 ? 0 : 1 + ilog2c(v >> 1); }
// stage + base/toff/rend tables (+ the a0 class table): 76 KiB at 1024 bins, two CTAs per SM
constexpr size_t wscatter_smem(uint32_t nbins, bool prefix) {
  return (size_t)kBinTile * 8 + (3 * nbins + 1) * 4 + (prefix ? 4096 * 4 : 0);
}
constexpr size_t kWApplySmem = 2 * 16384 * 4;                                   // two word groups, 128 KiB

// PREFIX: raw on-wire pairs, classified by the inner prefixes (a0) with the two 8 KiB bitmaps
// staged in shared memory; pairs with zero or two inner endpoints are skipped and counted here (every
// pair passes through this kernel, so the bin regions can still come from a sample).
// NB < 0: the paper geometry (r = 4, g = 4096: 1024 bins, shifts and masks as immediates); NB = 256..4096:
// any geometry with g ≥ 64 whose 2^r·g/64 bins number NB (run-time r and g).  Rank key of a pair:
// bin << (32 − log2 NB) | row mod 64 << (26 − log2 NB) | rank in the tile (the paper's cs << 28 | row << 16
// | rank when NB = 1024).
template <bool PREFIX, int NB>
__global__ void __launch_bounds__(kBinThreads, kBinMinBlocks) k_bin_scatter_w(const __grid_constant__ Geo G,
                                                             const uint32_t* __restrict__ src,
                                                             const uint32_t* __restrict__ dst, uint64_t n, uint64_t per,
                                                             int vec, uint32_t* __restrict__ cursor,
                                                             uint64_t* __restrict__ entries,
                                                             const uint32_t* __restrict__ start,
                                                             uint32_t* __restrict__ log_n, uint64_t* __restrict__ log_e,
                                                             unsigned long long* __restrict__ skipped,
                                                             uint32_t pf) {
  constexpr bool kPaperW = NB < 0;
  constexpr uint32_t nbins = kPaperW ? (uint32_t)kWBins : (uint32_t)NB;
  constexpr uint32_t kBB = ilog2c(nbins), kKeySh = 32 - kBB, kRB = 26 - kBB;   // bin bits, key shift, rank bits
  static_assert(nbins % kBinThreads == 0 && (1u << kBB) == nbins && kBinTile < (1u << kRB),
                "bins per thread whole, a power of two, rank field wide enough");
  constexpr uint32_t kPerLane = nbins / kBinThreads;      // 4 bins per thread at the paper geometry
  constexpr uint32_t wchunk = kPerLane * 32;              // 128 bins per warp
  extern __shared__ __align__(16) uint64_t smw[];
  uint64_t* stage = smw;                                  // [kBinTile] bin << 48 | entry, sorted by bin
  uint32_t* base = reinterpret_cast<uint32_t*>(stage + kBinTile);   // [nbins] this tile's slot base
  uint32_t* toff = base + nbins;                          // [nbins + 1] tile counts → exclusive offsets
  uint32_t* rend = toff + nbins + 1;                      // [nbins] region ends start[b + 1]
  uint32_t* scode = rend + nbins;                         // PREFIX: [4096] 2-bit class of every /16
  __shared__ uint32_t s_w[kBinThreads / 32];
  __shared__ int s_ovf;
  const uint32_t tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  for (uint32_t b = tid; b < nbins; b += kBinThreads) toff[b] = 0, rend[b] = start[b + 1];
  // the two /16 bitmaps of is_inner folded into one 2-bit code per /16 (0 outer, 1 inner, 2 exact check):
  // one shared-memory load per endpoint
  if (PREFIX)
    for (uint32_t j = tid; j < 4096; j += kBinThreads) {
      const uint32_t f = (G.full_bits[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
      const uint32_t q = (G.part_bits[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
      uint32_t c = 0;
      for (uint32_t e = 0; e < 16; ++e) c |= (((f >> e) & 1u) ? 1u : ((q >> e) & 1u) ? 2u : 0u) << (2 * e);
      scode[j] = c;
    }
  uint32_t skip = 0;
  auto inner = [&](uint32_t ip) {   // is_inner with the classes in shared memory
    const uint32_t t = ip >> 16, c = (scode[t >> 4] >> ((t & 15) << 1)) & 3u;
    if (c != 2u) return c == 1u;
    bool in = false;
    for (uint32_t k = 0; k < G.n_prefix; ++k) in |= (ip & G.pmask[k]) == G.prefix[k];
    return in;
  };
  if (tid == 0) s_ovf = 0;
  const uint64_t c0 = (uint64_t)blockIdx.x * per, c1 = min(n, c0 + per);
  const uint32_t pa = pin(G.mangle_a), pb = pin(G.mangle_b), pbv = pin(G.bv_seed), toff_sa = pin(smem_addr(toff));
  const uint32_t w0 = warp * wchunk;
  const uint32_t gm = kPaperW ? 4095u : pin(G.g - 1u), rm = kPaperW ? 15u : pin(G.rmask);
  const uint32_t rr = kPaperW ? 4u : pin(G.r), bpl = kPaperW ? 6u : pin(G.wpc_log2 - 1u);   // log2(g / 64)
  auto rank_key = [&](uint32_t mi, uint32_t row) {   // bin, row mod 64 and an empty rank field
    if (kPaperW) return (mi << 28) | (row << 16);                                   // r = 4: cs = mi mod 16
    return ((((mi & rm) << bpl) | (row >> 6)) << kKeySh) | ((row & 63u) << kRB);
  };
  // L2 prefetch of the CTA's next tile (pf = distance in tiles | issue point << 8; 0: off): one bulk
  // prefetch per array (32 KiB each) by one thread, so the next tile's loads wait on L2 rather than DRAM.
  // Issued after the rank barrier (point 1, the default), once this tile's own loads have returned:
  // issued at the tile start (point 0) it competes with them, issued before the write-out (point 2) it
  // lands late; distance 2+ is slower (profiles/r02_scatter_ab.md).
  const uint32_t pfd = vec ? (pf & 255u) : 0u, pfat = pf >> 8;
  auto prefetch_tile = [&](uint64_t tp) {
    if (tp + kBinTile <= c1) prefetch_l2(src + tp, kBinTile * 4), prefetch_l2(dst + tp, kBinTile * 4);
  };
  if (tid == 0)
    for (uint32_t j = 1; j < pfd; ++j) prefetch_tile(c0 + (uint64_t)j * kBinTile);
  __syncthreads();
  // key = cs << 28 | row << 16 | rank in the tile (bin = key >> 22); ent = LP
  uint32_t key[kBinPPT], ent[kBinPPT];
  auto load_whole = [&](uint64_t t) {
#pragma unroll
    for (int q = 0; q < kBinPPT / 4; ++q) {
      const uint64_t k = t + 4ull * ((uint64_t)q * kBinThreads + tid);
      const uint4 a = ld_stream4(src + k), b = ld_stream4(dst + k);
      key[4 * q] = a.x, key[4 * q + 1] = a.y, key[4 * q + 2] = a.z, key[4 * q + 3] = a.w;
      ent[4 * q] = b.x, ent[4 * q + 1] = b.y, ent[4 * q + 2] = b.z, ent[4 * q + 3] = b.w;
    }
  };
  bool pre = false;   // CBAA_SCW_EARLY_LOAD: this tile's pairs were loaded during the previous write-out
  for (uint64_t t0 = c0; t0 < c1; t0 += kBinTile) {
    auto prefetch_next = [&](uint32_t at) {
      if (pfd && pfat == at && tid == 0) prefetch_tile(t0 + (uint64_t)pfd * kBinTile);
    };
    prefetch_next(0);
    const bool whole = vec && t0 + kBinTile <= c1;
    if (whole) {
      if (!pre) load_whole(t0);
    } else {
#pragma unroll
      for (int i = 0; i < kBinPPT; ++i) {
        const uint64_t k = t0 + 4ull * ((uint64_t)(i >> 2) * kBinThreads + tid) + (i & 3);
        key[i] = k < c1 ? __ldcs(src + k) : 0u;
        ent[i] = k < c1 ? __ldcs(dst + k) : 0u;
      }
    }
    if (!PREFIX && whole) {   // every pair valid: unconditional rank (no branch around each ATOMS)
#pragma unroll
      for (int i = 0; i < kBinPPT; ++i) {
        const uint32_t mi = pa * key[i] + pb, mo = pa * ent[i] + pb;         // P:175, Q2
        const uint32_t row = mix32(mo ^ pbv) & gm;
        const uint32_t hi = rank_key(mi, row);
        ent[i] = mi >> rr;                                                  // LP
        key[i] = hi | atoms_inc(toff_sa + 4u * (hi >> kKeySh));             // bin (cs, row >> 6)
      }
    } else {
#pragma unroll
      for (int i = 0; i < kBinPPT; ++i) {
        bool ok = whole || t0 + 4ull * ((uint64_t)(i >> 2) * kBinThreads + tid) + (i & 3) < c1;
        uint32_t iip = key[i], oip = ent[i];
        if (PREFIX) {   // a0: keep inner→outer, swap outer→inner, skip the rest (Q25); branch-free
          const bool si = inner(iip), di = inner(oip);
          skip += (ok && si == di) ? 1u : 0u;
          ok = ok && si != di;
          iip = di ? ent[i] : key[i];
          oip = di ? key[i] : ent[i];
        }
        const uint32_t mi = pa * iip + pb, mo = pa * oip + pb;               // P:175, Q2
        const uint32_t row = mix32(mo ^ pbv) & gm;
        const uint32_t hi = rank_key(mi, row);
        ent[i] = mi >> rr;                                                  // LP
        const uint32_t rank = atoms_inc_if(toff_sa + 4u * (hi >> kKeySh), ok ? 1u : 0u);
        key[i] = ok ? hi | rank : 0xffffffffu;
      }
    }
    __syncthreads();
    prefetch_next(1);
    // per-bin reservation and offsets (rotated lane ownership as in k_bin_scatter)
    {
      uint32_t x[kPerLane], r[kPerLane], loc = 0;
      bool over = false;
#pragma unroll
      for (int j = 0; j < (int)kPerLane; ++j) x[j] = toff[w0 + 32 * j + ((lane + j) & 31)];
#pragma unroll
      for (int j = 0; j < (int)kPerLane; ++j)
        r[j] = x[j] ? atomicAdd(cursor + (w0 + 32 * j + ((lane + j) & 31)) * kCurStride, x[j]) : 0u;
#pragma unroll
      for (int j = 0; j < (int)kPerLane; ++j) {
        const uint32_t b = w0 + 32 * j + ((lane + j) & 31);
        if (x[j]) {
          base[b] = r[j];
          over |= r[j] + x[j] > rend[b];
        }
        loc += x[j];
      }
      if (over) s_ovf = 1;
      uint32_t incl = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) s_w[warp] = incl;
      __syncthreads();
      uint32_t run = incl - loc, tot = 0;
#pragma unroll
      for (int w = 0; w < kBinThreads / 32; ++w) {
        run += w < warp ? s_w[w] : 0u;
        tot += s_w[w];
      }
#pragma unroll
      for (int j = 0; j < (int)kPerLane; ++j) {
        const uint32_t b = w0 + 32 * j + ((lane + j) & 31);
        toff[b] = run;
        if (x[j]) base[b] -= run;   // base[b] + p is the slot of staging position p
        run += x[j];
      }
      if (tid == 0) toff[nbins] = tot;
    }
    __syncthreads();
    auto stage_one = [&](int i) {
      const uint32_t bin = key[i] >> kKeySh;
      const uint32_t pos = toff[bin] + (key[i] & ((1u << kRB) - 1u));
      stage[pos] = ((uint64_t)bin << 48) | ((uint64_t)ent[i] << 6) | ((key[i] >> kRB) & 63u);
    };
    if (!PREFIX && whole) {   // every pair of the tile is valid: no per-pair test (no reconvergence)
#pragma unroll
      for (int i = 0; i < kBinPPT; ++i) stage_one(i);
    } else {
#pragma unroll
      for (int i = 0; i < kBinPPT; ++i)
        if (key[i] != 0xffffffffu) stage_one(i);
    }
    __syncthreads();
    prefetch_next(2);
    const uint32_t total = toff[nbins];
    if (CBAA_SCW_EARLY_LOAD) {   // the next tile's loads go out before this tile's write-out
      pre = vec && t0 + 2 * (uint64_t)kBinTile <= c1;
      if (pre) load_whole(t0 + kBinTile);
    }
    if (!s_ovf && total == kBinTile) {   // a full tile: compile-time trip count, no bounds tests
#pragma unroll 8
      for (int k = 0; k < kBinTile / kBinThreads; ++k) {
        const uint32_t p = tid + k * kBinThreads;
        const uint64_t v = stage[p];
        entries[base[(uint32_t)(v >> 48)] + p] = v & kWEntMask;
      }
    } else if (!s_ovf) {
#pragma unroll 4
      for (uint32_t p = tid; p < total; p += kBinThreads) {
        const uint64_t v = stage[p];
        entries[base[(uint32_t)(v >> 48)] + p] = v & kWEntMask;
      }
    } else {   // past a region's end (a sampled capacity fell short): to the overflow log, bin included
      for (uint32_t p = tid; p < total; p += kBinThreads) {
        const uint64_t v = stage[p];
        const uint32_t bin = (uint32_t)(v >> 48), g = base[bin] + p;
        if (g < rend[bin]) entries[g] = v & kWEntMask;
        else log_e[atomicAdd(log_n, 1u)] = v;
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < (int)kPerLane; ++j) toff[w0 + 32 * j + lane] = 0;
    if (tid == 0) s_ovf = 0;
    __syncthreads();
  }
  if (PREFIX && skipped) {   // (null: an exact count already counted them)
    skip = warp_sum(skip);
    if (lane == 0 && skip) atomicAdd(skipped, (unsigned long long)skip);
  }
}

// The paper configuration's column extraction: RA(i) = bits [clbs(i), clbs(i) + 12) of the 28-bit LP
// (MSB-first, wrapping; clbs [0, 10, 20]: shifts 44/34/24 of the doubled LP), VA = mix32(LP ⊕ seed)
// (P:235); image offset of array a = 4096·a words.
__device__ __forceinline__ void paper_cols(uint32_t lp, uint32_t vseed, uint32_t c[4]) {
  const uint64_t dbl = ((uint64_t)lp << 28) | lp;
  c[0] = (uint32_t)(dbl >> 44) & 4095u;
  c[1] = (uint32_t)(dbl >> 34) & 4095u;
  c[2] = (uint32_t)(dbl >> 24) & 4095u;
  c[3] = mix32(lp ^ vseed) & 4095u;
}

// Apply of the wide entries: one CTA per bin (cs, row >> 6) = two word groups, image sub[h][16384]
// (h = bit 5 of the row); test-and-set in shared memory, then one RED per non-zero word.
__global__ void __launch_bounds__(kWApplyThreads, 1) k_bin_apply_w(const __grid_constant__ Geo G,
                                                                  const uint32_t* __restrict__ start,
                                                                  const uint32_t* __restrict__ end,
                                                                  const uint64_t* __restrict__ entries,
                                                                  uint32_t* __restrict__ cube) {
  extern __shared__ uint32_t sub[];
  constexpr uint32_t kCols = 16384;   // Σc(i) words of one word group (paper configuration)
  const uint32_t sbase = pin(smem_addr(sub));
  const uint32_t b = blockIdx.x, cs = b >> 6, wq = b & 63u;
  for (uint32_t i = threadIdx.x; i < 2 * kCols / 4; i += kWApplyThreads)
    reinterpret_cast<uint4*>(sub)[i] = make_uint4(0u, 0u, 0u, 0u);
  const uint32_t vseed = pin(G.va_seeds[0]);
  __syncthreads();
  const uint32_t P0 = start[b], E0 = min(end[b * kCurStride], start[b + 1]);
  const uint64_t* __restrict__ ent = entries + P0;
  const uint32_t len = E0 - P0;
  auto set_bits = [&](uint64_t e) {
    const uint32_t lp = (uint32_t)(e >> 6), r6 = (uint32_t)e & 63u;
    const uint32_t bit = 1u << (r6 & 31u), hb = sbase + (r6 >> 5) * (4u * kCols);
    uint32_t c[4], adr[4], v[4];
    paper_cols(lp, vseed, c);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      adr[a] = hb + 16384u * (uint32_t)a + 4u * c[a];
      v[a] = lds(adr[a]);
    }
    // one branch per entry (a predicated shared atomic compiles to a branch each): most entries repeat
    // an earlier one and find all four bits set; the rest OR each word with its missing bit (or 0)
    if (!(v[0] & v[1] & v[2] & v[3] & bit)) {
#pragma unroll
      for (int a = 0; a < 4; ++a) reds_or(adr[a], bit & ~v[a]);
    }
  };
  constexpr uint32_t kStep = kApplyUnroll * kWApplyThreads;
  uint64_t e[kApplyUnroll];
  uint32_t p = threadIdx.x;
#pragma unroll
  for (int u = 0; u < kApplyUnroll; ++u) e[u] = p + u * kWApplyThreads < len ? __ldcs(ent + p + u * kWApplyThreads) : 0ull;
  while (p < len) {
    const uint32_t pn = p + kStep;
    uint64_t en[kApplyUnroll];
#pragma unroll
    for (int u = 0; u < kApplyUnroll; ++u)
      en[u] = pn + u * kWApplyThreads < len ? __ldcs(ent + pn + u * kWApplyThreads) : 0ull;
    if (p + (kApplyUnroll - 1) * kWApplyThreads < len) {
#pragma unroll
      for (int u = 0; u < kApplyUnroll; ++u) set_bits(e[u]);
    } else {
#pragma unroll
      for (int u = 0; u < kApplyUnroll; ++u)
        if (p + u * kWApplyThreads < len) set_bits(e[u]);
    }
#pragma unroll
    for (int u = 0; u < kApplyUnroll; ++u) e[u] = en[u];
    p = pn;
  }
  __syncthreads();
  // image word h·16384 + i = word (2·wq + h) of column i of CS cs: the two halves of a column
  // are adjacent cube words, OR-ed in with one 64-bit RED (half the L2 atomics of two 32-bit ones)
  uint32_t* cw = cube + (uint64_t)cs * G.cs_words + 2u * wq;
  for (uint32_t i = threadIdx.x; i < kCols; i += kWApplyThreads) {
    const uint32_t v0 = sub[i], v1 = sub[kCols + i];
    if (v0 | v1) red_or64(reinterpret_cast<unsigned long long*>(cw + (uint64_t)i * G.wpc), ((uint64_t)v1 << 32) | v0);
  }
}

// Column of array a (RA: a CL_bs window of LP; VA: H_j(LP)) and its word-group index:
// the column's position among the CS's Σc(i) columns in S:116 order.
__device__ __forceinline__ uint32_t wg_col(const Geo& G, uint64_t dbl, uint32_t lp, uint32_t a) {
  const uint32_t c = a < G.num_ra ? (uint32_t)(dbl >> G.sh[a]) & G.colmask[a]
                                  : mix32(lp ^ G.va_seeds[a - G.num_ra]) & G.colmask[a];
  return (G.arr_off[a] >> G.wpc_log2) + c;
}

// Apply of the wide entries for other geometries (k_bin_scatter_w<·, NB ≥ 0>): bin b = (cs, row >> 6),
// image sub[h][ncols] of its two word groups (ncols = Σc(i) ≤ 16384, so ≤ 128 KiB), entries LP << 6 | row
// mod 64; the walk, test-and-set and 64-bit flush of k_bin_apply_w with run-time column extraction.
// NRA/NVA > 0: that array split at compile time (run-time shifts, masks and seeds).
template <int NRA, int NVA>
__global__ void __launch_bounds__(kWApplyThreads, 1) k_bin_apply_wg(const __grid_constant__ Geo G, uint32_t ncols,
                                                                   const uint32_t* __restrict__ start,
                                                                   const uint32_t* __restrict__ end,
                                                                   const uint64_t* __restrict__ entries,
                                                                   uint32_t* __restrict__ cube) {
  extern __shared__ uint32_t sub[];
  const uint32_t sbase = pin(smem_addr(sub));
  const uint32_t bpl = G.wpc_log2 - 1u;   // log2(bins per CS) = log2(g / 64)
  const uint32_t b = blockIdx.x, cs = b >> bpl, wq = b & ((1u << bpl) - 1u);
  for (uint32_t i = threadIdx.x; i < 2 * ncols / 4; i += kWApplyThreads)
    reinterpret_cast<uint4*>(sub)[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();
  const uint32_t narr = NRA > 0 ? (uint32_t)(NRA + NVA) : G.narr, L = G.L;
  const uint32_t P0 = start[b], E0 = min(end[b * kCurStride], start[b + 1]);
  const uint64_t* __restrict__ ent = entries + P0;
  const uint32_t len = E0 - P0;
  auto set_bits = [&](uint64_t e) {
    const uint32_t lp = (uint32_t)(e >> 6), r6 = (uint32_t)e & 63u;
    const uint32_t bit = 1u << (r6 & 31u), hb = sbase + (r6 >> 5) * (4u * ncols);
    const uint64_t dbl = ((uint64_t)lp << L) | lp;
    uint32_t adr[CBAA_MAX_ARRAYS], v[CBAA_MAX_ARRAYS], all = bit;
#pragma unroll
    for (uint32_t a = 0; a < CBAA_MAX_ARRAYS; ++a)
      if (a < narr) {
        adr[a] = hb + 4u * wg_col(G, dbl, lp, a);
        v[a] = lds(adr[a]);
        all &= v[a];
      }
    if (!all) {
#pragma unroll
      for (uint32_t a = 0; a < CBAA_MAX_ARRAYS; ++a)
        if (a < narr) reds_or(adr[a], bit & ~v[a]);
    }
  };
  constexpr uint32_t kStep = kApplyUnroll * kWApplyThreads;
  uint64_t e[kApplyUnroll];
  uint32_t p = threadIdx.x;
#pragma unroll
  for (int u = 0; u < kApplyUnroll; ++u) e[u] = p + u * kWApplyThreads < len ? __ldcs(ent + p + u * kWApplyThreads) : 0ull;
  while (p < len) {
    const uint32_t pn = p + kStep;
    uint64_t en[kApplyUnroll];
#pragma unroll
    for (int u = 0; u < kApplyUnroll; ++u)
      en[u] = pn + u * kWApplyThreads < len ? __ldcs(ent + pn + u * kWApplyThreads) : 0ull;
#pragma unroll
    for (int u = 0; u < kApplyUnroll; ++u)
      if (p + u * kWApplyThreads < len) set_bits(e[u]);
#pragma unroll
    for (int u = 0; u < kApplyUnroll; ++u) e[u] = en[u];
    p = pn;
  }
  __syncthreads();
  uint32_t* cw = cube + (uint64_t)cs * G.cs_words + 2u * wq;
  for (uint32_t i = threadIdx.x; i < ncols; i += kWApplyThreads) {
    const uint32_t v0 = sub[i], v1 = sub[ncols + i];
    if (v0 | v1) red_or64(reinterpret_cast<unsigned long long*>(cw + (uint64_t)i * G.wpc), ((uint64_t)v1 << 32) | v0);
  }
}

// Per-array apply of the wide entries (k_bin_scatter_w<·, NB>) when the word groups of all arrays do not
// fit shared memory together (Σc(i) > 16384, e.g. cbn = 14: 512 KiB) but each array's do (c(a) ≤ 16384):
// CTA (b, a) = blockIdx (b·narr + a) keeps the two word groups of array a only (≤ 128 KiB) and walks all of
// bin b's entries, setting one bit per entry; the narr CTAs of a bin are adjacent, so the entries come from
// DRAM once and from L2 for the others.  The cube is the same OR of bits.
__global__ void __launch_bounds__(kWApplyThreads, 1) k_bin_apply_wa(const __grid_constant__ Geo G,
                                                                   const uint32_t* __restrict__ start,
                                                                   const uint32_t* __restrict__ end,
                                                                   const uint64_t* __restrict__ entries,
                                                                   uint32_t* __restrict__ cube) {
  extern __shared__ uint32_t sub[];
  const uint32_t sbase = pin(smem_addr(sub));
  const uint32_t narr = G.narr, bpl = G.wpc_log2 - 1u;
  const uint32_t b = blockIdx.x / narr, a = blockIdx.x - b * narr;
  const uint32_t cs = b >> bpl, wq = b & ((1u << bpl) - 1u);
  const uint32_t cols = G.ncols[a], L = G.L;
  for (uint32_t i = threadIdx.x; i < 2 * cols / 4; i += kWApplyThreads)
    reinterpret_cast<uint4*>(sub)[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();
  const bool ra = a < G.num_ra;
  const uint32_t sh = ra ? G.sh[a] : 0u, cm = G.colmask[a], seed = ra ? 0u : G.va_seeds[a - G.num_ra];
  const uint32_t P0 = start[b], E0 = min(end[b * kCurStride], start[b + 1]);
  const uint64_t* __restrict__ ent = entries + P0;
  const uint32_t len = E0 - P0;
  auto set_bit = [&](uint64_t e) {
    const uint32_t lp = (uint32_t)(e >> 6), r6 = (uint32_t)e & 63u;
    const uint32_t c = ra ? (uint32_t)((((uint64_t)lp << L) | lp) >> sh) & cm : mix32(lp ^ seed) & cm;
    const uint32_t adr = sbase + (r6 >> 5) * (4u * cols) + 4u * c, bit = 1u << (r6 & 31u);
    if (!(lds(adr) & bit)) reds_or(adr, bit);
  };
  constexpr uint32_t kStep = kApplyUnroll * kWApplyThreads;
  uint64_t e[kApplyUnroll];
  uint32_t p = threadIdx.x;
#pragma unroll
  for (int u = 0; u < kApplyUnroll; ++u) e[u] = p + u * kWApplyThreads < len ? ent[p + u * kWApplyThreads] : 0ull;
  while (p < len) {
    const uint32_t pn = p + kStep;
    uint64_t en[kApplyUnroll];
#pragma unroll
    for (int u = 0; u < kApplyUnroll; ++u) en[u] = pn + u * kWApplyThreads < len ? ent[pn + u * kWApplyThreads] : 0ull;
#pragma unroll
    for (int u = 0; u < kApplyUnroll; ++u)
      if (p + u * kWApplyThreads < len) set_bit(e[u]);
#pragma unroll
    for (int u = 0; u < kApplyUnroll; ++u) e[u] = en[u];
    p = pn;
  }
  __syncthreads();
  uint32_t* cw = cube + (uint64_t)cs * G.cs_words + G.arr_off[a] + 2u * wq;
  for (uint32_t i = threadIdx.x; i < cols; i += kWApplyThreads) {
    const uint32_t v0 = sub[i], v1 = sub[cols + i];
    if (v0 | v1) red_or64(reinterpret_cast<unsigned long long*>(cw + (uint64_t)i * G.wpc), ((uint64_t)v1 << 32) | v0);
  }
}

// Overflow log of the generic wide scatter: records bin << 48 | LP << 6 | row mod 64, applied with the
// direct update's test-and-set.
__global__ void k_bin_log_wg(const __grid_constant__ Geo G, const uint32_t* __restrict__ log_n,
                             const uint64_t* __restrict__ log_e, uint32_t* __restrict__ cube) {
  const uint32_t nrec = *log_n;
  const uint32_t bpl = G.wpc_log2 - 1u;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nrec; i += gridDim.x * blockDim.x) {
    const uint64_t v = log_e[i];
    const uint32_t bin = (uint32_t)(v >> 48), cs = bin >> bpl;
    const uint32_t row = ((bin & ((1u << bpl) - 1u)) << 6) | ((uint32_t)v & 63u), bit = 1u << (row & 31u);
    const uint32_t lp = (uint32_t)((v & kWEntMask) >> 6);
    const uint64_t dbl = ((uint64_t)lp << G.L) | lp;
    for (uint32_t a = 0; a < G.narr; ++a) {
      uint32_t* w = cube + (uint64_t)cs * G.cs_words + (uint64_t)wg_col(G, dbl, lp, a) * G.wpc + (row >> 5);
      if (!(__ldca(w) & bit)) red_or(w, bit);
    }
  }
}

// Overflow log of the wide scatter: records bin << 48 | LP << 6 | row mod 64, applied with the direct
// update's test-and-set.
__global__ void k_bin_log_w(const __grid_constant__ Geo G, const uint32_t* __restrict__ log_n,
                            const uint64_t* __restrict__ log_e, uint32_t* __restrict__ cube) {
  const uint32_t nrec = *log_n;
  const uint32_t vseed = G.va_seeds[0];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nrec; i += gridDim.x * blockDim.x) {
    const uint64_t v = log_e[i];
    const uint32_t bin = (uint32_t)(v >> 48), cs = bin >> 6, row = ((bin & 63u) << 6) | ((uint32_t)v & 63u);
    const uint32_t lp = (uint32_t)(v >> 6) & ((1u << 28) - 1u), bit = 1u << (row & 31u);
    uint32_t c[4];
    paper_cols(lp, vseed, c);
    for (uint32_t a = 0; a < 4; ++a) {
      uint32_t* w = cube + (uint64_t)cs * G.cs_words + G.arr_off[a] + (uint64_t)c[a] * G.wpc + (row >> 5);
      if (!(__ldca(w) & bit)) red_or(w, bit);
    }
  }
}

// Phase 4: one CTA per word group (cs, w): its bins' entries set bits in a shared-memory image of the
// group (word i = word w of column i of CS cs, columns of all arrays in S:116 order), which is then
// OR-ed into the cube.  The CTA owns those words for the whole launch.  <3, 1>: paper shape unrolled.
// P: the paper's default configuration (3 RAs + 1 VA of 4096 columns, clbs [0, 10, 20], cbn 12, r = 4):
// extraction shifts, masks and array offsets in the image as immediates
template <int NRA, int NVA, int S, bool P = false>
__global__ void __launch_bounds__(kApplyThreads, 3) k_bin_apply(const __grid_constant__ Geo G,
                                                             const __grid_constant__ BinGeo B,
                                                             const uint32_t* __restrict__ start,
                                                             const uint32_t* __restrict__ end,
                                                             const uint32_t* __restrict__ entries,
                                                             uint32_t* __restrict__ cube) {
  // S: entry row bits known at compile time (4 = the paper's r = 4, hence also L = 28), −1: run time
  extern __shared__ uint32_t sub[];
  const uint32_t sbase = pin(smem_addr(sub));
  const uint32_t wg = blockIdx.x, cs = wg >> G.wpc_log2, w = wg & (G.wpc - 1u);
  for (uint32_t i = threadIdx.x; i < B.ncols; i += kApplyThreads) sub[i] = 0;
  uint32_t cbase[CBAA_MAX_ARRAYS];
  const uint32_t narr = NRA ? (uint32_t)(NRA + NVA) : G.narr;
#pragma unroll
  for (uint32_t a = 0; a < CBAA_MAX_ARRAYS; ++a) cbase[a] = a < narr ? G.arr_off[a] >> G.wpc_log2 : 0u;
  __syncthreads();
  // the word group's bins are adjacent in the entry array, bin k of the group gives row bits k << s;
  // loads of the next batch are issued before the current batch is applied
  const uint32_t es = S >= 0 ? (uint32_t)S : B.s;
  const uint32_t L = (S >= 0 && S < 5) ? 32u - (uint32_t)S : G.L;   // s < 5 ⇔ r = s
  const uint32_t kb = 1u << (5 - es), b0 = (cs << B.bpc_log2) + w * kb, smask = (1u << es) - 1u;
  // bin k of the group holds [start[b0 + k], min(cursor, start[b0 + k + 1])); the rest of its region (sector
  // padding, unused capacity) is skipped, and a cursor past the region's end means the excess is in the log
  const uint32_t P0 = start[b0], P1 = start[b0 + kb], B1 = pin(kb > 1 ? start[b0 + 1] : P1);
  const uint32_t E0 = pin(min(end[b0 * kCurStride], start[b0 + 1]));
  const uint32_t E1 = pin(kb > 1 ? min(end[(b0 + 1) * kCurStride], start[b0 + 2]) : E0);
  // paper shape: per-array shift, mask and shared base address pinned in registers
  uint32_t shv[NRA > 0 ? NRA : 1], mk[NRA > 0 ? NRA + NVA : 1], ab[NRA > 0 ? NRA + NVA : 1];
  uint32_t vseed = 0;
  if constexpr (NRA > 0) {
#pragma unroll
    for (int a = 0; a < NRA + NVA; ++a) {
      if (a < NRA) shv[a] = pin(G.sh[a]);
      mk[a] = pin(G.colmask[a]);
      ab[a] = pin(sbase + 4u * cbase[a]);
    }
    if constexpr (NVA == 1) vseed = pin(G.va_seeds[0]);
  }
  // the entry's |RA|+|VA| bits, row bit `hi | (e mod 2^s)`, set in the shared image (test first)
  auto set_bits = [&](uint32_t e, uint32_t hi) {
    const uint32_t lp = e >> es, bit = 1u << (hi | (e & smask));
    const uint64_t dbl = ((uint64_t)lp << L) | lp;
    if constexpr (NRA > 0) {
      uint32_t adr[NRA + NVA], v[NRA + NVA];
#pragma unroll
      for (int a = 0; a < NRA + NVA; ++a) {
        constexpr uint32_t kSh[3] = {44u, 34u, 24u};   // 2L − clbs(i) − cbn(i) at the paper configuration
        const uint32_t sh_a = P ? kSh[a < 3 ? a : 0] : shv[a < NRA ? a : 0];
        const uint32_t mk_a = P ? 4095u : mk[a];
        const uint32_t col = a < NRA ? (uint32_t)(dbl >> sh_a) & mk_a
                                     : mix32(lp ^ (NVA == 1 ? vseed : G.va_seeds[a - NRA])) & mk_a;
        adr[a] = (P ? sbase + 16384u * (uint32_t)a : ab[a]) + 4u * col;
        v[a] = lds(adr[a]);
      }
      uint32_t all = bit;   // one branch per entry (see k_bin_apply_w)
#pragma unroll
      for (int a = 0; a < NRA + NVA; ++a) all &= v[a];
      if (!all) {
#pragma unroll
        for (int a = 0; a < NRA + NVA; ++a) reds_or(adr[a], bit & ~v[a]);
      }
    } else {
      for (uint32_t a = 0; a < narr; ++a) {
        const uint32_t adr = sbase + 4u * ((G.arr_off[a] >> G.wpc_log2) + lp_col(G, dbl, lp, a));
        if (!(lds(adr) & bit)) reds_or(adr, bit);
      }
    }
  };
  // kb > 2: position q of [P0, P1) → its bin by search, skipped if past that bin's valid end
  auto set_bits_at = [&](uint32_t e, uint32_t v) {
    const uint32_t q = P0 + v;
    uint32_t k = 0;
    for (uint32_t j = 1; j < kb; ++j) k += q >= start[b0 + j] ? 1u : 0u;
    if (q >= min(end[(b0 + k) * kCurStride], start[b0 + k + 1])) return;
    set_bits(e, k << es);
  };
  // one contiguous range of entries, kApplyUnroll per thread in flight (the next batch's loads are
  // issued before the current batch is applied)
  auto walk = [&](const uint32_t* __restrict__ ent, uint32_t len, uint32_t hi, bool search) {
    constexpr uint32_t kStep = kApplyUnroll * kApplyThreads;
    uint32_t e[kApplyUnroll];
    uint32_t p = threadIdx.x;
#pragma unroll
    for (int u = 0; u < kApplyUnroll; ++u) e[u] = p + u * kApplyThreads < len ? __ldcs(ent + p + u * kApplyThreads) : 0u;
    while (p < len) {
      const uint32_t pn = p + kStep;
      uint32_t en[kApplyUnroll];
#pragma unroll
      for (int u = 0; u < kApplyUnroll; ++u)
        en[u] = pn + u * kApplyThreads < len ? __ldcs(ent + pn + u * kApplyThreads) : 0u;
      if (p + (kApplyUnroll - 1) * kApplyThreads < len) {   // whole batch: no per-entry bound checks
#pragma unroll
        for (int u = 0; u < kApplyUnroll; ++u) search ? set_bits_at(e[u], p + u * kApplyThreads) : set_bits(e[u], hi);
      } else {
#pragma unroll
        for (int u = 0; u < kApplyUnroll; ++u)
          if (p + u * kApplyThreads < len) search ? set_bits_at(e[u], p + u * kApplyThreads) : set_bits(e[u], hi);
      }
#pragma unroll
      for (int u = 0; u < kApplyUnroll; ++u) e[u] = en[u];
      p = pn;
    }
  };
  // kb ≤ 2 (r ≥ 4, the paper's geometry): each bin's valid entries [start, min(cursor, next start)) as its
  // own range with a constant row bit, so no padding or spare capacity is read and no entry needs a bin
  // lookup; kb > 2: positions [P0, P1) with the per-entry search
  if (kb <= 2) {
    walk(entries + P0, E0 - P0, 0u, false);
    if (kb == 2) walk(entries + B1, E1 - B1, 1u << es, false);
  } else {
    walk(entries + P0, P1 - P0, 0u, true);
  }
  __syncthreads();
  uint32_t* cw = cube + (uint64_t)cs * G.cs_words + w;
  for (uint32_t i = threadIdx.x; i < B.ncols; i += kApplyThreads) {
    const uint32_t v = sub[i];
    if (v) red_or(cw + (uint64_t)i * G.wpc, v);
  }
}

}  // namespace cbaa
