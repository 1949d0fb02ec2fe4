// Binned update (CBAA_UPDATE_BINNED): Alg. 1 with the random bit sets moved on chip.
//
// All |RA|+|VA| bits of one pair sit in the same CS (RP) and in the same row (H_bv(oip)),
// so a pair's bits all fall in one "word group" — word w = row/32 of every column of CS cs — a set of
// Σc(i) cube words (64 KiB at the paper geometry) that fits in shared memory.  The update then runs as
// three streaming kernels instead of 4 random L2 accesses per pair:
//   k_bin_count    histogram of bins (cs, row >> s) per CTA chunk               reads 8 B/pair
//   k_bin_scan_*   exclusive scan of the (bin, CTA) counts → write offsets
//   k_bin_scatter  tile-local counting sort, bin-contiguous runs of entries     reads 8, writes 4 B/pair
//                  entry = LP << s | (row mod 2^s), s = min(5, r) (fits 32 bits since |LP| = 32 − r)
//   k_bin_apply    one CTA per word group: the bits are set in a shared-memory copy of the word group
//                  (test-and-set, ATOMS.OR only when the bit is still 0), then OR-ed into the cube with
//                  one RED per non-zero word                                      reads 4 B/pair
// The cube is the same set of bits as the direct update's (OR is order-free): parity is bit-exact.
#pragma once
#include "kernels.cuh"

namespace cbaa {

struct BinGeo {
  uint32_t s;          // row bits kept in an entry, min(5, r)
  uint32_t bpc_log2;   // log2(bins per CS) = log2(g) − s
  uint32_t nbins;      // 2^r · g / 2^s
  uint32_t nblk;       // CTAs of k_bin_count / k_bin_scatter; CTA j owns pairs [j·per, (j+1)·per)
  uint32_t ncols;      // Σc(i): words of one word group
};

constexpr int kBinThreads = 256;
constexpr int kBinPPT = 32;                        // pairs per thread per scatter tile
constexpr int kBinTile = kBinThreads * kBinPPT;    // 8192 pairs
constexpr int kBinRankBits = 14;                   // key = bin << 14 | rank within the tile
constexpr int kApplyThreads = 256;
constexpr int kScanSeg = 8192;                     // elements per CTA of the offset scan

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

// Phase 1: per-CTA bin histogram, written bin-major: counts[bin · nblk + cta].
template <bool PREFIX>
__global__ void __launch_bounds__(kBinThreads) k_bin_count(const __grid_constant__ Geo G, const __grid_constant__ BinGeo B,
                                                           const uint32_t* __restrict__ src,
                                                           const uint32_t* __restrict__ dst, uint64_t n, uint64_t per,
                                                           int vec, uint32_t* __restrict__ counts,
                                                           unsigned long long* __restrict__ skipped) {
  extern __shared__ uint32_t hist[];
  for (uint32_t b = threadIdx.x; b < B.nbins; b += kBinThreads) hist[b] = 0;
  __syncthreads();
  const uint64_t c0 = (uint64_t)blockIdx.x * per, c1 = min(n, c0 + per);
  uint32_t skip = 0;
  for (uint64_t k = c0 + 4ull * threadIdx.x; k < c1; k += 4ull * kBinThreads * 2) {
    uint32_t ss[8], dd[8];
    bool in[8];
    load_quad(src, dst, k, c1, vec, ss, dd, in);
    load_quad(src, dst, k + 4ull * kBinThreads, c1, vec, ss + 4, dd + 4, in + 4);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      uint32_t bin, ent;
      if (!in[e]) continue;
      if (pair_bin<PREFIX>(G, B, ss[e], dd[e], bin, ent)) atomicAdd(&hist[bin], 1u);
      else ++skip;
    }
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < B.nbins; b += kBinThreads) counts[(uint64_t)b * B.nblk + blockIdx.x] = hist[b];
  if (PREFIX && skipped) {
    skip = warp_sum(skip);
    if ((threadIdx.x & 31) == 0 && skip) atomicAdd(skipped, (unsigned long long)skip);
  }
}

// Phase 2a: sum of each kScanSeg-element segment of the counts.
__global__ void __launch_bounds__(kBinThreads) k_bin_scan_reduce(const uint32_t* __restrict__ c, uint64_t m,
                                                                 uint32_t* __restrict__ part) {
  const uint64_t s0 = (uint64_t)blockIdx.x * kScanSeg;
  uint32_t v = 0;
  for (uint32_t i = threadIdx.x; i < kScanSeg; i += kBinThreads)
    if (s0 + i < m) v += c[s0 + i];
  v = warp_sum(v);
  __shared__ uint32_t s_w[kBinThreads / 32];
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kBinThreads / 32; ++w) t += s_w[w];
    part[blockIdx.x] = t;
  }
}

// Phase 2b: exclusive scan in place; c[m] = total.  Each CTA adds the sum of the segments before it.
__global__ void __launch_bounds__(kBinThreads) k_bin_scan_down(uint32_t* __restrict__ c, uint64_t m,
                                                               const uint32_t* __restrict__ part) {
  __shared__ uint32_t seg[kScanSeg];
  __shared__ uint32_t s_w[kBinThreads / 32];
  __shared__ uint32_t s_base;
  const uint64_t s0 = (uint64_t)blockIdx.x * kScanSeg;
  uint32_t pre = 0;
  for (uint32_t q = threadIdx.x; q < blockIdx.x; q += kBinThreads) pre += part[q];
  pre = warp_sum(pre);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = pre;
  for (uint32_t i = threadIdx.x; i < kScanSeg; i += kBinThreads) seg[i] = s0 + i < m ? c[s0 + i] : 0u;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kBinThreads / 32; ++w) t += s_w[w];
    s_base = t;
  }
  // each thread scans 32 consecutive elements; then a block scan of the thread totals
  constexpr int kPer = kScanSeg / kBinThreads;
  uint32_t loc = 0;
#pragma unroll 8
  for (int i = 0; i < kPer; ++i) loc += seg[threadIdx.x * kPer + i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  __syncthreads();
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  uint32_t run = s_base;
  for (int w = 0; w < warp; ++w) run += s_w[w];
  run += incl - loc;
#pragma unroll 8
  for (int i = 0; i < kPer; ++i) {
    const uint32_t x = seg[threadIdx.x * kPer + i];
    seg[threadIdx.x * kPer + i] = run;
    run += x;
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < kScanSeg; i += kBinThreads)
    if (s0 + i < m) c[s0 + i] = seg[i];
  if (s0 + kScanSeg >= m && threadIdx.x == kBinThreads - 1) c[m] = run;   // last CTA: the total
}

// Phase 3: entries of CTA j's chunk, tile by tile: rank within the tile by ATOMS on the tile's bin
// counts, a block scan of those counts, a shared-memory counting sort, then bin-contiguous runs written
// at the CTA's running offset of each bin.
template <bool PREFIX>
__global__ void __launch_bounds__(kBinThreads) k_bin_scatter(const __grid_constant__ Geo G,
                                                             const __grid_constant__ BinGeo B,
                                                             const uint32_t* __restrict__ src,
                                                             const uint32_t* __restrict__ dst, uint64_t n, uint64_t per,
                                                             int vec, const uint32_t* __restrict__ offs,
                                                             uint32_t* __restrict__ entries) {
  extern __shared__ uint32_t sm[];
  uint32_t* base = sm;                                   // [nbins] next write offset of each bin
  uint32_t* toff = base + B.nbins;                       // [nbins + 1] tile counts → exclusive offsets
  uint32_t* stage = toff + B.nbins + 1;                  // [kBinTile] entries sorted by bin
  uint16_t* sbin = reinterpret_cast<uint16_t*>(stage + kBinTile);   // [kBinTile] their bins
  __shared__ uint32_t s_w[kBinThreads / 32];
  const uint32_t tid = threadIdx.x;
  for (uint32_t b = tid; b < B.nbins; b += kBinThreads) {
    base[b] = offs[(uint64_t)b * B.nblk + blockIdx.x];
    toff[b] = 0;
  }
  const uint64_t c0 = (uint64_t)blockIdx.x * per, c1 = min(n, c0 + per);
  const uint32_t per_thr = (B.nbins + kBinThreads - 1) / kBinThreads;   // bins scanned per thread
  __syncthreads();
  for (uint64_t t0 = c0; t0 < c1; t0 += kBinTile) {
    uint32_t key[kBinPPT], ent[kBinPPT];
#pragma unroll
    for (int q = 0; q < kBinPPT / 4; ++q) {
      uint32_t ss[4], dd[4];
      bool in[4];
      load_quad(src, dst, t0 + 4ull * ((uint64_t)q * kBinThreads + tid), c1, vec, ss, dd, in);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        uint32_t bin = 0, en = 0;
        const bool ok = in[e] && pair_bin<PREFIX>(G, B, ss[e], dd[e], bin, en);
        key[4 * q + e] = ok ? (bin << kBinRankBits) | atomicAdd(&toff[bin], 1u) : 0xffffffffu;
        ent[4 * q + e] = en;
      }
    }
    __syncthreads();
    // exclusive scan of toff[0, nbins): thread t owns bins [t·per_thr, (t+1)·per_thr)
    {
      const uint32_t b0 = tid * per_thr, b1 = min(B.nbins, b0 + per_thr);
      uint32_t loc = 0;
      for (uint32_t b = b0; b < b1; ++b) loc += toff[b];
      uint32_t tot;
      const int lane = tid & 31, warp = tid >> 5;
      uint32_t incl = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) s_w[warp] = incl;
      __syncthreads();
      uint32_t run = incl - loc;
      tot = 0;
      for (int w = 0; w < kBinThreads / 32; ++w) {
        run += w < warp ? s_w[w] : 0u;
        tot += s_w[w];
      }
      for (uint32_t b = b0; b < b1; ++b) {
        const uint32_t x = toff[b];
        toff[b] = run;
        run += x;
      }
      if (tid == 0) toff[B.nbins] = tot;
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
    const uint32_t total = toff[B.nbins];
    for (uint32_t p = tid; p < total; p += kBinThreads) {
      const uint32_t b = sbin[p];
      entries[base[b] + (p - toff[b])] = stage[p];
    }
    __syncthreads();
    for (uint32_t b = tid; b < B.nbins; b += kBinThreads) base[b] += toff[b + 1] - toff[b];
    __syncthreads();
    for (uint32_t b = tid; b < B.nbins; b += kBinThreads) toff[b] = 0;
    __syncthreads();
  }
}

// Column of array a for LP (P:235 RA: CL_bs window of LP; P:239 VA: H_j(LP)).
__device__ __forceinline__ uint32_t lp_col(const Geo& G, uint64_t dbl, uint32_t lp, uint32_t a) {
  return a < G.num_ra ? (uint32_t)(dbl >> G.sh[a]) & G.colmask[a]
                      : mix32(lp ^ G.va_seeds[a - G.num_ra]) & G.colmask[a];
}

// Phase 4: one CTA per word group (cs, w): its bins' entries set bits in a shared-memory image of the
// group (word i = word w of column i of CS cs, columns of all arrays in S:116 order), which is then
// OR-ed into the cube.  The CTA owns those words for the whole launch.  <3, 1>: paper shape unrolled.
template <int NRA, int NVA>
__global__ void __launch_bounds__(kApplyThreads) k_bin_apply(const __grid_constant__ Geo G,
                                                             const __grid_constant__ BinGeo B,
                                                             const uint32_t* __restrict__ offs,
                                                             const uint32_t* __restrict__ entries,
                                                             uint32_t* __restrict__ cube) {
  extern __shared__ uint32_t sub[];
  const uint32_t wg = blockIdx.x, cs = wg >> G.wpc_log2, w = wg & (G.wpc - 1u);
  for (uint32_t i = threadIdx.x; i < B.ncols; i += kApplyThreads) sub[i] = 0;
  uint32_t cbase[CBAA_MAX_ARRAYS];
  const uint32_t narr = NRA ? (uint32_t)(NRA + NVA) : G.narr;
#pragma unroll
  for (uint32_t a = 0; a < CBAA_MAX_ARRAYS; ++a) cbase[a] = a < narr ? G.arr_off[a] >> G.wpc_log2 : 0u;
  __syncthreads();
  const uint32_t kb = 1u << (5 - B.s), b0 = (cs << B.bpc_log2) + w * kb, smask = (1u << B.s) - 1u;
  for (uint32_t k = 0; k < kb; ++k) {
    const uint32_t p0 = offs[(uint64_t)(b0 + k) * B.nblk], p1 = offs[(uint64_t)(b0 + k + 1) * B.nblk];
    const uint32_t hi = k << B.s;
    for (uint32_t p = p0 + threadIdx.x; p < p1; p += 4 * kApplyThreads) {
      uint32_t e[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t q = p + u * kApplyThreads;
        e[u] = q < p1 ? __ldcs(entries + q) : 0xffffffffu;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (p + u * kApplyThreads >= p1) continue;
        const uint32_t lp = e[u] >> B.s, bit = 1u << (hi | (e[u] & smask));
        const uint64_t dbl = ((uint64_t)lp << G.L) | lp;
        if constexpr (NRA > 0) {
#pragma unroll
          for (int a = 0; a < NRA + NVA; ++a) {
            const uint32_t col = a < NRA ? (uint32_t)(dbl >> G.sh[a]) & G.colmask[a]
                                         : mix32(lp ^ G.va_seeds[a - NRA]) & G.colmask[a];
            uint32_t* x = sub + cbase[a] + col;
            if (!(*x & bit)) atomicOr(x, bit);
          }
        } else {
          for (uint32_t a = 0; a < narr; ++a) {
            uint32_t* x = sub + (G.arr_off[a] >> G.wpc_log2) + lp_col(G, dbl, lp, a);
            if (!(*x & bit)) atomicOr(x, bit);
          }
        }
      }
    }
  }
  __syncthreads();
  uint32_t* cw = cube + (uint64_t)cs * G.cs_words + w;
  for (uint32_t i = threadIdx.x; i < B.ncols; i += kApplyThreads) {
    const uint32_t v = sub[i];
    if (v) red_or(cw + (uint64_t)i * G.wpc, v);
  }
}

}  // namespace cbaa
