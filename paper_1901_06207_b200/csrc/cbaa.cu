// libcbaa.so — host side of the C ABI declared in include/cbaa.h.
// Validation, handle/scratch ownership, launch configuration, the double-buffered
// host-ingest pipeline, and result ordering.  All per-pair, per-column and per-tuple
// work runs in the sm_100a kernels of kernels.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <type_traits>
#include <vector>

#include "cbaa.h"
#include "geometry.cuh"
#include "kernels.cuh"
#include "binned.cuh"

using namespace cbaa;

struct DetectKey {   // what a captured detect graph depends on (θ is not part of it: see hot_node)
  uint32_t cs_lo = 0, cs_hi = 0;
  int record = 0;
  const void* cand = nullptr;
  const void* h_res = nullptr;
  int join = 0;
  bool operator==(const DetectKey& o) const {
    return cs_lo == o.cs_lo && cs_hi == o.cs_hi && record == o.record && cand == o.cand &&
           h_res == o.h_res && join == o.join;
  }
};

struct DetectGraph {
  cudaGraph_t graph = nullptr;          // kept alive: hot_node belongs to it
  cudaGraphExec_t exec = nullptr;
  DetectKey key{};
  cudaGraphNode_t hot_node = nullptr;   // the k_hot node: θ is set per detect by a kernel-node parameter update
  cudaKernelNodeParams hot_params{};
  uint32_t theta = 0;                   // θ currently in the instantiated graph
  int kernels = 0;
};

struct cbaa_handle {
  cbaa_config cfg;
  Geo G;
  int device = 0;
  int sms = 148;
  int l2_bytes = 0;
  uint32_t passes = 1;
  uint32_t* cube = nullptr;
  bool cube_external = false;   // cube memory owned by the caller (cbaa_create_ext)
  uint32_t* prefix_bits = nullptr;   // a0 classifier bitmaps (direction = inner prefix)
  uint64_t cube_bytes = 0;
  uint64_t cube_words = 0;
  // detect scratch (one allocation, see alloc_scratch)
  void* scratch = nullptr;
  DetectScratch D{};
  unsigned long long* skipped = nullptr;
  // pinned host staging
  cbaa_cs_stats* h_rec = nullptr;
  unsigned long long* h_cnt = nullptr;
  void* h_res = nullptr;        // pinned mirror of the device result block
  cbaa_host* h_hits = nullptr;  // = h_res + 64
  uint64_t h_hits_cap = 0;
  // candidate recording (debug)
  int record = 0;
  int force_cartesian = 0;   // CBAA_FORCE_CARTESIAN=1: use k_tuples even for |RA| = 3 (A/B testing)
  int no_tma = 0;            // CBAA_NO_TMA=1: register-load zero counts instead of the TMA pipeline (A/B)
  // host-ingest pipeline
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
  uint32_t* stage[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  uint64_t stage_pairs = 0;
  uint64_t launches = 0;
  int upd_blocks = 0;
  // detect graphs (captured on cap_stream, launched on the caller's stream): [0] full, [1] without the
  // zero-count pass (its counts came from cbaa_merge_slice_zc)
  cudaStream_t cap_stream = nullptr;
  DetectGraph dgs[2];
  int zc_fresh = 0;                     // zc holds the zero counts of CSs [zc_lo, zc_hi) of the current cube
  uint32_t zc_lo = 0, zc_hi = 0;
  // device barrier (cbaa_peer_barrier): signal area after the cube in the same allocation
  unsigned long long* sig = nullptr;
  int use_join = 0;          // |RA| = 3 and not forced Cartesian
  // binned update (CBAA_UPDATE_BINNED, binned.cuh)
  BinGeo B{};
  int binnable = 0;          // geometry fits the binned kernels' shared-memory tables
  uint64_t bin_min = 0;      // fewer pairs per call than this take the direct kernel
  uint64_t bin_chunk = 1ull << 28;   // pairs per count/scatter/apply round (CBAA_BIN_CHUNK, tests)
  uint32_t* bin_ent = nullptr;
  uint64_t bin_cap = 0;
  uint32_t* bin_tab = nullptr;    // counts | start | cursor | log count
  void* bin_log = nullptr;        // k_bin_wc overflow log
  int bin_wc = 0;                 // scatter: tile sort k_bin_scatter (0, default) or write-combining k_bin_wc (1)
  int bin_wide = 0;               // the paper configuration: 64-bit entries, 1024 bins (k_bin_scatter_w, binned.cuh)
  int bin_wide_gen = 0;           // other geometries with 256-2048 wide bins (k_bin_scatter_w<·, NB>, k_bin_apply_wg)
  int bin_narrow_ok = 0;          // the 32-bit-entry kernels' tables fit (nbins ≤ 4096, Σc(i) ≤ 28672)
  int bin_gen_ok = 0;             // the generic wide kernels fit
  int bin_gen_pref = 0;           // ... and are preferred over the 32-bit-entry kernels
  int bin_gen_per_array = 0;      // ... with one apply CTA per (bin, array): Σc(i) > 16384 (k_bin_apply_wa)
  BinGeo BW{};                    // bin geometry of the wide path
  uint32_t sample_ctas = 0;       // k_bin_sample grid (0: one CTA per SM; CBAA_SAMPLE_CTAS)
  uint32_t scatter_pf = 1 | 1u << 8;   // k_bin_scatter_w L2 prefetch: distance in tiles | issue point << 8 (CBAA_SCATTER_PF)
  bool apply_paper = false;       // k_bin_apply<3, 1, 4, true>: the paper's default configuration
  uint32_t bin_sample_log2 = 9;   // regions sized from 8 pairs of every 2^L (0: exact count; CBAA_BIN_SAMPLE)
  uint64_t bin_sample_min = 1ull << 24;   // chunks with fewer pairs are counted exactly (CBAA_BIN_SAMPLE_MIN)
  // per-kernel update timing (cbaa_set_phase_timing)
  int timing = 0;
  std::vector<cudaEvent_t> tev;   // pairs: tev[2k], tev[2k+1]
  std::vector<int> tphase;        // phase of pair k
  size_t tused = 0;
  uint64_t tcalls = 0;
  std::string err;
};

namespace {

const char* g_codes[] = {"ok", "invalid config", "invalid argument", "CUDA error", "cube mismatch",
                         "output capacity exceeded", "tuple cap exceeded", "out of device memory"};

int fail(cbaa_handle* h, int code, const std::string& msg) {
  if (h) h->err = msg;
  return code;
}

int cuda_fail(cbaa_handle* h, cudaError_t e, const char* what) {
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  if (h) h->err = m;
  return e == cudaErrorMemoryAllocation ? CBAA_E_NOMEM : CBAA_E_CUDA;
}

#define CK(h, call)                                      \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(h, e_, #call); \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

bool pow2(uint64_t x) { return x && !(x & (x - 1)); }

// EP/CP lengths: |EP(i)| = CL_bs((i+1) mod |RA|) − CL_bs(i) mod L (Q6); |CP(i)| = cbn(i) − |EP(i)|.
void ep_cp(const cbaa_config& c, int* ep, int* cp) {
  int L = 32 - (int)c.r;
  for (uint32_t i = 0; i < c.num_ra; ++i) {
    int e = ((int)c.clbs[(i + 1) % c.num_ra] - (int)c.clbs[i]) % L;
    if (e < 0) e += L;
    ep[i] = e;
    cp[i] = (int)c.cbn[i] - e;
  }
}

int validate(const cbaa_config* c, std::string* why) {
  auto bad = [&](const char* m) {
    if (why) *why = m;
    return CBAA_E_CONFIG;
  };
  if (!c) return bad("config is null");
  if (c->r > 16) return bad("r must be <= 16");
  if (c->num_ra < 2 || c->num_ra > CBAA_MAX_RA) return bad("num_ra must be in [2, 8] (a single RA cannot restore LP, S:66)");
  if (c->num_va > CBAA_MAX_VA) return bad("num_va must be <= 8");
  if (!pow2(c->g) || c->g < 32) return bad("g must be a power of two >= 32 (S:40, Q28)");
  if (!(c->mangle_a & 1u)) return bad("mangle_a must be odd (S:40)");
  int L = 32 - (int)c->r;
  for (uint32_t i = 0; i < c->num_ra + c->num_va; ++i)
    if (c->cbn[i] < 1 || (int)c->cbn[i] > L || c->cbn[i] > 24) return bad("cbn(i) must be in [1, min(L, 24)]");
  for (uint32_t i = 0; i < c->num_ra; ++i) {
    if ((int)c->clbs[i] >= L) return bad("clbs(i) must be < L = 32 - r (Q6)");
    if (i && c->clbs[i] <= c->clbs[i - 1]) return bad("clbs must be strictly increasing (S:41)");
  }
  int ep[CBAA_MAX_RA], cp[CBAA_MAX_RA], sum = 0;
  ep_cp(*c, ep, cp);
  for (uint32_t i = 0; i < c->num_ra; ++i) sum += ep[i];
  if (sum != L) return bad("sum of ep(i) must equal L = 32 - r (S:38)");
  for (uint32_t i = 0; i < c->num_ra; ++i) {
    if (cp[i] < 0) return bad("cp(i) = cbn(i) - ep(i) must be >= 0 (S:39)");
    if (cp[i] > ep[(i + 1) % c->num_ra]) return bad("cp(i) must be <= ep((i+1) mod num_ra) (S:39)");
  }
  if (c->theta_formula != CBAA_THETA_PAPER && c->theta_formula != CBAA_THETA_INVERTED)
    return bad("theta_formula must be CBAA_THETA_PAPER or CBAA_THETA_INVERTED");
  if (c->union_threshold != CBAA_UNION_SAME && c->union_threshold != CBAA_UNION_THM2)
    return bad("union_threshold must be CBAA_UNION_SAME or CBAA_UNION_THM2 (Q20)");
  if (c->direction != CBAA_DIR_NORMALIZED && c->direction != CBAA_DIR_INNER_PREFIX)
    return bad("direction must be CBAA_DIR_NORMALIZED or CBAA_DIR_INNER_PREFIX");
  if (c->n_prefixes > CBAA_MAX_PREFIXES) return bad("at most 16 inner prefixes");
  for (uint32_t k = 0; k < c->n_prefixes && k < CBAA_MAX_PREFIXES; ++k) {
    const uint32_t m = c->inner_mask[k];
    if ((~m) & ((~m) + 1u)) return bad("inner_mask must be a CIDR mask (leading ones, then zeros)");
  }
  if (c->update_mode != CBAA_UPDATE_TEST_SET && c->update_mode != CBAA_UPDATE_RED &&
      c->update_mode != CBAA_UPDATE_BINNED)
    return bad("update_mode must be CBAA_UPDATE_TEST_SET, CBAA_UPDATE_RED or CBAA_UPDATE_BINNED");
  uint64_t csb = 0;
  for (uint32_t a = 0; a < c->num_ra + c->num_va; ++a) csb += ((uint64_t)1 << c->cbn[a]) * c->g;
  if ((csb << c->r) / 8 > (16ull << 30) - 16) return bad("cube must be smaller than 16 GiB");
  // reset/merge/zero-count kernels move 16-byte words and address CS slices directly: every CS must be
  // a whole number of them (only g = 32 with a 2-column array can miss this)
  if ((csb / 8) % 16 != 0) return bad("bytes per CS (sum of c(i)*g/8) must be a multiple of 16 (GPU word layout)");
  return CBAA_OK;
}

uint32_t inv_mod32(uint32_t a) {   // Newton iteration for the inverse of odd a modulo 2^32
  uint32_t x = a;
  for (int k = 0; k < 5; ++k) x *= 2u - a * x;
  return x;
}

Geo derive(const cbaa_config& c) {
  Geo G;
  std::memset(&G, 0, sizeof G);
  G.r = c.r;
  G.L = 32 - c.r;
  G.num_ra = c.num_ra;
  G.num_va = c.num_va;
  G.narr = c.num_ra + c.num_va;
  G.g = c.g;
  G.wpc = c.g / 32;
  while ((1u << G.wpc_log2) < G.wpc) ++G.wpc_log2;
  G.n_cs = 1u << c.r;
  G.rmask = G.n_cs - 1u;
  uint32_t off = 0;
  for (uint32_t a = 0; a < G.narr; ++a) {
    G.arr_off[a] = off;
    G.cbn[a] = c.cbn[a];
    G.ncols[a] = 1u << c.cbn[a];
    G.colmask[a] = G.ncols[a] - 1u;
    off += G.ncols[a] * G.wpc;
  }
  G.cs_words = off;
  int ep[CBAA_MAX_RA], cp[CBAA_MAX_RA];
  ep_cp(c, ep, cp);
  uint32_t raoff = 0;
  for (uint32_t i = 0; i < c.num_ra; ++i) {
    G.clbs[i] = c.clbs[i];
    G.ep[i] = (uint32_t)ep[i];
    G.cp[i] = (uint32_t)cp[i];
    G.sh[i] = 2 * G.L - c.clbs[i] - c.cbn[i];
    G.ra_off[i] = raoff;
    raoff += G.ncols[i];
  }
  G.ra_cols = raoff;
  G.mangle_a = c.mangle_a;
  G.mangle_b = c.mangle_b;
  G.inv_a = inv_mod32(c.mangle_a);
  G.bv_seed = c.bv_seed;
  for (uint32_t j = 0; j < c.num_va; ++j) G.va_seeds[j] = c.va_seeds[j];
  G.direction = c.direction;
  G.theta_formula = c.theta_formula;
  G.union_threshold = c.union_threshold;
  G.n_prefix = c.n_prefixes;
  for (uint32_t k = 0; k < c.n_prefixes; ++k) {
    G.prefix[k] = c.inner_prefix[k] & c.inner_mask[k];
    G.pmask[k] = c.inner_mask[k];
  }
  G.tuple_cap = c.tuple_cap;
  return G;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int alloc_scratch(cbaa_handle* h) {
  const Geo& G = h->G;
  const size_t n_cs = G.n_cs;
  const uint32_t hit_cap = h->cfg.hit_capacity ? h->cfg.hit_capacity : (1u << 20);
  // counters: done[n_cs] done_all n_cand n_join (zeroed inside each detect), skipped (zeroed by reset)
  size_t off = 0;
  size_t o_done = off;
  off += align_up(n_cs * 4, 8);
  size_t o_done_all = off;
  off += 8;
  size_t o_ncand = off;
  off += 8;
  size_t o_njoin = off;
  off += 8;
  size_t o_skipped = off;
  off += 8;
  off = align_up(off, 256);
  size_t o_rec = off;
  off += align_up(n_cs * sizeof(cbaa_cs_stats), 256);
  size_t o_prefix = off;
  off += align_up((n_cs + 1) * 8, 256);
  size_t o_units = off;
  off += align_up(n_cs * 8, 256);
  // (cs, lp) chains of the join: 2^22 = 32 MiB by default; beyond it detect falls back (cbaa_detect_range)
  const uint64_t join_cap = h->cfg.join_capacity ? h->cfg.join_capacity : (1ull << 22);
  size_t o_join = off;
  off += align_up(join_cap * 8, 256);
  size_t o_zc = off;
  off += align_up(n_cs * G.ra_cols * 4, 256);
  size_t o_hc = off;
  off += align_up(n_cs * G.ra_cols * 4, 256);
  size_t o_nhits = off;            // result block: [n_hits | pad to 64 B | hits ...], copied to the host in one go
  size_t o_hits = off + 64;
  off += 64 + align_up((size_t)hit_cap * sizeof(cbaa_host), 256);
  char* base = nullptr;
  CK(h, cudaMalloc(&base, off));
  CK(h, cudaMemset(base, 0, off));
  h->scratch = base;
  DetectScratch& D = h->D;
  D.done = (unsigned int*)(base + o_done);
  D.done_all = (unsigned int*)(base + o_done_all);
  D.n_hits = (unsigned long long*)(base + o_nhits);
  D.n_cand = (unsigned long long*)(base + o_ncand);
  h->skipped = (unsigned long long*)(base + o_skipped);
  D.rec = (cbaa_cs_stats*)(base + o_rec);
  D.prefix = (unsigned long long*)(base + o_prefix);
  D.units = (unsigned long long*)(base + o_units);
  D.n_join = (unsigned long long*)(base + o_njoin);
  D.join = (unsigned long long*)(base + o_join);
  D.join_cap = join_cap;
  D.zc = (uint32_t*)(base + o_zc);
  D.hc = (uint32_t*)(base + o_hc);
  D.hits = (cbaa_host*)(base + o_hits);
  D.hit_cap = hit_cap;
  D.cand = nullptr;
  D.cand_cap = 0;
  CK(h, cudaMallocHost(&h->h_rec, n_cs * sizeof(cbaa_cs_stats) + 64));
  CK(h, cudaMallocHost(&h->h_cnt, 64));
  h->h_hits_cap = 4096;
  CK(h, cudaMallocHost(&h->h_res, 64 + h->h_hits_cap * sizeof(cbaa_host)));
  h->h_hits = (cbaa_host*)((char*)h->h_res + 64);
  return CBAA_OK;
}

// The a0 classifier's two 65536-bit maps over the top 16 address bits (see Geo::full_bits).
int upload_prefix_bits(cbaa_handle* h) {
  std::vector<uint32_t> bits(2 * 2048, 0);
  uint32_t* full = bits.data();
  uint32_t* part = bits.data() + 2048;
  for (uint32_t k = 0; k < h->cfg.n_prefixes; ++k) {
    const uint32_t m = h->cfg.inner_mask[k], pre = h->cfg.inner_prefix[k] & m;
    const uint32_t len = (uint32_t)__builtin_popcount(m);
    if (len <= 16) {   // covers whole top-16 buckets
      const uint32_t lo = pre >> 16, cnt = 1u << (16 - len);
      for (uint32_t t = lo; t < lo + cnt; ++t) full[t >> 5] |= 1u << (t & 31);
    } else {
      const uint32_t t = pre >> 16;
      part[t >> 5] |= 1u << (t & 31);
    }
  }
  void* d = nullptr;
  CK(h, cudaMalloc(&d, bits.size() * 4));
  CK(h, cudaMemcpy(d, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice));
  h->prefix_bits = (uint32_t*)d;
  h->G.full_bits = h->prefix_bits;
  h->G.part_bits = h->prefix_bits + 2048;
  return CBAA_OK;
}

int launch_check(cbaa_handle* h, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(h, e, what);
  ++h->launches;
  return CBAA_OK;
}

int grid_for(const cbaa_handle* h, uint64_t work_items, int per_sm) {
  uint64_t want = (work_items + kThreads - 1) / kThreads;
  uint64_t cap = (uint64_t)h->sms * per_sm;
  return (int)std::max<uint64_t>(1, std::min(want, cap));
}

// Calls f(NRA, NVA, MODE, PREFIX) with the compile-time variant of the update kernels that matches the
// handle: the paper shape (|RA| = 3, |VA| = 1) or the generic geometry, test-and-set or plain RED, and
// normalised or inner-prefix input.
template <class F>
void dispatch_update(const cbaa_handle* h, F&& f) {
  using T = std::integral_constant<int, CBAA_UPDATE_TEST_SET>;
  using R = std::integral_constant<int, CBAA_UPDATE_RED>;
  const bool prefix = h->cfg.direction == CBAA_DIR_INNER_PREFIX;
  const bool test = h->cfg.update_mode != CBAA_UPDATE_RED;   // BINNED falls back to test-and-set
  auto go = [&](auto nra, auto nva) {
    if (test) {
      if (prefix) f(nra, nva, T{}, std::true_type{});
      else f(nra, nva, T{}, std::false_type{});
    } else {
      if (prefix) f(nra, nva, R{}, std::true_type{});
      else f(nra, nva, R{}, std::false_type{});
    }
  };
  using RT = std::integral_constant<int, -1>;   // RA/VA split at run time
  const uint32_t na = h->G.narr;
  if (h->G.num_ra == 3 && h->G.num_va == 1) go(std::integral_constant<int, 3>{}, std::integral_constant<int, 1>{});
  else if (na == 2) go(std::integral_constant<int, 2>{}, RT{});
  else if (na == 3) go(std::integral_constant<int, 3>{}, RT{});
  else if (na == 4) go(std::integral_constant<int, 4>{}, RT{});
  else if (na == 5) go(std::integral_constant<int, 5>{}, RT{});
  else if (na == 6) go(std::integral_constant<int, 6>{}, RT{});
  else go(std::integral_constant<int, 0>{}, std::integral_constant<int, 0>{});
}

// One pass of Alg. 1 over n device pairs, restricted to cube words [lo, lo+span).
int launch_update(cbaa_handle* h, const uint32_t* src, const uint32_t* dst, uint64_t n, uint32_t lo, uint32_t span,
                  bool count_skips, cudaStream_t s) {
  uint64_t head = 0;
  uintptr_t as = (uintptr_t)src, ad = (uintptr_t)dst;
  bool vec = (as % 4 == 0) && (as % 16 == ad % 16);
  if (vec) head = std::min<uint64_t>(n, ((16 - as % 16) % 16) / 4);
  uint64_t n4 = vec ? (n - head) / 4 : 0;
  if (!vec) head = n;   // everything scalar
  uint64_t scalar = head + (n - head - 4 * n4);
  const int grid = grid_for(h, std::max(n4, scalar), h->upd_blocks);
  unsigned long long* sk = count_skips ? h->skipped : nullptr;
  dispatch_update(h, [&](auto nra, auto nva, auto mode, auto pfx) {
    k_update<decltype(nra)::value, decltype(nva)::value, decltype(mode)::value, decltype(pfx)::value>
        <<<grid, kThreads, 0, s>>>(h->G, src, dst, head, n4, n, h->cube, lo, span, sk);
  });
  return launch_check(h, "k_update");
}

// One pass of Alg. 1 over n interleaved device pairs (src, dst, src, dst, ...).
int launch_update_aos(cbaa_handle* h, const uint32_t* pairs, uint64_t n, uint32_t lo, uint32_t span,
                      bool count_skips, cudaStream_t s) {
  const uintptr_t a = (uintptr_t)pairs;
  const uint64_t head = std::min<uint64_t>(n, (a & 15) ? 1 : 0);   // 8-B aligned: at most one pair to peel
  const uint64_t n8 = (n - head) / 8;
  const uint64_t scalar = head + (n - head - 8 * n8);
  const int grid = grid_for(h, std::max(n8, scalar), h->upd_blocks);
  unsigned long long* sk = count_skips ? h->skipped : nullptr;
  const uint2* p2 = (const uint2*)pairs;
  dispatch_update(h, [&](auto nra, auto nva, auto mode, auto pfx) {
    k_update_aos<decltype(nra)::value, decltype(nva)::value, decltype(mode)::value, decltype(pfx)::value>
        <<<grid, kThreads, 0, s>>>(h->G, p2, head, n8, n, h->cube, lo, span, sk);
  });
  return launch_check(h, "k_update_aos");
}

// Phase timing: t_begin records the start event of the next kernel (returns its slot, or -1 when off);
// t_end records its end.
int t_begin(cbaa_handle* h, int phase, cudaStream_t s) {
  if (!h->timing) return -1;
  if (h->tused == h->tphase.size()) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return -1;
    h->tev.push_back(a);
    h->tev.push_back(b);
    h->tphase.push_back(0);
  }
  const size_t k = h->tused++;
  h->tphase[k] = phase;
  cudaEventRecord(h->tev[2 * k], s);
  return (int)k;
}
void t_end(cbaa_handle* h, int k, cudaStream_t s) {
  if (k >= 0) cudaEventRecord(h->tev[2 * k + 1], s);
}

// the binned path can run: wide entries (paper or generic geometry), or the 32-bit-entry kernels' tables fit
bool binned_ok(const cbaa_handle* h) {
  const bool wide = (h->bin_wide || h->bin_wide_gen) && !h->bin_wc;
  return h->binnable && (wide || h->bin_narrow_ok);
}

// the largest dynamic shared memory a kernel may request: the opt-in maximum less its static shared memory
void set_dyn_smem_max(const void* f, int smax) {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, f) == cudaSuccess)
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smax - (int)fa.sharedSizeBytes);
}

template <int NB>
void set_wscatter_attrs(int smax) {
  set_dyn_smem_max((const void*)k_bin_scatter_w<false, NB>, smax);
  cudaFuncSetAttribute(k_bin_scatter_w<false, NB>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  set_dyn_smem_max((const void*)k_bin_scatter_w<true, NB>, smax);
  cudaFuncSetAttribute(k_bin_scatter_w<true, NB>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

// Launch of the wide scatter: NB < 0 the paper geometry, else the bin count of a generic wide geometry.
template <int NB>
void launch_wscatter(bool prefix, const Geo& G, uint32_t nblk, cudaStream_t s, const uint32_t* a, const uint32_t* b,
                     uint64_t m, uint64_t per, int vec, uint32_t* cursor, uint64_t* ent, const uint32_t* start,
                     uint32_t* log_n, uint64_t* lg, unsigned long long* skipped, uint32_t pf) {
  const uint32_t nb = NB < 0 ? (uint32_t)kWBins : (uint32_t)NB;
  if (prefix)
    k_bin_scatter_w<true, NB><<<nblk, kBinThreads, wscatter_smem(nb, true), s>>>(G, a, b, m, per, vec, cursor, ent, start,
                                                                                 log_n, lg, skipped, pf);
  else
    k_bin_scatter_w<false, NB><<<nblk, kBinThreads, wscatter_smem(nb, false), s>>>(G, a, b, m, per, vec, cursor, ent,
                                                                                   start, log_n, lg, nullptr, pf);
}

// Binned update (binned.cuh): count → starts → scatter → apply, in chunks of at most 2^28 pairs.
int update_binned(cbaa_handle* h, const uint32_t* src, const uint32_t* dst, uint64_t n, cudaStream_t s) {
  const uint64_t kChunk = h->bin_chunk;
  const bool prefix = h->cfg.direction == CBAA_DIR_INNER_PREFIX;
  const bool wide = (h->bin_wide || h->bin_wide_gen) && !h->bin_wc;   // 64-bit entries, (cs, row >> 6) bins
  const BinGeo& B = wide ? h->BW : h->B;
  // + per bin: sector alignment and the write-combining scatter's duplicate padding (8 per CTA)
  const uint32_t slack = h->bin_wc ? 8u * (uint32_t)h->sms : 0u;
  // sampled region sizing (k_bin_sample): normalised input, tile scatter, chunks of ≥ bin_sample_min pairs
  // (prefix mode: only on the wide path, whose scatter counts the skipped pairs itself)
  const uint32_t samp = ((!prefix || wide) && !h->bin_wc) ? h->bin_sample_log2 : 0u;
  const uint64_t mx = std::min(n, kChunk);
  const bool any_sampled = samp && mx >= h->bin_sample_min;
  // Σ cap(b) ≤ exact: m + nbins·(slack + 7); sampled (Σ est ≤ m + 2^L, Cauchy-Schwarz on the √ terms):
  // 1.25·(m + 2^L) + 2·√(nbins·2^L·(m + 2^L)) + nbins·(64 + slack + 7 + 2 for sqrtf rounding)
  const double sm_ = (double)(mx + (1ull << samp));
  const uint64_t want = std::max<uint64_t>(
      mx + (uint64_t)(slack + 8) * B.nbins,
      any_sampled ? (uint64_t)(1.25 * sm_ + 2.0 * std::sqrt((double)B.nbins * (double)(1ull << samp) * sm_)) +
                        (uint64_t)(slack + 80) * B.nbins + 64   // + 7 alignment, + sqrtf rounding per bin
                  : 0);
  if (h->bin_cap < want) {
    if (h->bin_ent) CK(h, cudaFree(h->bin_ent));
    h->bin_ent = nullptr;
    h->bin_cap = 0;
    CK(h, cudaMalloc(&h->bin_ent, want * 8));   // 8 B per entry: either entry width fits
    if (h->bin_log) CK(h, cudaFree(h->bin_log));
    h->bin_log = nullptr;
    // overflow log: u32 entries | u16 bins, or u64 records (wide)
    CK(h, cudaMalloc(&h->bin_log, std::min(n, kChunk) * 8 + 16));
    h->bin_cap = want;   // only once both buffers exist (a failed allocation is retried on the next call)
  }
  if (!h->bin_tab) {   // counts [nbins] | start [nbins + 1] | cursor [nbins · kCurStride] | log count
    const uint64_t nb = std::max(h->B.nbins, h->BW.nbins);   // one table serves both entry widths
    CK(h, cudaMalloc(&h->bin_tab, ((2ull + kCurStride) * nb + 2) * 4));
    CK(h, cudaMemsetAsync(h->bin_tab, 0, nb * 4, s));
  }
  uint32_t* counts = h->bin_tab;
  uint32_t* start = counts + B.nbins;
  uint32_t* cursor = start + B.nbins + 1;
  uint32_t* log_n = cursor + (uint64_t)B.nbins * kCurStride;
  uint32_t* log_e = reinterpret_cast<uint32_t*>(h->bin_log);
  uint16_t* log_b = reinterpret_cast<uint16_t*>(log_e + std::min(n, kChunk));
  const size_t sm_cnt = (size_t)B.nbins * 4;
  const size_t sm_sc = (size_t)(3 * B.nbins + 1) * 4 + (size_t)kBinTile * 6;
  const size_t sm_wc = wc_smem_bytes(B.nbins);
  const size_t sm_ap = (size_t)B.ncols * 4;
  const uint32_t n_wg = h->G.n_cs * h->G.wpc;
  for (uint64_t off = 0; off < n; off += kChunk) {
    const uint64_t m = std::min(kChunk, n - off);
    const uint32_t* a = src + off;
    const uint32_t* b = dst + off;
    const uint64_t per = (((m + B.nblk - 1) / B.nblk) + 3) & ~3ull;
    const int vec = ((uintptr_t)a % 16 == 0) && ((uintptr_t)b % 16 == 0);
    const uint32_t nc = 2 * (uint32_t)h->sms;   // count grid: any chunking works (global totals)
    const uint64_t per_c = (((m + nc - 1) / nc) + 3) & ~3ull;
    const uint32_t sl = samp && m >= h->bin_sample_min ? samp : 0u;
    int tk = t_begin(h, 0, s);
    const uint32_t ns = h->sample_ctas ? h->sample_ctas : (uint32_t)h->sms;   // 1.5 µs faster than 2 per SM
    if (sl && prefix)
      k_bin_sample<true><<<ns, kCountThreads, sm_cnt, s>>>(h->G, B, a, b, m, sl, vec, counts);
    else if (sl)
      k_bin_sample<false><<<ns, kCountThreads, sm_cnt, s>>>(h->G, B, a, b, m, sl, vec, counts);
    else if (prefix)
      k_bin_count<true><<<nc, kCountThreads, sm_cnt, s>>>(h->G, B, a, b, m, per_c, vec, counts, h->skipped);
    else
      k_bin_count<false><<<nc, kCountThreads, sm_cnt, s>>>(h->G, B, a, b, m, per_c, vec, counts, nullptr);
    t_end(h, tk, s);
    int rc = launch_check(h, sl ? "k_bin_sample" : "k_bin_count");
    if (rc) return rc;
    tk = t_begin(h, 1, s);
    k_bin_starts<<<1, kStartThreads, 0, s>>>(B.nbins, slack, sl, counts, start, cursor, log_n);
    t_end(h, tk, s);
    if ((rc = launch_check(h, "k_bin_starts"))) return rc;
    tk = t_begin(h, 2, s);
    if (wide) {
      auto* ent = (uint64_t*)h->bin_ent;
      auto* lgw = (uint64_t*)h->bin_log;
      unsigned long long* sk = sl ? h->skipped : nullptr;
      if (h->bin_wide)
        launch_wscatter<-1>(prefix, h->G, B.nblk, s, a, b, m, per, vec, cursor, ent, start, log_n, lgw, sk, h->scatter_pf);
      else if (B.nbins == 256)
        launch_wscatter<256>(prefix, h->G, B.nblk, s, a, b, m, per, vec, cursor, ent, start, log_n, lgw, sk, h->scatter_pf);
      else if (B.nbins == 512)
        launch_wscatter<512>(prefix, h->G, B.nblk, s, a, b, m, per, vec, cursor, ent, start, log_n, lgw, sk, h->scatter_pf);
      else if (B.nbins == 1024)
        launch_wscatter<1024>(prefix, h->G, B.nblk, s, a, b, m, per, vec, cursor, ent, start, log_n, lgw, sk, h->scatter_pf);
      else if (B.nbins == 2048)
        launch_wscatter<2048>(prefix, h->G, B.nblk, s, a, b, m, per, vec, cursor, ent, start, log_n, lgw, sk, h->scatter_pf);
      else
        launch_wscatter<4096>(prefix, h->G, B.nblk, s, a, b, m, per, vec, cursor, ent, start, log_n, lgw, sk, h->scatter_pf);
    } else if (h->bin_wc) {   // write-combining scatter (CBAA_BIN_SCATTER=wc), one CTA per SM
      const uint32_t nw = (uint32_t)h->sms;
      const uint64_t per_w = (((m + nw - 1) / nw) + 3) & ~3ull;
      if (prefix)
        k_bin_wc<true><<<nw, kWcThreads, sm_wc, s>>>(h->G, B, a, b, m, per_w, vec, cursor, h->bin_ent, log_n, log_e, log_b);
      else
        k_bin_wc<false><<<nw, kWcThreads, sm_wc, s>>>(h->G, B, a, b, m, per_w, vec, cursor, h->bin_ent, log_n, log_e, log_b);
    } else {           // tile counting sort (default)
      if (prefix)
        k_bin_scatter<true, 0><<<B.nblk, kBinThreads, sm_sc, s>>>(h->G, B, a, b, m, per, vec, cursor, h->bin_ent,
                                                                  start, log_n, log_e, log_b, h->scatter_pf);
      else if (B.nbins == 4096 && h->G.r == 4 && h->G.g == 4096)   // the paper geometry: constants inlined
        k_bin_scatter<false, -1><<<B.nblk, kBinThreads, sm_sc, s>>>(h->G, B, a, b, m, per, vec, cursor, h->bin_ent,
                                                                    start, log_n, log_e, log_b, h->scatter_pf);
      else if (B.nbins == 4096)   // bin loops with compile-time trip counts
        k_bin_scatter<false, 4096><<<B.nblk, kBinThreads, sm_sc, s>>>(h->G, B, a, b, m, per, vec, cursor, h->bin_ent,
                                                                      start, log_n, log_e, log_b, h->scatter_pf);
      else
        k_bin_scatter<false, 0><<<B.nblk, kBinThreads, sm_sc, s>>>(h->G, B, a, b, m, per, vec, cursor, h->bin_ent,
                                                                   start, log_n, log_e, log_b, h->scatter_pf);
    }
    t_end(h, tk, s);
    if ((rc = launch_check(h, h->bin_wc ? "k_bin_wc" : "k_bin_scatter"))) return rc;
    tk = t_begin(h, 3, s);
    if (wide && h->bin_wide)
      k_bin_apply_w<<<B.nbins, kWApplyThreads, kWApplySmem, s>>>(h->G, start, cursor, (const uint64_t*)h->bin_ent,
                                                                 h->cube);
    else if (wide && h->bin_gen_per_array) {
      uint32_t maxc = 0;
      for (uint32_t q = 0; q < h->G.narr; ++q) maxc = std::max(maxc, h->G.ncols[q]);
      k_bin_apply_wa<<<B.nbins * h->G.narr, kWApplyThreads, (size_t)maxc * 8, s>>>(h->G, start, cursor,
                                                                                 (const uint64_t*)h->bin_ent, h->cube);
    } else if (wide && h->G.num_ra == 3 && h->G.num_va == 1)
      k_bin_apply_wg<3, 1><<<B.nbins, kWApplyThreads, (size_t)B.ncols * 8, s>>>(h->G, B.ncols, start, cursor,
                                                                              (const uint64_t*)h->bin_ent, h->cube);
    else if (wide)
      k_bin_apply_wg<0, 0><<<B.nbins, kWApplyThreads, (size_t)B.ncols * 8, s>>>(h->G, B.ncols, start, cursor,
                                                                              (const uint64_t*)h->bin_ent, h->cube);
    else if (h->apply_paper)
      k_bin_apply<3, 1, 4, true><<<n_wg, kApplyThreads, sm_ap, s>>>(h->G, B, start, cursor, h->bin_ent, h->cube);
    else if (h->G.num_ra == 3 && h->G.num_va == 1 && B.s == 4)
      k_bin_apply<3, 1, 4><<<n_wg, kApplyThreads, sm_ap, s>>>(h->G, B, start, cursor, h->bin_ent, h->cube);
    else if (h->G.num_ra == 3 && h->G.num_va == 1)
      k_bin_apply<3, 1, -1><<<n_wg, kApplyThreads, sm_ap, s>>>(h->G, B, start, cursor, h->bin_ent, h->cube);
    else
      k_bin_apply<0, 0, -1><<<n_wg, kApplyThreads, sm_ap, s>>>(h->G, B, start, cursor, h->bin_ent, h->cube);
    if ((rc = launch_check(h, "k_bin_apply"))) return rc;
    if (wide && sl && !h->bin_wide) {
      k_bin_log_wg<<<h->sms, 256, 0, s>>>(h->G, log_n, (const uint64_t*)h->bin_log, h->cube);
      if ((rc = launch_check(h, "k_bin_log_wg"))) return rc;
    } else if (wide && sl) {
      k_bin_log_w<<<h->sms, 256, 0, s>>>(h->G, log_n, (const uint64_t*)h->bin_log, h->cube);
      if ((rc = launch_check(h, "k_bin_log_w"))) return rc;
    } else if (h->bin_wc || sl) {   // the scatter's overflow log (usually empty: the kernel exits at once)
      k_bin_log<<<h->sms, 256, 0, s>>>(h->G, B, log_n, log_e, log_b, h->cube);
      if ((rc = launch_check(h, "k_bin_log"))) return rc;
    }
    t_end(h, tk, s);   // the apply phase includes the overflow log
  }
  return CBAA_OK;
}

int update_all_passes(cbaa_handle* h, const uint32_t* src, const uint32_t* dst, uint64_t n, cudaStream_t s) {
  ++h->tcalls;
  if (h->cfg.update_mode == CBAA_UPDATE_BINNED && binned_ok(h) && n >= h->bin_min)
    return update_binned(h, src, dst, n, s);
  const uint64_t W = h->cube_words;
  for (uint32_t p = 0; p < h->passes; ++p) {
    uint64_t lo = W * p / h->passes, hi = W * (p + 1) / h->passes;
    const int tk = t_begin(h, 0, s);
    int rc = launch_update(h, src, dst, n, (uint32_t)lo, (uint32_t)(hi - lo), p == 0, s);
    t_end(h, tk, s);
    if (rc) return rc;
  }
  return CBAA_OK;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

const char* cbaa_strerror(int code) {
  int k = -code;
  if (k < 0 || k >= (int)(sizeof g_codes / sizeof g_codes[0])) return "unknown error";
  return g_codes[k];
}

const char* cbaa_last_error(const cbaa_handle* h) { return h ? h->err.c_str() : ""; }

int cbaa_config_default(cbaa_config* out) {
  if (!out) return CBAA_E_ARG;
  std::memset(out, 0, sizeof *out);
  out->r = 4;
  out->num_ra = 3;
  out->num_va = 1;
  out->g = 4096;
  for (int a = 0; a < 4; ++a) out->cbn[a] = 12;   // c(i) = 2^12 (Q9)
  out->clbs[0] = 0;      // Q8
  out->clbs[1] = 10;
  out->clbs[2] = 20;
  out->mangle_a = 0x9E3779B1u;   // Q3
  out->mangle_b = 0x7F4A7C15u;
  out->bv_seed = 0x85EBCA6Bu;    // Q4
  out->va_seeds[0] = 0xC2B2AE35u;
  out->theta_formula = CBAA_THETA_PAPER;
  out->direction = CBAA_DIR_NORMALIZED;
  out->tuple_cap = 1ull << 24;
  out->update_mode = CBAA_UPDATE_BINNED;   // large windows binned, small ones test-and-set
  return CBAA_OK;
}

int cbaa_config_validate(const cbaa_config* cfg, char* err, uint64_t errlen) {
  std::string why;
  int rc = validate(cfg, &why);
  if (err && errlen) {
    std::snprintf(err, (size_t)errlen, "%s", rc ? why.c_str() : "");
  }
  return rc;
}

uint64_t cbaa_cube_bytes(const cbaa_config* cfg) {
  if (validate(cfg, nullptr)) return 0;
  uint64_t csb = 0;
  for (uint32_t a = 0; a < cfg->num_ra + cfg->num_va; ++a) csb += ((uint64_t)1 << cfg->cbn[a]) * cfg->g;
  return (csb << cfg->r) / 8;
}

static uint64_t sig_offset(uint64_t cube_bytes) { return (cube_bytes + 255) & ~255ull; }

int cbaa_create_ext(const cbaa_config* cfg, int device, void* cube, uint64_t cube_nbytes, cbaa_handle** out) {
  if (!out) return CBAA_E_ARG;
  *out = nullptr;
  std::string why;
  if (validate(cfg, &why)) {
    std::fprintf(stderr, "cbaa_create: %s\n", why.c_str());
    return CBAA_E_CONFIG;
  }
  cbaa_handle* h = new (std::nothrow) cbaa_handle();
  if (!h) return CBAA_E_NOMEM;
  h->cfg = *cfg;
  h->G = derive(*cfg);
  h->device = device;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    delete h;
    return CBAA_E_ARG;
  }
  DeviceGuard dg(device);
  cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&h->l2_bytes, cudaDevAttrL2CacheSize, device);
  h->cube_bytes = cbaa_cube_bytes(cfg);
  h->cube_words = h->cube_bytes / 4;
  int rc = CBAA_OK;
  cudaError_t e = cudaSuccess;
  if (cube) {   // caller-owned cube, e.g. a symmetric-memory buffer peers map over NVLink
    if (cube_nbytes < h->cube_bytes || ((uintptr_t)cube & 255)) {
      delete h;
      return CBAA_E_ARG;
    }
    h->cube = (uint32_t*)cube;
    h->cube_external = true;
    if (cube_nbytes >= sig_offset(h->cube_bytes) + kSigBytes)   // room for the barrier's signal area
      h->sig = (unsigned long long*)((char*)cube + sig_offset(h->cube_bytes));
  } else {
    // the cube and, after it, the signal area of cbaa_peer_barrier: one allocation, one IPC handle
    e = cudaMalloc(&h->cube, sig_offset(h->cube_bytes) + kSigBytes);
    if (e != cudaSuccess) rc = cuda_fail(h, e, "cudaMalloc(cube)");
    else h->sig = (unsigned long long*)((char*)h->cube + sig_offset(h->cube_bytes));
  }
  if (!rc) {
    e = cudaMemset(h->cube, 0, h->cube_bytes);
    if (e != cudaSuccess) rc = cuda_fail(h, e, "cudaMemset(cube)");
  }
  if (!rc && h->sig) {
    e = cudaMemset(h->sig, 0, kSigBytes);
    if (e != cudaSuccess) rc = cuda_fail(h, e, "cudaMemset(signals)");
  }
  if (!rc) rc = alloc_scratch(h);
  if (!rc && cfg->direction == CBAA_DIR_INNER_PREFIX) rc = upload_prefix_bits(h);
  if (rc) {
    std::fprintf(stderr, "cbaa_create: %s\n", h->err.c_str());
    cbaa_destroy(h);
    return rc;
  }
  // Update passes: random access rates collapse 2.4-3x once the working set spills L2
  // (profiles/r01_redbench.jsonl), so the cube is split into address ranges.
  if (cfg->update_passes) {
    h->passes = cfg->update_passes;
  } else {
    // Measured optimum (profiles/r01_passes.jsonl, 100M-500M-pair windows): each pass re-reads and
    // re-hashes the whole input (~4 ps per pair), so the touched part of each pass's range — not the
    // whole range — has to fit L2; in units of L2: ≤ 0.8 → 1, ≤ 3 → 2, ≤ 5 → 3, ≤ 10 → 4, ≤ 20 → 6,
    // else 12.
    const double x = (double)h->cube_bytes / (double)(h->l2_bytes > 0 ? h->l2_bytes : (126 << 20));
    h->passes = x <= 0.8 ? 1 : x <= 3 ? 2 : x <= 5 ? 3 : x <= 10 ? 4 : x <= 20 ? 6 : 12;
  }
  const char* fc = std::getenv("CBAA_FORCE_CARTESIAN");
  h->force_cartesian = fc && fc[0] == '1';
  h->use_join = h->G.num_ra == 3 && !h->force_cartesian;
  const char* nt = std::getenv("CBAA_NO_TMA");
  h->no_tma = nt && nt[0] == '1';
  {   // binned update geometry (binned.cuh): bins (cs, row >> s), word groups of Σc(i) words
    BinGeo& B = h->B;
    B.s = std::min<uint32_t>(5, cfg->r);
    uint32_t lg = 0;
    while ((1u << lg) < cfg->g) ++lg;
    B.bpc_log2 = lg - B.s;
    B.nbins = h->G.n_cs << B.bpc_log2;
    B.nblk = (uint32_t)h->sms * kBinMinBlocks;
    B.ncols = h->G.cs_words / h->G.wpc;
    // scatter tables ≤ 48 KiB (≥ 2 pairs per bin in an 8192-pair tile), word group ≤ 112 KiB
    h->bin_narrow_ok = B.nbins <= 4096 && B.ncols <= 28672;
    // wide entries (LP << 6 | row mod 64) for any geometry with g ≥ 64, 256-2048 bins (cs, row >> 6) and
    // two word groups in 128 KiB (Σc(i) ≤ 16384); the paper geometry keeps its constant-folded kernels
    {
      const uint32_t nbw = lg >= 6 ? h->G.n_cs << (lg - 6) : 0u;
      const char* bw = std::getenv("CBAA_BIN_WIDE");
      const char* bg = std::getenv("CBAA_BIN_WIDE_GEN");
      uint32_t maxc = 0;   // the largest array: its two word groups must fit 128 KiB for the per-array apply
      for (uint32_t a = 0; a < h->G.narr; ++a) maxc = std::max(maxc, h->G.ncols[a]);
      h->bin_gen_ok = lg >= 6 && nbw >= 256 && nbw <= 4096 && maxc <= 16384 && h->G.narr <= CBAA_MAX_ARRAYS &&
                      !(bw && bw[0] == '0') && !(bg && bg[0] == '0');
      h->bin_gen_per_array = B.ncols > 16384;   // k_bin_apply_wa: one CTA per (bin, array)
    }
    h->binnable = h->bin_narrow_ok || h->bin_gen_ok;
    // generic wide entries unless the 32-bit entries already keep 5 row bits (r ≥ 5: one word group per
    // bin, 4-B entries), which measured faster (profiles/r02_wide_generic.jsonl)
    // (CBAA_BIN_WIDE_GEN=2 forces them wherever they fit: tests and A/Bs)
    const char* bgf = std::getenv("CBAA_BIN_WIDE_GEN");
    h->bin_gen_pref = h->bin_gen_ok && (!h->bin_narrow_ok || cfg->r < 5 || (bgf && bgf[0] == '2'));
    // auto (bin_min_pairs = 0): cubes up to 0.6 of L2 stay on the direct kernel when only 32-bit entries
    // with < 4 row bits are available (r < 4: runs of ~1-2 entries per tile; profiles/r02_wide_generic.jsonl:
    // r = 2, g ≤ 2048 is faster direct); with wide entries or r ≥ 4 the binned path wins for every cube size
    if (!cfg->bin_min_pairs && h->cube_bytes <= 0.6 * (double)(h->l2_bytes > 0 ? h->l2_bytes : (126 << 20)) &&
        !(h->bin_gen_pref || (h->bin_narrow_ok && cfg->r >= 4)))
      h->binnable = 0;
    const char* bm = std::getenv("CBAA_BIN_MIN");
    h->bin_min = cfg->bin_min_pairs ? cfg->bin_min_pairs
                 : bm                 ? std::strtoull(bm, nullptr, 10)
                                      : std::max<uint64_t>(1u << 20, h->cube_words / 4);
    if (const char* e = std::getenv("CBAA_SAMPLE_CTAS")) h->sample_ctas = (uint32_t)std::strtoul(e, nullptr, 10);
    if (const char* e = std::getenv("CBAA_SCATTER_PF")) h->scatter_pf = (uint32_t)std::strtoul(e, nullptr, 10);
    const char* bc = std::getenv("CBAA_BIN_CHUNK");
    if (bc && std::strtoull(bc, nullptr, 10) > 0)
      h->bin_chunk = std::min<uint64_t>(1ull << 28, std::strtoull(bc, nullptr, 10));
    if (h->binnable) {
      // every binned kernel may use up to the opt-in maximum of dynamic shared memory: the attribute is
      // per function and process-wide, so a per-handle size would cap another handle's (larger) launches;
      // the launch's own size still sets the occupancy
      int smax = 0;
      cudaDeviceGetAttribute(&smax, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
      set_dyn_smem_max((const void*)k_bin_sample<false>, smax);
      set_dyn_smem_max((const void*)k_bin_sample<true>, smax);
      const char* sp = std::getenv("CBAA_BIN_SAMPLE");
      if (sp) {
        const unsigned long v = std::strtoul(sp, nullptr, 10);
        h->bin_sample_log2 = v == 0 ? 0u : (uint32_t)std::min(16ul, std::max(3ul, v));
      }
      const char* spm = std::getenv("CBAA_BIN_SAMPLE_MIN");
      if (spm) h->bin_sample_min = std::strtoull(spm, nullptr, 10);
      set_dyn_smem_max((const void*)k_bin_count<false>, smax);
      set_dyn_smem_max((const void*)k_bin_count<true>, smax);
      const char* bs = std::getenv("CBAA_BIN_SCATTER");
      h->bin_wc = bs && std::strcmp(bs, "wc") == 0;
      set_dyn_smem_max((const void*)k_bin_wc<false>, smax);
      set_dyn_smem_max((const void*)k_bin_wc<true>, smax);
      set_dyn_smem_max((const void*)k_bin_scatter<false, 0>, smax);
      set_dyn_smem_max((const void*)k_bin_scatter<false, 4096>, smax);
      set_dyn_smem_max((const void*)k_bin_scatter<false, -1>, smax);
      cudaFuncSetAttribute(k_bin_scatter<false, -1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      set_dyn_smem_max((const void*)k_bin_scatter<true, 0>, smax);
      cudaFuncSetAttribute(k_bin_scatter<false, 0>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      cudaFuncSetAttribute(k_bin_scatter<false, 4096>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      cudaFuncSetAttribute(k_bin_scatter<true, 0>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      set_dyn_smem_max((const void*)k_bin_apply<3, 1, 4>, smax);
      set_dyn_smem_max((const void*)k_bin_apply<3, 1, 4, true>, smax);
      {   // the paper's default configuration: k_bin_apply<3, 1, 4, true> with constants inlined
        const Geo& g = h->G;
        bool pp = g.num_ra == 3 && g.num_va == 1 && B.s == 4 && g.sh[0] == 44 && g.sh[1] == 34 && g.sh[2] == 24;
        for (uint32_t a = 0; a < 4 && pp; ++a) pp = g.colmask[a] == 4095u && (g.arr_off[a] >> g.wpc_log2) == 4096u * a;
        h->apply_paper = pp;
        // wide entries for the paper configuration (r = 4, g = 4096): CBAA_BIN_WIDE=0 keeps 32-bit entries
        const char* bw = std::getenv("CBAA_BIN_WIDE");
        h->bin_wide = pp && g.r == 4 && g.g == 4096 && !(bw && bw[0] == '0');
        h->bin_wide_gen = !h->bin_wide && h->bin_gen_pref;
        BinGeo& W = h->BW;
        W.s = 6;
        W.bpc_log2 = lg >= 6 ? lg - 6 : 0;
        W.nbins = h->G.n_cs << W.bpc_log2;
        W.nblk = B.nblk;
        W.ncols = B.ncols;
        set_wscatter_attrs<-1>(smax);
        set_wscatter_attrs<256>(smax);
        set_wscatter_attrs<512>(smax);
        set_wscatter_attrs<1024>(smax);
        set_wscatter_attrs<2048>(smax);
        set_wscatter_attrs<4096>(smax);
        set_dyn_smem_max((const void*)k_bin_apply_w, smax);
        set_dyn_smem_max((const void*)k_bin_apply_wg<3, 1>, smax);
        set_dyn_smem_max((const void*)k_bin_apply_wg<0, 0>, smax);
        set_dyn_smem_max((const void*)k_bin_apply_wa, smax);
      }
      set_dyn_smem_max((const void*)k_bin_apply<3, 1, -1>, smax);
      set_dyn_smem_max((const void*)k_bin_apply<0, 0, -1>, smax);
      (void)cudaGetLastError();   // an attribute the device refused must not surface at a later launch check
    }
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_update<3, 1, CBAA_UPDATE_TEST_SET, false>, kThreads, 0);
  h->upd_blocks = std::max(1, occ);
  *out = h;
  return CBAA_OK;
}

int cbaa_create(const cbaa_config* cfg, int device, cbaa_handle** out) {
  return cbaa_create_ext(cfg, device, nullptr, 0, out);
}

void cbaa_destroy(cbaa_handle* h) {
  if (!h) return;
  DeviceGuard dg(h->device);
  if (h->cube && !h->cube_external) cudaFree(h->cube);
  if (h->scratch) cudaFree(h->scratch);
  if (h->bin_ent) cudaFree(h->bin_ent);
  if (h->bin_tab) cudaFree(h->bin_tab);
  if (h->bin_log) cudaFree(h->bin_log);
  for (cudaEvent_t e : h->tev) cudaEventDestroy(e);
  if (h->prefix_bits) cudaFree(h->prefix_bits);
  if (h->D.cand) cudaFree(h->D.cand);
  if (h->h_rec) cudaFreeHost(h->h_rec);
  if (h->h_cnt) cudaFreeHost(h->h_cnt);
  if (h->h_res) cudaFreeHost(h->h_res);
  for (int b = 0; b < 2; ++b) {
    for (int a = 0; a < 2; ++a)
      if (h->stage[b][a]) cudaFree(h->stage[b][a]);
    if (h->ev_copied[b]) cudaEventDestroy(h->ev_copied[b]);
    if (h->ev_free[b]) cudaEventDestroy(h->ev_free[b]);
  }
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  for (DetectGraph& d : h->dgs) {
    if (d.exec) cudaGraphExecDestroy(d.exec);
    if (d.graph) cudaGraphDestroy(d.graph);
  }
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  delete h;
}

int cbaa_get_config(const cbaa_handle* h, cbaa_config* out) {
  if (!h || !out) return CBAA_E_ARG;
  *out = h->cfg;
  return CBAA_OK;
}

int cbaa_reset(cbaa_handle* h, cbaa_stream stream) {
  if (!h) return CBAA_E_ARG;
  h->zc_fresh = 0;   // the cube changes: zero counts of an earlier pull-OR are stale
  DeviceGuard dg(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t n16 = h->cube_bytes / 16;
  k_zero<<<grid_for(h, n16, 4), kThreads, 0, s>>>((uint4*)h->cube, n16);
  int rc = launch_check(h, "k_zero");
  if (rc) return rc;
  CK(h, cudaMemsetAsync(h->skipped, 0, 8, s));
  return CBAA_OK;
}

int cbaa_update(cbaa_handle* h, const uint32_t* src, const uint32_t* dst, uint64_t n, cbaa_stream stream) {
  if (!h) return CBAA_E_ARG;
  h->zc_fresh = 0;   // the cube changes: zero counts of an earlier pull-OR are stale
  if (n == 0) return CBAA_OK;
  if (!src || !dst) return fail(h, CBAA_E_ARG, "cbaa_update: null src/dst");
  if (((uintptr_t)src | (uintptr_t)dst) & 3) return fail(h, CBAA_E_ARG, "cbaa_update: src/dst must be 4-byte aligned");
  DeviceGuard dg(h->device);
  return update_all_passes(h, src, dst, n, (cudaStream_t)stream);
}

int cbaa_update_pairs(cbaa_handle* h, const uint32_t* pairs, uint64_t n, cbaa_stream stream) {
  if (!h) return CBAA_E_ARG;
  h->zc_fresh = 0;   // the cube changes: zero counts of an earlier pull-OR are stale
  if (n == 0) return CBAA_OK;
  if (!pairs) return fail(h, CBAA_E_ARG, "cbaa_update_pairs: null pairs");
  if ((uintptr_t)pairs & 7) return fail(h, CBAA_E_ARG, "cbaa_update_pairs: pairs must be 8-byte aligned");
  DeviceGuard dg(h->device);
  const uint64_t W = h->cube_words;
  for (uint32_t p = 0; p < h->passes; ++p) {
    uint64_t lo = W * p / h->passes, hi = W * (p + 1) / h->passes;
    int rc = launch_update_aos(h, pairs, n, (uint32_t)lo, (uint32_t)(hi - lo), p == 0, (cudaStream_t)stream);
    if (rc) return rc;
  }
  return CBAA_OK;
}

int cbaa_update_host(cbaa_handle* h, const uint32_t* src, const uint32_t* dst, uint64_t n, cbaa_stream stream) {
  if (!h) return CBAA_E_ARG;
  h->zc_fresh = 0;   // the cube changes: zero counts of an earlier pull-OR are stale
  if (n == 0) return CBAA_OK;
  if (!src || !dst) return fail(h, CBAA_E_ARG, "cbaa_update_host: null src/dst");
  DeviceGuard dg(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t chunk = 1ull << 23;   // 8 Mi pairs = 64 MiB per buffer pair
  if (!h->copy_stream) {
    CK(h, cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      CK(h, cudaEventCreateWithFlags(&h->ev_copied[b], cudaEventDisableTiming));
      CK(h, cudaEventCreateWithFlags(&h->ev_free[b], cudaEventDisableTiming));
      CK(h, cudaEventRecord(h->ev_free[b], h->copy_stream));   // both staging buffers start free
      for (int a = 0; a < 2; ++a) CK(h, cudaMalloc(&h->stage[b][a], chunk * 4));
    }
    h->stage_pairs = chunk;
  }
  // ev_free[b] always marks the end of the last update that read staging buffer b — on whatever
  // stream that call used — so a copy into b waits for it even across calls on different streams
  uint64_t k = 0;
  for (uint64_t off = 0; off < n; off += h->stage_pairs, ++k) {
    const int b = (int)(k & 1);
    const uint64_t m = std::min(h->stage_pairs, n - off);
    CK(h, cudaStreamWaitEvent(h->copy_stream, h->ev_free[b], 0));
    CK(h, cudaMemcpyAsync(h->stage[b][0], src + off, m * 4, cudaMemcpyHostToDevice, h->copy_stream));
    CK(h, cudaMemcpyAsync(h->stage[b][1], dst + off, m * 4, cudaMemcpyHostToDevice, h->copy_stream));
    CK(h, cudaEventRecord(h->ev_copied[b], h->copy_stream));
    CK(h, cudaStreamWaitEvent(s, h->ev_copied[b], 0));
    int rc = update_all_passes(h, h->stage[b][0], h->stage[b][1], m, s);
    if (rc) return rc;
    CK(h, cudaEventRecord(h->ev_free[b], s));
  }
  return CBAA_OK;
}

int cbaa_skipped(cbaa_handle* h, uint64_t* out, cbaa_stream stream) {
  if (!h || !out) return CBAA_E_ARG;
  DeviceGuard dg(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  CK(h, cudaMemcpyAsync(h->h_cnt, h->skipped, 8, cudaMemcpyDeviceToHost, s));
  CK(h, cudaStreamSynchronize(s));
  *out = h->h_cnt[0];
  return CBAA_OK;
}

int cbaa_merge(cbaa_handle* h, const void* const* cubes, int k, uint64_t nbytes, cbaa_stream stream) {
  if (!h) return CBAA_E_ARG;
  h->zc_fresh = 0;   // the cube changes: zero counts of an earlier pull-OR are stale
  if (k < 0 || k > CBAA_MAX_MERGE || (k && !cubes)) return fail(h, CBAA_E_ARG, "cbaa_merge: bad k/cubes");
  if (nbytes != h->cube_bytes)
    return fail(h, CBAA_E_MISMATCH, "cbaa_merge: cube size differs from this handle's geometry (S:103)");
  DeviceGuard dg(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t n16 = h->cube_bytes / 16;
  for (int j0 = 0; j0 < k; j0 += 16) {
    MergeSrcs S{};
    S.k = std::min(16, k - j0);
    for (int j = 0; j < S.k; ++j) {
      if (!cubes[j0 + j] || ((uintptr_t)cubes[j0 + j] & 15))
        return fail(h, CBAA_E_ARG, "cbaa_merge: null or non-16-byte-aligned cube pointer");
      S.p[j] = (const uint4*)cubes[j0 + j];
    }
    k_or_merge<<<grid_for(h, n16, 4), kThreads, 0, s>>>((uint4*)h->cube, S, n16);
    int rc = launch_check(h, "k_or_merge");
    if (rc) return rc;
  }
  return CBAA_OK;
}

int cbaa_merge_slice(cbaa_handle* h, const void* const* slices, int k, uint32_t cs_lo, uint32_t cs_hi,
                     cbaa_stream stream) {
  if (!h) return CBAA_E_ARG;
  h->zc_fresh = 0;   // the cube changes: zero counts of an earlier pull-OR are stale
  if (cs_lo >= cs_hi || cs_hi > h->G.n_cs) return fail(h, CBAA_E_ARG, "cbaa_merge_slice: bad CS range");
  if (k < 0 || k > CBAA_MAX_MERGE || (k && !slices)) return fail(h, CBAA_E_ARG, "cbaa_merge_slice: bad k/slices");
  DeviceGuard dg(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t cs_bytes = (uint64_t)h->G.cs_words * 4;
  uint64_t n16 = cs_bytes * (cs_hi - cs_lo) / 16;
  uint4* dst = (uint4*)((char*)h->cube + cs_bytes * cs_lo);
  for (int j0 = 0; j0 < k; j0 += 16) {
    MergeSrcs S{};
    S.k = std::min(16, k - j0);
    for (int j = 0; j < S.k; ++j) {
      if (!slices[j0 + j] || ((uintptr_t)slices[j0 + j] & 15))
        return fail(h, CBAA_E_ARG, "cbaa_merge_slice: null or non-16-byte-aligned slice pointer");
      S.p[j] = (const uint4*)slices[j0 + j];
    }
    k_or_merge<<<grid_for(h, n16, 4), kThreads, 0, s>>>(dst, S, n16);
    int rc = launch_check(h, "k_or_merge");
    if (rc) return rc;
  }
  return CBAA_OK;
}

static int launch_zero_hot(cbaa_handle* h, uint32_t cs_lo, uint32_t n_range, uint32_t theta, int finish,
                           cudaStream_t s, int join = 0, int zc_given = 0) {
  const Geo& G = h->G;
  uint64_t groups = 0;
  for (uint32_t i = 0; i < G.num_ra; ++i) groups += (G.ncols[i] + 15) / 16;
  groups *= n_range;
  const int grid =
      (int)std::min<uint64_t>((uint64_t)h->sms * 16, std::max<uint64_t>(1, (groups + kDetWarps - 1) / kDetWarps));
  // g = 4096 with RA blocks of whole 16-column tiles (every c(i) ≥ 16): TMA-streamed zero counts
  bool tma = G.wpc == 128 && !h->no_tma && !h->cfg.detect_overlap;
  for (uint32_t i = 0; i < G.num_ra; ++i) tma = tma && G.ncols[i] % kZcTileCols == 0;
  if (zc_given)
    ;   // counts (and the per-detect counter reset) came from k_or_merge_zc
  else if (tma)
    k_zero_counts_tma<<<h->sms * 4, kDetThreads, 0, s>>>(G, h->cube, h->D, cs_lo, n_range, finish);
  else if (G.wpc == 128)   // g = 4096: one 16-byte load per lane covers a column
    k_zero_counts<true><<<grid, kDetThreads, 0, s>>>(G, h->cube, h->D, cs_lo, n_range, finish);
  else
    k_zero_counts<false><<<grid, kDetThreads, 0, s>>>(G, h->cube, h->D, cs_lo, n_range, finish);
  int rc = zc_given ? CBAA_OK : launch_check(h, "k_zero_counts");
  if (rc || !finish) return rc;
  const uint64_t hot_grid = (uint64_t)n_range * G.num_ra;
  if (hot_grid > 0x7fffffffull) return fail(h, CBAA_E_ARG, "detect grid too large");
  k_hot<<<(unsigned)hot_grid, kDetThreads, 0, s>>>(G, h->D, cs_lo, n_range, theta, join);
  return launch_check(h, "k_hot");
}

int cbaa_zero_counts(cbaa_handle* h, uint32_t* out, cbaa_stream stream) {
  if (!h || !out) return CBAA_E_ARG;
  DeviceGuard dg(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  int rc = launch_zero_hot(h, 0, h->G.n_cs, 0, 0, s);
  if (rc) return rc;
  CK(h, cudaMemcpyAsync(out, h->D.zc, (size_t)h->G.n_cs * h->G.ra_cols * 4, cudaMemcpyDeviceToDevice, s));
  return CBAA_OK;
}

int cbaa_detect_range(cbaa_handle* h, uint32_t theta, uint32_t cs_lo, uint32_t cs_hi, cbaa_host* out, uint64_t cap,
                      uint64_t* n_out, cbaa_cs_stats* stats, cbaa_stream stream) {
  if (!h || !n_out) return CBAA_E_ARG;
  if (cs_lo >= cs_hi || cs_hi > h->G.n_cs) return fail(h, CBAA_E_ARG, "cbaa_detect: bad CS range");
  if (cap && !out) return fail(h, CBAA_E_ARG, "cbaa_detect: out is null");
  DeviceGuard dg(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const uint32_t n_range = cs_hi - cs_lo;
  DetectScratch& D = h->D;
  // The whole device side of a detect — zeroing, zero counts, k_hot, the Alg. 3 kernels and the copy
  // of the CS records and [n_hits | first kFirst hits] to pinned memory — is one CUDA graph, captured
  // once per (range, buffers) and relaunched every window (θ rewritten in place): one launch and one
  // host sync per detect.
  const uint64_t kFirst = std::min<uint64_t>(1024, D.hit_cap);
  // zero counts already computed by cbaa_merge_slice_zc for exactly this range: the graph without them
  const int zg = (h->zc_fresh && h->zc_lo == cs_lo && h->zc_hi == cs_hi) ? 1 : 0;
  h->zc_fresh = 0;   // consumed: that kernel also zeroed the per-detect counters, once
  DetectGraph& dgr = h->dgs[zg];
  const DetectKey key{cs_lo, cs_hi, h->record, (const void*)D.cand, (const void*)h->h_res, h->use_join};
  if (!dgr.exec || !(dgr.key == key)) {
    if (dgr.exec) {
      cudaGraphExecDestroy(dgr.exec);
      dgr.exec = nullptr;
    }
    if (dgr.graph) {
      cudaGraphDestroy(dgr.graph);
      dgr.graph = nullptr;
    }
    dgr.hot_node = nullptr;
    if (!h->cap_stream) CK(h, cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
    cudaStream_t c = h->cap_stream;
    CK(h, cudaStreamBeginCapture(c, cudaStreamCaptureModeThreadLocal));
    // (the per-detect counters are zeroed inside the zero-count kernel and k_hot: no memset nodes)
    // |RA| = 3: range join over the sorted hot lists, then one warp per chain; otherwise (or after a
    // join-buffer overflow) the Cartesian enumeration with the union check inline
    const int join = h->use_join;
    int rc = launch_zero_hot(h, cs_lo, n_range, theta, 1, c, join, zg);
    const int grid = h->sms * 8;
    if (!rc) {
      if (join) {
        k_join3<<<grid, kDetThreads, 0, c>>>(h->G, D, cs_lo, n_range);
        rc = launch_check(h, "k_join3");
        if (!rc) {
          k_union<<<grid, kDetThreads, 0, c>>>(h->G, h->cube, D, h->record);
          rc = launch_check(h, "k_union");
        }
      } else {
        if (h->G.num_ra == 3) k_tuples<3><<<grid, kDetThreads, 0, c>>>(h->G, h->cube, D, cs_lo, n_range, h->record);
        else k_tuples<0><<<grid, kDetThreads, 0, c>>>(h->G, h->cube, D, cs_lo, n_range, h->record);
        rc = launch_check(h, "k_tuples");
      }
    }
    // S:418 order on the device (a standalone detect; with detect_overlap the host sorts, because the
    // sort's shared memory would keep it from running beside another handle's update)
    if (!rc && !h->cfg.detect_overlap) {
      k_sort_hits<<<1, 1024, 0, c>>>(D);
      rc = launch_check(h, "k_sort_hits");
    }
    cudaMemcpyAsync(h->h_rec, D.rec + cs_lo, (size_t)n_range * sizeof(cbaa_cs_stats), cudaMemcpyDeviceToHost, c);
    cudaMemcpyAsync(h->h_res, D.n_hits, 64 + kFirst * sizeof(cbaa_host), cudaMemcpyDeviceToHost, c);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(c, &graph);
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (e != cudaSuccess) return cuda_fail(h, e, "cudaStreamEndCapture(detect)");
    e = cudaGraphInstantiate(&dgr.exec, graph, 0);
    if (e != cudaSuccess) {
      cudaGraphDestroy(graph);
      return cuda_fail(h, e, "cudaGraphInstantiate(detect)");
    }
    dgr.graph = graph;
    // find the k_hot node: a later θ only rewrites that node's parameters in the executable graph
    size_t nn = 0;
    CK(h, cudaGraphGetNodes(graph, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    CK(h, cudaGraphGetNodes(graph, nodes.data(), &nn));
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType t;
      CK(h, cudaGraphNodeGetType(nd, &t));
      if (t != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeParams kp{};
      CK(h, cudaGraphKernelNodeGetParams(nd, &kp));
      if (kp.func == (void*)k_hot) {
        dgr.hot_node = nd;
        dgr.hot_params = kp;
      }
    }
    if (!dgr.hot_node) return fail(h, CBAA_E_CUDA, "detect graph: k_hot node not found");
    dgr.theta = theta;
    dgr.key = key;
    dgr.kernels = (join ? 4 : 3) - zg + (h->cfg.detect_overlap ? 0 : 1);
    h->launches -= dgr.kernels;   // counted at capture; counted again per graph launch below
  }
  if (dgr.theta != theta) {   // same graph, new θ: k_hot(G, D, cs_lo, n_range, theta, join)
    void* args[6];
    for (int i = 0; i < 6; ++i) args[i] = dgr.hot_params.kernelParams[i];
    uint32_t th = theta;
    args[4] = &th;
    cudaKernelNodeParams kp = dgr.hot_params;
    kp.kernelParams = args;
    kp.extra = nullptr;
    CK(h, cudaGraphExecKernelNodeSetParams(dgr.exec, dgr.hot_node, &kp));
    dgr.theta = theta;
  }
  CK(h, cudaGraphLaunch(dgr.exec, s));
  h->launches += dgr.kernels;
  CK(h, cudaStreamSynchronize(s));
  if (h->use_join && ((const unsigned long long*)h->h_res)[1] > D.join_cap) {
    // more CP chains than the join buffer holds: redo this window with the Cartesian enumeration
    // (bounded by tuple_cap per CS, no buffer); the stats and hits are recomputed from scratch
    h->use_join = 0;
    int rc2 = cbaa_detect_range(h, theta, cs_lo, cs_hi, out, cap, n_out, stats, stream);
    h->use_join = 1;
    return rc2;
  }
  const uint64_t total = *(const unsigned long long*)h->h_res;
  const uint64_t got = std::min<uint64_t>(total, D.hit_cap);
  if (got > kFirst) {
    if (got > h->h_hits_cap) {
      void* bigger = nullptr;
      uint64_t cap2 = std::max<uint64_t>(got, 2 * h->h_hits_cap);
      CK(h, cudaMallocHost(&bigger, 64 + cap2 * sizeof(cbaa_host)));
      std::memcpy(bigger, h->h_res, 64 + kFirst * sizeof(cbaa_host));
      cudaFreeHost(h->h_res);
      h->h_res = bigger;
      h->h_hits = (cbaa_host*)((char*)bigger + 64);
      h->h_hits_cap = cap2;
    }
    CK(h, cudaMemcpyAsync(h->h_hits + kFirst, D.hits + kFirst, (got - kFirst) * sizeof(cbaa_host),
                          cudaMemcpyDeviceToHost, s));
    CK(h, cudaStreamSynchronize(s));
  }
  // output order of S:418: estimate descending, then ip ascending (already done on the device for a
  // standalone detect of at most kSortMax hits)
  if (h->cfg.detect_overlap || got > (uint64_t)kSortMax) cbaa_sort_hosts(h->h_hits, got);
  const uint64_t ncopy = std::min<uint64_t>(got, cap);
  if (ncopy) std::memcpy(out, h->h_hits, ncopy * sizeof(cbaa_host));
  *n_out = total;
  if (stats) std::memcpy(stats, h->h_rec, (size_t)n_range * sizeof(cbaa_cs_stats));
  bool overflow = false;
  for (uint32_t k = 0; k < n_range; ++k) overflow |= h->h_rec[k].overflow != 0;
  if (total > D.hit_cap)
    return fail(h, CBAA_E_CAPACITY, "device hit buffer too small: raise cbaa_config.hit_capacity");
  if (total > cap) return fail(h, CBAA_E_CAPACITY, "more hosts than cap: *n_out holds the required count");
  if (overflow) return fail(h, CBAA_E_TUPLE_CAP, "a CS exceeded tuple_cap and was skipped (see stats.overflow)");
  return CBAA_OK;
}

int cbaa_detect(cbaa_handle* h, uint32_t theta, cbaa_host* out, uint64_t cap, uint64_t* n_out, cbaa_cs_stats* stats,
                cbaa_stream stream) {
  if (!h) return CBAA_E_ARG;
  return cbaa_detect_range(h, theta, 0, h->G.n_cs, out, cap, n_out, stats, stream);
}

int cbaa_cube_view(cbaa_handle* h, void** dev_ptr, uint64_t* nbytes) {
  if (!h || !dev_ptr || !nbytes) return CBAA_E_ARG;
  *dev_ptr = h->cube;
  *nbytes = h->cube_bytes;
  return CBAA_OK;
}

int cbaa_hot_columns(cbaa_handle* h, uint32_t* out, cbaa_stream stream) {
  if (!h || !out) return CBAA_E_ARG;
  DeviceGuard dg(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  CK(h, cudaMemcpyAsync(out, h->D.hc, (size_t)h->G.n_cs * h->G.ra_cols * 4, cudaMemcpyDeviceToHost, s));
  CK(h, cudaStreamSynchronize(s));
  return CBAA_OK;
}

int cbaa_set_record_candidates(cbaa_handle* h, int enable, uint64_t capacity) {
  if (!h) return CBAA_E_ARG;
  DeviceGuard dg(h->device);
  if (h->D.cand) {
    cudaFree(h->D.cand);
    h->D.cand = nullptr;
    h->D.cand_cap = 0;
  }
  h->record = enable ? 1 : 0;
  if (enable) {
    CK(h, cudaMalloc(&h->D.cand, std::max<uint64_t>(capacity, 1) * 8));
    h->D.cand_cap = std::max<uint64_t>(capacity, 1);
  }
  return CBAA_OK;
}

int cbaa_candidates(cbaa_handle* h, uint64_t* out, uint64_t cap, uint64_t* n_out, cbaa_stream stream) {
  if (!h || !n_out) return CBAA_E_ARG;
  if (!h->record) return fail(h, CBAA_E_ARG, "candidate recording is off");
  DeviceGuard dg(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  CK(h, cudaMemcpyAsync(h->h_cnt, h->D.n_cand, 8, cudaMemcpyDeviceToHost, s));
  CK(h, cudaStreamSynchronize(s));
  uint64_t total = h->h_cnt[0];
  uint64_t m = std::min(std::min(total, cap), h->D.cand_cap);
  if (m) CK(h, cudaMemcpy(out, h->D.cand, m * 8, cudaMemcpyDeviceToHost));
  *n_out = total;
  return total > h->D.cand_cap ? fail(h, CBAA_E_CAPACITY, "candidate buffer too small") : CBAA_OK;
}

int cbaa_debug_map(cbaa_handle* h, const uint32_t* iip, const uint32_t* oip, uint64_t n, uint32_t* cs, uint32_t* cols,
                   uint32_t* row, cbaa_stream stream) {
  if (!h) return CBAA_E_ARG;
  if (n == 0) return CBAA_OK;
  if (!iip || !oip || !cs || !cols || !row) return fail(h, CBAA_E_ARG, "cbaa_debug_map: null pointer");
  DeviceGuard dg(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  k_debug_map<<<grid_for(h, n, 8), kThreads, 0, s>>>(h->G, iip, oip, n, cs, cols, row);
  return launch_check(h, "k_debug_map");
}

// ------------------------------------------------------------------ SketchFile "CBA1"
static uint64_t sketch_header_bytes(const cbaa_config& c) {
  return 4 + 2 + 3 + 4 + (c.num_ra + c.num_va) + c.num_ra + 12 + 4ull * c.num_va + 8;
}

uint64_t cbaa_sketch_bytes(const cbaa_handle* h) {
  return h ? sketch_header_bytes(h->cfg) + h->cube_bytes : 0;
}

namespace {
struct Writer {
  uint8_t* p;
  void u8(uint32_t v) { *p++ = (uint8_t)v; }
  void u16(uint32_t v) { u8(v & 0xff); u8(v >> 8); }
  void u32(uint32_t v) { for (int k = 0; k < 4; ++k) u8((v >> (8 * k)) & 0xff); }
  void u64(uint64_t v) { for (int k = 0; k < 8; ++k) u8((uint32_t)((v >> (8 * k)) & 0xff)); }
};
struct Reader {
  const uint8_t* p;
  const uint8_t* end;
  bool ok = true;
  uint32_t u8() {
    if (p >= end) { ok = false; return 0; }
    return *p++;
  }
  uint32_t u16() { uint32_t a = u8(); return a | (u8() << 8); }
  uint32_t u32() { uint32_t v = 0; for (int k = 0; k < 4; ++k) v |= u8() << (8 * k); return v; }
  uint64_t u64() { uint64_t v = 0; for (int k = 0; k < 8; ++k) v |= (uint64_t)u8() << (8 * k); return v; }
};

// Parses the header; on success *payload points at the cube bytes and *plen is their length.
int parse_sketch(const void* in, uint64_t n, cbaa_config* out, const uint8_t** payload, uint64_t* plen,
                 std::string* why, bool* sparse = nullptr) {
  auto bad = [&](const std::string& m) {
    if (why) *why = m;
    return CBAA_E_CONFIG;
  };
  if (!in || !out) return bad("null buffer");
  Reader R{(const uint8_t*)in, (const uint8_t*)in + n};
  char magic[4];
  for (int k = 0; k < 4; ++k) magic[k] = (char)R.u8();
  const bool sp = R.ok && std::memcmp(magic, "CBA2", 4) == 0;   // the sparse form
  if (!R.ok || (!sp && std::memcmp(magic, "CBA1", 4) != 0)) return bad("magic: expected \"CBA1\" or \"CBA2\"");
  if (sparse) *sparse = sp;
  uint32_t version = R.u16();
  if (!R.ok || version != 1) return bad("version: expected 1");
  cbaa_config c;
  cbaa_config_default(&c);
  c.r = R.u8();
  c.num_ra = R.u8();
  c.num_va = R.u8();
  c.g = R.u32();
  if (!R.ok) return bad("header truncated");
  if (c.num_ra > CBAA_MAX_RA || c.num_va > CBAA_MAX_VA) return bad("num_ra/num_va out of range");
  std::memset(c.cbn, 0, sizeof c.cbn);
  std::memset(c.clbs, 0, sizeof c.clbs);
  std::memset(c.va_seeds, 0, sizeof c.va_seeds);
  for (uint32_t a = 0; a < c.num_ra + c.num_va; ++a) c.cbn[a] = (uint8_t)R.u8();
  for (uint32_t i = 0; i < c.num_ra; ++i) c.clbs[i] = (uint8_t)R.u8();
  c.mangle_a = R.u32();
  c.mangle_b = R.u32();
  c.bv_seed = R.u32();
  for (uint32_t j = 0; j < c.num_va; ++j) c.va_seeds[j] = R.u32();
  uint64_t len = R.u64();
  if (!R.ok) return bad("header truncated");
  std::string inv;
  if (validate(&c, &inv)) return bad("config invariant: " + inv);
  uint64_t want = cbaa_cube_bytes(&c);
  if (len != want)
    return bad("payload length field " + std::to_string(len) + " != cube size " + std::to_string(want));
  uint64_t have = (uint64_t)(R.end - R.p);
  if (sp) {   // u32 block bits, u64 blocks, (blocks + 1) × u64 offsets, streams
    const uint64_t nb = (len * 8 + 32767) / 32768;
    if (have < 12 || R.u32() != 32768u) return bad("sparse block bits: expected 32768");
    if (R.u64() != nb) return bad("sparse block count: expected " + std::to_string(nb));
    const uint64_t need = 8 * (nb + 1);
    if ((uint64_t)(R.end - R.p) < need) return bad("sparse offsets truncated");
    const uint8_t* offs = R.p;
    uint64_t prev = 0, last = 0;
    for (uint64_t b = 0; b <= nb; ++b) {   // offsets must start at 0 and never decrease
      uint64_t v = 0;
      for (int k = 0; k < 8; ++k) v |= (uint64_t)offs[8 * b + k] << (8 * k);
      if ((b == 0 && v != 0) || v < prev) return bad("sparse offsets not ascending from 0");
      prev = last = v;
    }
    if ((uint64_t)(R.end - R.p) - need < last)
      return bad("payload truncated: expected " + std::to_string(last) + " stream bytes");
    *out = c;
    if (payload) *payload = R.p;   // offsets, then the streams
    if (plen) *plen = need + last;
    return CBAA_OK;
  }
  if (have < len)
    return bad("payload truncated: expected " + std::to_string(len) + " bytes, got " + std::to_string(have));
  *out = c;
  if (payload) *payload = R.p;
  if (plen) *plen = len;
  return CBAA_OK;
}
}  // namespace

static void write_sketch_header(const cbaa_config& c, uint64_t cube_bytes, uint8_t* out, char kind) {
  Writer W{out};
  W.u8('C'); W.u8('B'); W.u8('A'); W.u8((uint8_t)kind);
  W.u16(1);
  W.u8(c.r); W.u8(c.num_ra); W.u8(c.num_va);
  W.u32(c.g);
  for (uint32_t a = 0; a < c.num_ra + c.num_va; ++a) W.u8(c.cbn[a]);
  for (uint32_t i = 0; i < c.num_ra; ++i) W.u8(c.clbs[i]);
  W.u32(c.mangle_a); W.u32(c.mangle_b); W.u32(c.bv_seed);
  for (uint32_t j = 0; j < c.num_va; ++j) W.u32(c.va_seeds[j]);
  W.u64(cube_bytes);
}

int cbaa_serialize_sparse(cbaa_handle* h, void* out, uint64_t cap, uint64_t* n_written, cbaa_stream stream) {
  if (!h || !n_written) return CBAA_E_ARG;
  DeviceGuard dg(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t nwords = h->cube_words, nb = (nwords + kSparseBlockWords - 1) / kSparseBlockWords;
  const uint64_t hb = sketch_header_bytes(h->cfg) + 12 + 8 * (nb + 1);
  void* scratch = nullptr;   // u32 bytes[nb] | u64 off[nb + 1]
  CK(h, cudaMalloc(&scratch, nb * 4 + 8 * (nb + 1) + 16));
  uint32_t* bytes = (uint32_t*)scratch;
  unsigned long long* off = (unsigned long long*)((char*)scratch + ((nb * 4 + 15) & ~15ull));
  const int grid = (int)std::min<uint64_t>((uint64_t)h->sms * 16, (nb + 3) / 4);
  k_sparse_size<<<grid, 128, 0, s>>>(h->cube, nwords, nb, bytes);
  int rc = launch_check(h, "k_sparse_size");
  if (!rc) {
    k_sparse_offsets<<<1, 1024, 0, s>>>(bytes, nb, off);
    rc = launch_check(h, "k_sparse_offsets");
  }
  unsigned long long total = 0;
  cudaError_t e = cudaSuccess;
  if (!rc) {
    e = cudaMemcpyAsync(&total, off + nb, 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = cuda_fail(h, e, "sparse size");
  }
  *n_written = hb + total;
  if (!rc && (cap < hb + total || !out))
    rc = fail(h, CBAA_E_CAPACITY, "cbaa_serialize_sparse: buffer smaller than *n_written");
  void* dpay = nullptr;
  if (!rc && total) {
    e = cudaMalloc(&dpay, total);
    if (e != cudaSuccess) rc = cuda_fail(h, e, "cudaMalloc(sparse payload)");
    if (!rc) {
      k_sparse_write<<<grid, 128, 0, s>>>(h->cube, nwords, nb, off, (uint8_t*)dpay);
      rc = launch_check(h, "k_sparse_write");
    }
  }
  if (!rc) {
    uint8_t* o = (uint8_t*)out;
    write_sketch_header(h->cfg, h->cube_bytes, o, '2');
    Writer W{o + sketch_header_bytes(h->cfg)};
    W.u32(32768);
    W.u64(nb);
    e = cudaMemcpyAsync(W.p, off, 8 * (nb + 1), cudaMemcpyDeviceToHost, s);   // little-endian host
    if (e == cudaSuccess && total) e = cudaMemcpyAsync(o + hb, dpay, total, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = cuda_fail(h, e, "sparse copy-out");
  }
  if (dpay) cudaFree(dpay);
  cudaFree(scratch);
  return rc;
}

int cbaa_serialize(cbaa_handle* h, void* out, uint64_t cap, uint64_t* n_written, cbaa_stream stream) {
  if (!h || !n_written) return CBAA_E_ARG;
  const cbaa_config& c = h->cfg;
  const uint64_t hb = sketch_header_bytes(c), total = hb + h->cube_bytes;
  *n_written = total;
  if (cap < total || !out) return fail(h, CBAA_E_CAPACITY, "cbaa_serialize: buffer smaller than cbaa_sketch_bytes");
  DeviceGuard dg(h->device);
  write_sketch_header(c, h->cube_bytes, (uint8_t*)out, '1');
  cudaStream_t s = (cudaStream_t)stream;
  CK(h, cudaMemcpyAsync((uint8_t*)out + hb, h->cube, h->cube_bytes, cudaMemcpyDeviceToHost, s));
  CK(h, cudaStreamSynchronize(s));
  return CBAA_OK;
}

int cbaa_sketch_config(const void* in, uint64_t n, cbaa_config* out, char* err, uint64_t errlen) {
  std::string why;
  int rc = parse_sketch(in, n, out, nullptr, nullptr, &why);
  if (err && errlen) std::snprintf(err, (size_t)errlen, "%s", rc ? why.c_str() : "");
  return rc;
}

int cbaa_deserialize(cbaa_handle* h, const void* in, uint64_t n, int mode, cbaa_stream stream) {
  if (!h) return CBAA_E_ARG;
  h->zc_fresh = 0;   // the cube changes: zero counts of an earlier pull-OR are stale
  if (mode != CBAA_SKETCH_REPLACE && mode != CBAA_SKETCH_MERGE) return fail(h, CBAA_E_ARG, "bad mode");
  cbaa_config fc;
  const uint8_t* payload = nullptr;
  uint64_t plen = 0;
  std::string why;
  bool sparse = false;
  if (parse_sketch(in, n, &fc, &payload, &plen, &why, &sparse)) return fail(h, CBAA_E_CONFIG, "SketchFile: " + why);
  const cbaa_config& c = h->cfg;
  auto mismatch = [&](const char* field) {
    return fail(h, CBAA_E_MISMATCH, std::string("SketchFile refused: field '") + field + "' differs from this cube");
  };
  if (fc.r != c.r) return mismatch("r");
  if (fc.num_ra != c.num_ra) return mismatch("num_ra");
  if (fc.num_va != c.num_va) return mismatch("num_va");
  if (fc.g != c.g) return mismatch("g");
  for (uint32_t a = 0; a < c.num_ra + c.num_va; ++a)
    if (fc.cbn[a] != c.cbn[a]) return mismatch("cbn");
  for (uint32_t i = 0; i < c.num_ra; ++i)
    if (fc.clbs[i] != c.clbs[i]) return mismatch("clbs");
  if (fc.mangle_a != c.mangle_a) return mismatch("mangle_a");
  if (fc.mangle_b != c.mangle_b) return mismatch("mangle_b");
  if (fc.bv_seed != c.bv_seed) return mismatch("bv_seed");
  for (uint32_t j = 0; j < c.num_va; ++j)
    if (fc.va_seeds[j] != c.va_seeds[j]) return mismatch("va_seeds");
  DeviceGuard dg(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (sparse) {   // offsets + streams to the device, then one thread per block ORs its bits in
    const uint64_t nb = (h->cube_words + kSparseBlockWords - 1) / kSparseBlockWords;
    void* d = nullptr;   // u32 bad flag | offsets | streams
    CK(h, cudaMalloc(&d, 16 + plen));
    int rc = CBAA_OK;
    cudaError_t e = cudaMemsetAsync(d, 0, 16, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync((char*)d + 16, payload, plen, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && mode == CBAA_SKETCH_REPLACE) e = cudaMemsetAsync(h->cube, 0, h->cube_bytes, s);
    if (e != cudaSuccess) rc = cuda_fail(h, e, "sparse SketchFile copy-in");
    if (!rc) {
      const unsigned long long* off = (const unsigned long long*)((char*)d + 16);
      const int grid = (int)std::min<uint64_t>((uint64_t)h->sms * 8, (nb + 127) / 128);
      k_sparse_decode<<<grid, 128, 0, s>>>((const uint8_t*)(off + nb + 1), off, nb, h->cube_words, h->cube,
                                           (uint32_t*)d);
      rc = launch_check(h, "k_sparse_decode");
    }
    uint32_t bad = 0;
    if (!rc) {
      e = cudaMemcpyAsync(&bad, d, 4, cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) rc = cuda_fail(h, e, "sparse SketchFile decode");
    }
    cudaFree(d);
    if (!rc && bad) rc = fail(h, CBAA_E_CONFIG, "SketchFile: malformed sparse stream (varint or position out of range)");
    return rc;
  }
  if (mode == CBAA_SKETCH_REPLACE) {
    CK(h, cudaMemcpyAsync(h->cube, payload, plen, cudaMemcpyHostToDevice, s));
    CK(h, cudaStreamSynchronize(s));
    return CBAA_OK;
  }
  // MERGE: stage the payload on the device in 64 MiB slices and OR them in
  const uint64_t slice = 64ull << 20;
  void* stage = nullptr;
  CK(h, cudaMalloc(&stage, std::min(slice, plen)));
  int rc = CBAA_OK;
  for (uint64_t off = 0; off < plen && rc == CBAA_OK; off += slice) {
    const uint64_t m = std::min(slice, plen - off);
    cudaError_t e = cudaMemcpyAsync(stage, payload + off, m, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) { rc = cuda_fail(h, e, "cudaMemcpyAsync(sketch payload)"); break; }
    MergeSrcs S{};
    S.k = 1;
    S.p[0] = (const uint4*)stage;
    k_or_merge<<<grid_for(h, m / 16, 4), kThreads, 0, s>>>((uint4*)((char*)h->cube + off), S, m / 16);
    rc = launch_check(h, "k_or_merge(sketch)");
    if (rc == CBAA_OK) {
      e = cudaStreamSynchronize(s);   // the staging slice is reused by the next copy
      if (e != cudaSuccess) rc = cuda_fail(h, e, "cudaStreamSynchronize");
    }
  }
  cudaFree(stage);
  return rc;
}

// ------------------------------------------------------------------ peer cubes (CUDA IPC)
static_assert(sizeof(cudaIpcMemHandle_t) == CBAA_IPC_HANDLE_BYTES, "IPC handle size");
static_assert(kSigBytes == CBAA_SIGNAL_BYTES && (kMaxRanks + 1) * 8 <= kSigBytes, "signal area");

int cbaa_ipc_export(cbaa_handle* h, void* out) {
  if (!h || !out) return CBAA_E_ARG;
  if (h->cube_external) return fail(h, CBAA_E_ARG, "cbaa_ipc_export: the cube is caller memory");
  DeviceGuard dg(h->device);
  cudaIpcMemHandle_t mh;
  CK(h, cudaIpcGetMemHandle(&mh, h->cube));
  std::memcpy(out, &mh, sizeof mh);
  return CBAA_OK;
}

int cbaa_ipc_open(cbaa_handle* h, const void* handle, void** dev_ptr) {
  if (!h || !handle || !dev_ptr) return CBAA_E_ARG;
  DeviceGuard dg(h->device);
  cudaIpcMemHandle_t mh;
  std::memcpy(&mh, handle, sizeof mh);
  CK(h, cudaIpcOpenMemHandle(dev_ptr, mh, cudaIpcMemLazyEnablePeerAccess));
  return CBAA_OK;
}

int cbaa_ipc_close(cbaa_handle* h, void* dev_ptr) {
  if (!h || !dev_ptr) return CBAA_E_ARG;
  DeviceGuard dg(h->device);
  CK(h, cudaIpcCloseMemHandle(dev_ptr));
  return CBAA_OK;
}

// ------------------------------------------------------------------ multi-GPU window end
uint64_t cbaa_signal_offset(const cbaa_handle* h) { return h ? sig_offset(h->cube_bytes) : 0; }

int cbaa_peer_barrier(cbaa_handle* h, void* const* peer_cubes, int world, int rank, uint64_t epoch,
                      cbaa_stream stream) {
  if (!h || !peer_cubes || world < 1 || world > kMaxRanks || rank < 0 || rank >= world || epoch == 0)
    return fail(h, CBAA_E_ARG, "cbaa_peer_barrier: bad arguments");
  if (!h->sig) return fail(h, CBAA_E_ARG, "cbaa_peer_barrier: caller memory without room for the signal area");
  DeviceGuard dg(h->device);
  PeerSigs P{};
  for (int k = 0; k < world; ++k) {
    char* base = k == rank ? (char*)h->cube : (char*)peer_cubes[k];
    if (!base) return fail(h, CBAA_E_ARG, "cbaa_peer_barrier: null peer cube");
    P.sig[k] = (unsigned long long*)(base + sig_offset(h->cube_bytes));
  }
  const char* to = std::getenv("CBAA_BARRIER_TIMEOUT_MS");
  const unsigned long long ns = 1000000ull * (to ? std::strtoull(to, nullptr, 10) : 10000ull);
  k_peer_barrier<<<1, kMaxRanks, 0, (cudaStream_t)stream>>>(P, world, rank, (unsigned long long)epoch, ns,
                                                             (uint32_t*)(h->sig + kMaxRanks));
  return launch_check(h, "k_peer_barrier");
}

int cbaa_peer_status(cbaa_handle* h, uint32_t* status) {
  if (!h || !status || !h->sig) return CBAA_E_ARG;
  DeviceGuard dg(h->device);
  CK(h, cudaMemcpy(status, h->sig + kMaxRanks, 4, cudaMemcpyDeviceToHost));
  return CBAA_OK;
}

int cbaa_merge_slice_zc(cbaa_handle* h, const void* const* slices, int k, uint32_t cs_lo, uint32_t cs_hi,
                        cbaa_stream stream) {
  if (!h) return CBAA_E_ARG;
  if (h->G.wpc != 128 || k > 16)   // fused kernel: g = 4096, ≤ 16 peers; otherwise merge, detect counts
    return cbaa_merge_slice(h, slices, k, cs_lo, cs_hi, stream);
  h->zc_fresh = 0;
  if (cs_lo >= cs_hi || cs_hi > h->G.n_cs) return fail(h, CBAA_E_ARG, "cbaa_merge_slice_zc: bad CS range");
  if (k < 0 || (k && !slices)) return fail(h, CBAA_E_ARG, "cbaa_merge_slice_zc: bad k/slices");
  DeviceGuard dg(h->device);
  MergeSrcs S{};
  S.k = k;
  for (int j = 0; j < k; ++j) {
    if (!slices[j] || ((uintptr_t)slices[j] & 15))
      return fail(h, CBAA_E_ARG, "cbaa_merge_slice_zc: null or non-16-byte-aligned slice pointer");
    S.p[j] = (const uint4*)slices[j];
  }
  const uint64_t cols = (uint64_t)(cs_hi - cs_lo) * (h->G.cs_words >> h->G.wpc_log2);
  const int grid = (int)std::min<uint64_t>((uint64_t)h->sms * 8, (cols + kDetWarps - 1) / kDetWarps);
  k_or_merge_zc<<<grid, kDetThreads, 0, (cudaStream_t)stream>>>(h->G, h->cube, S, cs_lo, cs_hi - cs_lo, h->D);
  int rc = launch_check(h, "k_or_merge_zc");
  if (rc) return rc;
  h->zc_fresh = 1;
  h->zc_lo = cs_lo;
  h->zc_hi = cs_hi;
  return CBAA_OK;
}

int cbaa_merge_multicast(cbaa_handle* h, const void* mc_cube, uint32_t cs_lo, uint32_t cs_hi, cbaa_stream stream) {
  if (!h) return CBAA_E_ARG;
  h->zc_fresh = 0;
  if (!mc_cube || ((uintptr_t)mc_cube & 15)) return fail(h, CBAA_E_ARG, "cbaa_merge_multicast: bad multicast address");
  if (cs_lo >= cs_hi || cs_hi > h->G.n_cs) return fail(h, CBAA_E_ARG, "cbaa_merge_multicast: bad CS range");
  DeviceGuard dg(h->device);
  const uint64_t csb = (uint64_t)h->G.cs_words * 4, off = csb * cs_lo, n8 = csb * (cs_hi - cs_lo) / 8;
  k_or_multicast<<<grid_for(h, n8, 4), kThreads, 0, (cudaStream_t)stream>>>(
      (uint64_t*)((char*)h->cube + off), (const uint64_t*)((const char*)mc_cube + off), n8);
  return launch_check(h, "k_or_multicast");
}

void cbaa_sort_hosts(cbaa_host* hosts, uint64_t n) {
  if (!hosts || n < 2) return;
  std::sort(hosts, hosts + n, [](const cbaa_host& a, const cbaa_host& b) {
    if (a.estimate != b.estimate) return a.estimate > b.estimate;
    return a.ip < b.ip;
  });
}

uint64_t cbaa_kernel_launches(const cbaa_handle* h) { return h ? h->launches : 0; }

uint32_t cbaa_update_passes(const cbaa_handle* h) { return h ? h->passes : 0; }

int cbaa_update_plan(const cbaa_handle* h, uint64_t n, char* buf, uint64_t buflen) {
  if (!h || !buf || !buflen) return CBAA_E_ARG;
  std::string p;
  if (h->cfg.update_mode == CBAA_UPDATE_BINNED && binned_ok(h) && n >= h->bin_min) {
    const bool prefix = h->cfg.direction == CBAA_DIR_INNER_PREFIX;
    const bool wide = (h->bin_wide || h->bin_wide_gen) && !h->bin_wc;
    const bool gen = wide && !h->bin_wide;
    const uint32_t samp = ((!prefix || wide) && !h->bin_wc) ? h->bin_sample_log2 : 0u;
    const bool sampled = samp && std::min(n, h->bin_chunk) >= h->bin_sample_min;
    p = std::string(gen ? "binned-wide-generic " : wide ? "binned-wide " : "binned ") +
        (sampled ? "k_bin_sample" : "k_bin_count") + " k_bin_starts " +
        (wide ? "k_bin_scatter_w" : h->bin_wc ? "k_bin_wc" : "k_bin_scatter") + " " +
        (gen ? (h->bin_gen_per_array ? "k_bin_apply_wa+k_bin_log_wg" : "k_bin_apply_wg+k_bin_log_wg")
             : wide ? "k_bin_apply_w+k_bin_log_w" : "k_bin_apply+k_bin_log") +
        (wide ? " entry_bytes=8" : " entry_bytes=4") + (gen ? " bins=" + std::to_string(h->BW.nbins) : "");
  } else {
    p = "direct k_update passes=" + std::to_string(h->passes);
  }
  std::snprintf(buf, buflen, "%s", p.c_str());
  return CBAA_OK;
}

int cbaa_set_phase_timing(cbaa_handle* h, int enable) {
  if (!h) return CBAA_E_ARG;
  h->timing = enable ? 1 : 0;
  h->tused = 0;
  h->tcalls = 0;
  return CBAA_OK;
}

int cbaa_update_phase_ms(cbaa_handle* h, double* ms, int cap, uint64_t* calls) {
  if (!h || !ms || cap < 4) return CBAA_E_ARG;
  DeviceGuard dg(h->device);
  for (int i = 0; i < 4; ++i) ms[i] = 0;
  for (size_t k = 0; k < h->tused; ++k) {
    CK(h, cudaEventSynchronize(h->tev[2 * k + 1]));
    float t = 0;
    CK(h, cudaEventElapsedTime(&t, h->tev[2 * k], h->tev[2 * k + 1]));
    ms[h->tphase[k]] += t;
  }
  if (calls) *calls = h->tcalls;
  h->tused = 0;
  h->tcalls = 0;
  return CBAA_OK;
}

}  // extern "C"
