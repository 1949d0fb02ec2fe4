/*
 * cbaa.h — C ABI of the B200-native CBAA window path (libcbaa.so).
 *
 * CBAA = "Cube of Bits Array Algorithm" of Xu, Ding, Hu, "GPU based Real-time
 * Super Hosts Detection at Distributed Edge Routers" (arXiv 1901.06207).
 * Citations: "P:n" = line n of the paper text, "S:n" = line n of
 * SPEC.md, "Qn" = reading n of DESIGN.md §3.
 *
 * Problem statement: the pairs <inner ip, outer ip> of a
 * time window go in; the inner hosts with at least θ distinct opposite IPs
 * (super hosts, Def. 1) come out.  One handle = one local server's cube of
 * bits arrays (CBA) on one GPU.  Per window the caller does
 *     cbaa_reset → cbaa_update* → [cbaa_merge*] → cbaa_detect.
 *
 * Conventions for every entry point:
 *  - Return value: CBAA_OK (0) or a negative CBAA_E_* code; never throws.
 *    cbaa_last_error(h) holds a one-line explanation of the last failure.
 *  - Pointers named "device" are CUDA device pointers on the handle's device;
 *    "host" pointers are ordinary (optionally pinned) host memory.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Calls are asynchronous and stream-ordered unless documented otherwise;
 *    the caller keeps every buffer it passes alive until `stream` completes.
 *  - IPv4 addresses are host-order uint32 (192.168.1.1 = 0xC0A80101, Q31).
 *  - A handle is single-stream and not thread-safe; distinct handles are
 *    independent (k handles on one GPU simulate k edge routers).
 *
 * Memory layout of the cube (Q27): CSs ascending; inside a CS the
 * arrays RA(0..num_ra-1) then VA(0..num_va-1); inside an array the columns
 * ascending; inside a column the g rows, row j = bit (j mod 32) of 32-bit word
 * j/32 (little-endian), i.e. bit (j mod 8) of byte j/8 — the SPEC's byte format.
 */
#ifndef CBAA_H_
#define CBAA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CBAA_MAX_RA 8
#define CBAA_MAX_VA 8
#define CBAA_MAX_ARRAYS 16
#define CBAA_MAX_PREFIXES 16
#define CBAA_MAX_MERGE 64

/* Status codes. */
#define CBAA_OK 0
#define CBAA_E_CONFIG (-1)    /* config violates an invariant of S:37-41; last_error names it */
#define CBAA_E_ARG (-2)       /* null / misaligned pointer, bad range, wrong device               */
#define CBAA_E_CUDA (-3)      /* a CUDA call failed; last_error carries cudaGetErrorString         */
#define CBAA_E_MISMATCH (-4)  /* merge of cubes that are not the same size                 */
#define CBAA_E_CAPACITY (-5)  /* more hosts than `cap`: *n_out = required count, out = first cap  */
#define CBAA_E_TUPLE_CAP (-6) /* ≥1 CS skipped: ∏|HC(i)| > tuple_cap; others still output */
#define CBAA_E_NOMEM (-7)     /* device allocation failed                                         */

#define CBAA_THETA_PAPER 0    /* θ_bn = g(1+ε)e^{−θ/g} − gε, P:261 (default)                     */
#define CBAA_THETA_INVERTED 1 /* θ_bn = g(1−ε)e^{−θ/g}, Theorem 2 inverted (Q15)           */

/* How the update kernel sets a bit; the resulting cube is identical (bits only go 0 -> 1). */
/* Union-column threshold of Alg. 3 (Q20). */
#define CBAA_UNION_SAME 0     /* reuse the per-CS θ_bn of Alg. 2 for the union column (paper as written)  */
#define CBAA_UNION_THM2 1     /* θ_uc = g(1−ε)e^{−θ/g}: accept iff the Thm. 2 estimate of UC is ≥ θ         */

#define CBAA_UPDATE_TEST_SET 0  /* L1-cached load of the word; RED.OR only if the bit is still 0           */
#define CBAA_UPDATE_RED 1       /* unconditional RED.OR per bit: the paper's write-only update   */
#define CBAA_UPDATE_BINNED 2    /* pairs binned by (CS, row group) and applied in shared memory (large n) */

#define CBAA_DIR_NORMALIZED 0   /* src = inner, dst = outer as given (Q25)                 */
#define CBAA_DIR_INNER_PREFIX 1 /* classify by inner prefixes; swap or skip              */

typedef void* cbaa_stream; /* cudaStream_t */
typedef struct cbaa_handle cbaa_handle;

/* Sketch geometry and seeds (SketchConfig).  Invariants checked by
 * cbaa_config_validate: 1 ≤ r ≤ 16 (or 0); 2 ≤ num_ra ≤ 8; num_va ≤ 8;
 * g a power of two ≥ 32 (Q28); mangle_a odd; 1 ≤ cbn(i) ≤ min(32−r, 24);
 * clbs strictly increasing and < L = 32−r (Q6); Σ|EP(i)| = L; 0 ≤ |CP(i)| ≤
 * |EP((i+1) mod num_ra)|; cube ≤ 16 GiB; bytes per CS (Σ c(i)·g/8) a multiple
 * of 16 (GPU word layout: only g = 32 with a 2-column array can miss it). */
typedef struct {
  uint32_t r;                          /* right bits of the mangled inner IP selecting the CS */
  uint32_t num_ra, num_va;             /* |RA|, |VA|                                            */
  uint32_t g;                          /* rows (bits) per column                                */
  uint8_t cbn[CBAA_MAX_ARRAYS];        /* c(i) = 2^cbn(i) columns of array i (Q9)                */
  uint8_t clbs[CBAA_MAX_RA];           /* CL_bs(i): LP-relative, MSB-first start offsets (Q6, Q7)       */
  uint32_t mangle_a, mangle_b;         /* mangle(x) = a·x + b mod 2^32, a odd (Q3)               */
  uint32_t bv_seed;                    /* row hash H_bv = mix32(mangled oip ⊕ bv_seed) (Q2, Q4)  */
  uint32_t va_seeds[CBAA_MAX_VA];      /* H_j = mix32(LP ⊕ va_seeds[j]) (Q4, Q10)                */
  int32_t theta_formula;               /* CBAA_THETA_PAPER | CBAA_THETA_INVERTED                         */
  int32_t direction;                   /* CBAA_DIR_NORMALIZED | CBAA_DIR_INNER_PREFIX                    */
  uint64_t tuple_cap;                  /* per-CS cap on ∏|HC(i)|, default 2^24                   */
  uint32_t n_prefixes;                 /* inner prefixes used with CBAA_DIR_INNER_PREFIX                 */
  uint32_t inner_prefix[CBAA_MAX_PREFIXES];
  uint32_t inner_mask[CBAA_MAX_PREFIXES]; /* ip is inner iff (ip & mask[k]) == prefix[k] for some k      */
  uint32_t update_passes;              /* address-range passes of the update (0 = auto)   */
  uint32_t hit_capacity;               /* device hit buffer entries per detect (0 = 2^20)               */
  uint32_t update_mode;                /* CBAA_UPDATE_* (cbaa_config_default: BINNED)      */
  uint32_t join_capacity;              /* CP-chain buffer of the |RA| = 3 join (0 = 2^22); on overflow    */
                                       /* detect redoes the window with the Cartesian enumeration          */
  uint32_t detect_overlap;             /* 1: detect will run beside another handle's update (pipelined    */
                                       /* windows): window-end kernels use no shared memory so they fit   */
                                       /* next to the update's CTAs; 0: fastest standalone detect (TMA)   */
  uint32_t bin_min_pairs;              /* CBAA_UPDATE_BINNED: calls with fewer pairs take the direct      */
                                       /* kernel (0 = auto: max(2^20, cube words / 4), and cubes up to    */
                                       /* 0.6 of L2 always direct)                                         */
  int32_t union_threshold;             /* Alg. 3 threshold (Q20): CBAA_UNION_SAME (default, θ_bn of Alg. 2 as */
                                       /* written at P:309) | CBAA_UNION_THM2 (θ_uc = g(1−ε)e^{−θ/g}: Thm. 2  */
                                       /* solved for Z, so a host is output iff its estimate ≥ θ)    */
  uint32_t reserved;
} cbaa_config;

/* One restored super host (Alg. 3 output). */
typedef struct {
  uint32_t ip;       /* original inner IP = unmangle((lp << r) | cs) */
  uint32_t cs;       /* CS index = RP                                               */
  uint32_t lp;       /* restored left part                                  */
  uint32_t z;        /* zero bits of the union column (Def. 2)               */
  double estimate;   /* −g·ln(Z/(g−g·ε)) (Thm. 2); +inf if Z = 0 (Q21)      */
} cbaa_host;

/* Per-CS window statistics of a detect. */
typedef struct {
  uint64_t ztot;          /* zero bits of RA(0) of the CS (η source, Q12)                 */
  double eta;             /* −c0·g·ln(ztot/(c0·g)); +inf if ztot = 0                        */
  double eps;             /* Theorem 1 over all arrays, capped at 1−2^−20   */
  double theta_bn;        /* zero-bit threshold (P:261 or Q15), clamped ≥ 0                 */
  uint32_t zmax;          /* ⌊θ_bn⌋ clamped to [0, g]: accept iff Z ≤ zmax (Q16)            */
  uint32_t n_hot[CBAA_MAX_RA]; /* |HC(i)| (Alg. 2)                                          */
  uint64_t tuples;        /* ∏|HC(i)| (saturating)                                          */
  uint64_t candidates;    /* tuples passing the CP check (Alg. 3)                 */
  uint64_t hits;          /* candidates accepted by the union-column test           */
  int32_t overflow;       /* 1: tuples > tuple_cap, CS skipped                      */
  uint32_t zmax_uc;       /* ⌊θ_uc⌋ clamped to [0, g]: Alg. 3 accepts Z_uc ≤ zmax_uc (= zmax   */
                          /* unless union_threshold = CBAA_UNION_THM2)                         */
  double theta_uc;        /* union-column threshold of Alg. 3 (= theta_bn by default, Q20)   */
} cbaa_cs_stats;

/* ---------------------------------------------------------------- host only
 * These three need no GPU. */

/* Paper geometry (r=4, |RA|=3, |VA|=1, g=c=2^12) with clbs = [0,10,20]
 * (Q8) and the seeds of Q3/Q4; θ formula = paper; tuple_cap = 2^24. */
int cbaa_config_default(cbaa_config* out);

/* Checks every invariant above.  On failure returns CBAA_E_CONFIG and writes
 * the violated rule into err (errlen bytes, NUL-terminated) when non-null. */
int cbaa_config_validate(const cbaa_config* cfg, char* err, uint64_t errlen);

/* Cube size 2^r·Σ_i c(i)·g/8 bytes; 0 for an invalid config. */
uint64_t cbaa_cube_bytes(const cbaa_config* cfg);

/* ----------------------------------------------------------------- lifetime */

/* Validates cfg, selects `device`, allocates the cube (zeroed) and all detect
 * scratch.  *out owns everything until cbaa_destroy. */
int cbaa_create(const cbaa_config* cfg, int device, cbaa_handle** out);

/* Same, but the cube lives in caller-owned DEVICE memory `cube` (≥ cube_bytes,
 * 256-byte aligned), e.g. a symmetric-memory buffer that peer GPUs map over
 * NVLink so cbaa_merge_slice can pull their slices directly.
 * The memory is zeroed here and never freed by the library.  With
 * cube_nbytes ≥ cbaa_signal_offset + CBAA_SIGNAL_BYTES the tail also holds the
 * signal area of cbaa_peer_barrier (library-owned cubes always have one). */
int cbaa_create_ext(const cbaa_config* cfg, int device, void* cube, uint64_t cube_nbytes, cbaa_handle** out);
void cbaa_destroy(cbaa_handle* h);
int cbaa_get_config(const cbaa_handle* h, cbaa_config* out);

/* Window reset: cube := 0 (implicit per window). Async on stream. */
int cbaa_reset(cbaa_handle* h, cbaa_stream stream);

/* ------------------------------------------------------------------- update */

/* Alg. 1 for n pairs: src[k], dst[k] are DEVICE arrays of
 * host-order IPv4 (src = inner, dst = outer unless direction = INNER_PREFIX).
 * Sets |RA|+|VA| bits per pair with 32-bit atomic OR (Q11); with the default
 * update_mode the word is loaded first and only a missing bit is ORed in — the
 * cube is identical either way.  With CBAA_UPDATE_BINNED and n above the
 * handle's threshold the pairs are first binned by (CS, row group) into a
 * device scratch of ~4-6 B per pair plus a 6 B/pair overflow log (≤ 2^28 pairs
 * per chunk, allocated on first use) and the bits are set in shared memory,
 * then OR-ed into the cube; below the threshold, or for geometries whose
 * tables do not fit, the call takes the test-and-set kernel.  Chunks of
 * ≥ 2^24 normalised pairs size their bin regions from a sample (8 of every
 * 512 pairs); entries that overflow a region are applied from the overflow
 * log, so the cube never depends on the sample.  Environment knobs read at
 * cbaa_create (tests, A/B): CBAA_BIN_SAMPLE (log2 of the sampling period,
 * 0 = exact count), CBAA_BIN_SAMPLE_MIN, CBAA_BIN_SCATTER=wc (write-combining
 * scatter, exact count), CBAA_BIN_CHUNK, CBAA_BIN_MIN, CBAA_BIN_WIDE=0 (32-bit
 * entries only), CBAA_BIN_WIDE_GEN=0/2 (generic wide entries off / wherever
 * they fit), CBAA_SCATTER_PF (the scatter's L2 prefetch; 0 = off).  Updates accumulate until cbaa_reset; calls on
 * one handle must be stream-ordered with its detect/merge/reset.  Any 4-byte
 * alignment is accepted (16-B aligned arrays take the vector path).  Async on
 * stream. */
int cbaa_update(cbaa_handle* h, const uint32_t* src, const uint32_t* dst, uint64_t n, cbaa_stream stream);

/* Same for interleaved ("packed") pairs in one DEVICE array: pairs[2k] = src,
 * pairs[2k+1] = dst (8-byte aligned; 16-byte aligned arrays take 128-bit loads
 * of two pairs).  Async on stream. */
int cbaa_update_pairs(cbaa_handle* h, const uint32_t* pairs, uint64_t n, cbaa_stream stream);

/* Same as cbaa_update for HOST arrays (pinned or pageable): the library copies
 * them to the device in chunks on its own copy stream, double-buffered and
 * overlapped with the update kernels (the local-server buffer → GPU copy of
 * P:338).  Returns after every copy has been enqueued; stream-ordered. */
int cbaa_update_host(cbaa_handle* h, const uint32_t* src, const uint32_t* dst, uint64_t n, cbaa_stream stream);

/* Pairs dropped by the INNER_PREFIX classification since the last reset
 * (zero or two inner endpoints).  Synchronizes stream. */
int cbaa_skipped(cbaa_handle* h, uint64_t* out, cbaa_stream stream);

/* -------------------------------------------------------------------- merge */

/* Global merge by bitwise OR (Q1): cube |= cubes[0] | … | cubes[k−1].
 * Each cubes[j] is a DEVICE pointer to a full cube of identical geometry
 * (nbytes must equal cbaa_cube_bytes; the caller checks seed identity).
 * k ≤ CBAA_MAX_MERGE.  Peer pointers are allowed. Async on stream. */
int cbaa_merge(cbaa_handle* h, const void* const* cubes, int k, uint64_t nbytes, cbaa_stream stream);

/* Merge of a CS range only: slices[j] points at the bytes of CSs
 * [cs_lo, cs_hi) of a cube of identical geometry (contiguous, CS-aligned).
 * Used when each rank owns a CS range. Async on stream. */
int cbaa_merge_slice(cbaa_handle* h, const void* const* slices, int k, uint32_t cs_lo, uint32_t cs_hi,
                     cbaa_stream stream);

/* Pull-OR of a CS range fused with the window-end zero counts (a8 + a9, P:249,
 * P:258-261): like cbaa_merge_slice, and in the same pass over the owned bytes
 * the zero count of every RA column of [cs_lo, cs_hi) is recorded, so the next
 * cbaa_detect_range over exactly that range skips its own zero-count pass.  Any
 * later reset/update/merge discards those counts.  g ≠ 4096 or k > 16: plain
 * cbaa_merge_slice (the detect counts as usual).  Async on stream. */
int cbaa_merge_slice_zc(cbaa_handle* h, const void* const* slices, int k, uint32_t cs_lo, uint32_t cs_hi,
                        cbaa_stream stream);

/* NVLink SHARP (NVLS) merge: mc_cube is the MULTICAST address of a cube buffer
 * that every rank holds at the same offsets (e.g. torch symmetric memory's
 * multicast_ptr); the switch ORs the ranks' bytes of CSs [cs_lo, cs_hi)
 * (multimem.ld_reduce .or.b64) and this handle's cube receives the result.
 * The caller orders it after every rank's update (cbaa_peer_barrier or the
 * symmetric-memory barrier).  Requires multicast support.  Async on stream. */
int cbaa_merge_multicast(cbaa_handle* h, const void* mc_cube, uint32_t cs_lo, uint32_t cs_hi, cbaa_stream stream);

/* ------------------------------------------------------------------- detect */

/* Window end over every CS: zero counts → η, ε, θ_bn, zmax per CS
 * → hot columns (Alg. 2) → tuple CP-join and union-column check (Alg. 3) →
 * hosts sorted by estimate descending then ip ascending.
 * out: HOST array of `cap` entries; *n_out = number of hosts found.
 * stats: HOST array of 2^r entries, or NULL.  SYNCHRONIZES stream.
 * Returns CBAA_E_CAPACITY if *n_out > cap, CBAA_E_TUPLE_CAP if a CS overflowed
 * (both still fill out/stats). */
int cbaa_detect(cbaa_handle* h, uint32_t theta, cbaa_host* out, uint64_t cap, uint64_t* n_out,
                cbaa_cs_stats* stats, cbaa_stream stream);

/* Same restricted to CSs [cs_lo, cs_hi); stats then holds cs_hi − cs_lo entries. */
int cbaa_detect_range(cbaa_handle* h, uint32_t theta, uint32_t cs_lo, uint32_t cs_hi, cbaa_host* out,
                      uint64_t cap, uint64_t* n_out, cbaa_cs_stats* stats, cbaa_stream stream);

/* ------------------------------------------------------- SketchFile "CBA1"
 * The transport of a local CBA to the global server ("each local server
 * will send its CBA"), in SPEC's exact wire format (little-
 * endian): "CBA1", u16 version = 1, u8 r, u8 num_ra, u8 num_va, u32 g,
 * (num_ra+num_va) × u8 cbn, num_ra × u8 clbs, u32 mangle_a, u32 mangle_b,
 * u32 bv_seed, num_va × u32 va_seeds, u64 payload bytes, payload = the cube in
 * the byte layout above.  θ formula, tuple cap and direction are not part of a
 * sketch's identity and are not stored. */
#define CBAA_SKETCH_REPLACE 0  /* cube := file payload            */
#define CBAA_SKETCH_MERGE 1    /* cube |= file payload     */

/* Size in bytes of the SketchFile of this handle's cube. */
uint64_t cbaa_sketch_bytes(const cbaa_handle* h);

/* Writes the SketchFile into the HOST buffer out (cap bytes); *n_written = size.
 * Returns CBAA_E_CAPACITY (and the required size) if cap is too small.
 * Synchronizes stream (the cube is read after earlier work on it). */
int cbaa_serialize(cbaa_handle* h, void* out, uint64_t cap, uint64_t* n_written, cbaa_stream stream);

/* The optional sparse form ("optionally sparse"): the
 * same header with magic "CBA2" (its u64 = the dense cube length), then u32
 * block bits = 32768, u64 blocks = ⌈cube bits / 32768⌉, (blocks + 1) × u64 byte
 * offsets of the blocks' streams (from 0, ascending), then the streams: a
 * block's set-bit positions p0 < p1 < … as the gaps p0, p1 − p0 − 1, … in
 * LEB128 (7 bits per byte, low group first, bit 7 = more).  Encoded on the
 * device (two passes: stream sizes, then the streams); *n_written = file size
 * (CBAA_E_CAPACITY with that size if cap is too small).  cbaa_sketch_config and
 * cbaa_deserialize accept both forms.  Synchronizes stream. */
int cbaa_serialize_sparse(cbaa_handle* h, void* out, uint64_t cap, uint64_t* n_written, cbaa_stream stream);

/* Parses a SketchFile header from HOST bytes into *out (other fields default).
 * No GPU needed.  CBAA_E_CONFIG with last-error-style text in err (errlen bytes)
 * names the bad field: magic, version, a geometry invariant, or the payload length. */
int cbaa_sketch_config(const void* in, uint64_t n, cbaa_config* out, char* err, uint64_t errlen);

/* Loads (REPLACE) or OR-merges (MERGE) a HOST SketchFile into the cube.  The
 * header must match this handle's geometry and seeds exactly; otherwise
 * CBAA_E_MISMATCH and last_error names the first differing field.
 * Returns after the payload has been copied (the host buffer may be reused). */
int cbaa_deserialize(cbaa_handle* h, const void* in, uint64_t n, int mode, cbaa_stream stream);

/* ------------------------------------------------------- peer cubes (CUDA IPC)
 * For the window-end exchange between router processes without a staging
 * collective: each process exports its cube, opens its peers' cubes (NVLink
 * P2P mappings on a multi-GPU node; the same device also works), and
 * cbaa_merge_slice reads the peers' CS slices directly. */
#define CBAA_IPC_HANDLE_BYTES 64

/* Writes this handle's cube IPC handle (CBAA_IPC_HANDLE_BYTES) into out.
 * Fails with CBAA_E_ARG for cubes created by cbaa_create_ext. */
int cbaa_ipc_export(cbaa_handle* h, void* out);

/* Maps a peer process's exported cube; *dev_ptr is valid on this handle's
 * device until cbaa_ipc_close.  The peer cube must have the same geometry. */
int cbaa_ipc_open(cbaa_handle* h, const void* handle, void** dev_ptr);
int cbaa_ipc_close(cbaa_handle* h, void* dev_ptr);

/* ------------------------------------------------- device-side router barrier
 * A cube allocation carries, after the cube (at cbaa_signal_offset bytes from
 * its start), CBAA_SIGNAL_BYTES of signals: u64 epoch slots (one per rank, at
 * most 64 ranks) and a u32 status.  Peers reach it through the same mapping as
 * the cube (CUDA IPC or symmetric memory), so no host round trip is needed. */
#define CBAA_SIGNAL_BYTES 4096
uint64_t cbaa_signal_offset(const cbaa_handle* h);

/* Stream-ordered barrier of `world` routers: after every prior operation on
 * `stream` (the window's update) is complete and visible system-wide, writes
 * `epoch` (> 0, increasing per barrier) into slot `rank` of every peer's signal
 * area and waits ON THE DEVICE until all peers have written it into this
 * handle's.  peer_cubes[k] = rank k's cube base as mapped here (this rank's
 * entry is ignored).  One one-CTA kernel; after CBAA_BARRIER_TIMEOUT_MS
 * (default 10000) it stops waiting and sets the status word (cbaa_peer_status)
 * instead of hanging the GPU.  Async on stream. */
int cbaa_peer_barrier(cbaa_handle* h, void* const* peer_cubes, int world, int rank, uint64_t epoch,
                      cbaa_stream stream);
/* Synchronous read of the status word: 0 = every barrier completed, 1 = one timed out. */
int cbaa_peer_status(cbaa_handle* h, uint32_t* status);

/* The output order of S:418 (estimate descending, then ip ascending) on a HOST
 * array, e.g. for host lists gathered from several ranks' detect_range calls. */
void cbaa_sort_hosts(cbaa_host* hosts, uint64_t n);

/* ---------------------------------------------------------------- inspection */

/* Device pointer and size of the cube (for NCCL exchange and parity dumps). */
int cbaa_cube_view(cbaa_handle* h, void** dev_ptr, uint64_t* nbytes);

/* Zero count of every RA column (Alg. 2 input), DEVICE out of
 * 2^r·Σ_{i<num_ra} c(i) uint32 in the order cs → RA(i) → column.  Async. */
int cbaa_zero_counts(cbaa_handle* h, uint32_t* out, cbaa_stream stream);

/* After a detect: HOST copies of the hot-column lists (per CS, per RA(i),
 * ascending; counts in stats.n_hot) — `out` holds 2^r·Σ c(i) entries laid
 * out like cbaa_zero_counts with each (cs, i) block's first n_hot entries
 * valid.  Synchronizes stream. */
int cbaa_hot_columns(cbaa_handle* h, uint32_t* out, cbaa_stream stream);

/* Record candidate LPs during the next detects (debug; costs one atomic per
 * candidate).  cbaa_candidates copies (cs << 32 | lp) of the last detect into
 * a HOST array of cap entries, unordered; *n_out = total.  Synchronizes. */
int cbaa_set_record_candidates(cbaa_handle* h, int enable, uint64_t capacity);
int cbaa_candidates(cbaa_handle* h, uint64_t* out, uint64_t cap, uint64_t* n_out, cbaa_stream stream);

/* Test-only: the device-side mapping of Alg. 1 for n pairs (DEVICE arrays):
 * cs[k], cols[k·(num_ra+num_va) + a], row[k].  Async on stream. */
int cbaa_debug_map(cbaa_handle* h, const uint32_t* iip, const uint32_t* oip, uint64_t n, uint32_t* cs,
                   uint32_t* cols, uint32_t* row, cbaa_stream stream);

/* Number of kernels this handle has launched since creation (bench evidence). */
uint64_t cbaa_kernel_launches(const cbaa_handle* h);

/* Update passes the handle uses (resolved from update_passes = 0). */
uint32_t cbaa_update_passes(const cbaa_handle* h);

/* Per-kernel timing of the update path (bench evidence).  With enable = 1 the
 * handle records a CUDA event pair around every update kernel it launches, on
 * the stream that kernel is launched on.  cbaa_update_phase_ms synchronizes
 * those events and writes the milliseconds summed per phase over all update
 * calls since the previous query (or since enabling) into ms[0..3]:
 *   binned path: ms[0] k_bin_sample or k_bin_count, ms[1] k_bin_starts,
 *                ms[2] k_bin_scatter (or k_bin_wc), ms[3] k_bin_apply + k_bin_log;
 *   direct path: ms[0] k_update (every pass), ms[1..3] = 0,
 * and the number of update calls in *calls (nullable).  ms needs cap >= 4
 * (CBAA_E_ARG otherwise).  Host-side bookkeeping only; kernels are unchanged. */
int cbaa_set_phase_timing(cbaa_handle* h, int enable);
int cbaa_update_phase_ms(cbaa_handle* h, double* ms, int cap, uint64_t* calls);

/* The kernels a cbaa_update call of n pairs would launch, per phase, as one NUL-terminated line written
 * into buf (buflen bytes, truncated): "binned-wide k_bin_sample k_bin_starts k_bin_scatter_w
 * k_bin_apply_w+k_bin_log_w entry_bytes=8" (paper geometry), "binned-wide-generic ... k_bin_apply_wg (or
 * k_bin_apply_wa, one CTA per bin and array)+k_bin_log_wg entry_bytes=8 bins=B" (other geometries with
 * 256-4096 wide bins), "binned ... entry_bytes=4", or "direct k_update passes=P".
 * Host only, no GPU work; CBAA_E_ARG if h or buf is null (bench evidence: which kernel is dominant). */
int cbaa_update_plan(const cbaa_handle* h, uint64_t n, char* buf, uint64_t buflen);

const char* cbaa_strerror(int code);
const char* cbaa_last_error(const cbaa_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* CBAA_H_ */
