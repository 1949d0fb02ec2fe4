// Derived sketch geometry shared by the host library and the sm_100a kernels.
// Everything here is a function of cbaa_config (include/cbaa.h) only; it is
// passed to every kernel by value as a __grid_constant__ parameter.
#pragma once
#include <stdint.h>

#include "cbaa.h"

namespace cbaa {

struct Geo {
  uint32_t r, L, num_ra, num_va, narr;
  uint32_t g, wpc, wpc_log2;       // rows per column, 32-bit words per column (g/32), log2(wpc)
  uint32_t rmask;                  // 2^r − 1
  uint32_t n_cs;                   // 2^r
  uint32_t cs_words;               // words per CS = Σ c(i)·g/32
  uint32_t arr_off[CBAA_MAX_ARRAYS];   // word offset of array a inside a CS (S:116 order)
  uint32_t cbn[CBAA_MAX_ARRAYS];
  uint32_t colmask[CBAA_MAX_ARRAYS];   // c(a) − 1
  uint32_t ncols[CBAA_MAX_ARRAYS];     // c(a)
  uint32_t sh[CBAA_MAX_RA];            // RA extraction shift: 2L − clbs(i) − cbn(i)
  uint32_t ep[CBAA_MAX_RA], cp[CBAA_MAX_RA], clbs[CBAA_MAX_RA];
  uint32_t ra_off[CBAA_MAX_RA];        // offset of RA(i) in a CS's zero-count block
  uint32_t ra_cols;                    // Σ_{i<num_ra} c(i)
  uint32_t mangle_a, mangle_b, inv_a, bv_seed;
  uint32_t va_seeds[CBAA_MAX_VA];
  int32_t direction, theta_formula, union_threshold;
  uint32_t n_prefix;
  uint32_t prefix[CBAA_MAX_PREFIXES], pmask[CBAA_MAX_PREFIXES];
  // inner-prefix classification by the top 16 address bits: bit t of full_bits set ⇔ every address with
  // top-16 value t is inner (prefixes /0-/16); bit t of part_bits set ⇔ some are (longer prefixes,
  // exact check).  Device pointers to 2 × 2048 words owned by the handle; null if direction = normalised.
  const uint32_t* full_bits;
  const uint32_t* part_bits;
  uint64_t tuple_cap;
};

// mix32, the fixed avalanche mix of SPEC S:224 (hash family of Q4).
__host__ __device__ __forceinline__ uint32_t mix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x45D9F3Bu;
  h ^= h >> 16;
  h *= 0x45D9F3Bu;
  h ^= h >> 16;
  return h;
}

}  // namespace cbaa
