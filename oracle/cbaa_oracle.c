/*
 * CBAA CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, scalar C implementation of the CBAA window path of
 *   Xu, Ding, Hu, "GPU based Real-time Super Hosts Detection at Distributed
 *   Edge Routers" (arXiv 1901.06207), /root/reference/PAPER.md (cited "P:n"),
 * following the readings pinned in /root/reference/SPEC.md ("S:n") and in
 * DESIGN.md §3 ("Q<n>" = SURVEY.md §8(c) reading table).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (include/cbaa.h, paper_1901_06207_b200/) never links, imports or calls it,
 * and shares no code with it (no headers, helpers or tables).
 *
 * Style: one scalar loop per step, per-bit loops where the paper speaks of
 * bits, the paper's order and notation, fp64 for every real number.
 * No blocking, fusion or reordering beyond what the algorithm states.
 *
 * Parity status of every function: pinned by tests/test_oracle_pins.py
 * (see the pin named next to each function).  None is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MAX_ARR 16
#define ORC_MAX_RA 8
#define ORC_MAX_VA 8
#define ORC_MAX_PREFIX 16

/* Oracle-private configuration record.  Deliberately NOT the
 * layout of cbaa_config in include/cbaa.h: the two sides share nothing. */
typedef struct {
  uint32_t r;                    /* right bits selecting the CS        */
  uint32_t num_ra, num_va;       /* |RA|, |VA|                          */
  uint32_t g;                    /* rows per column                     */
  uint32_t cbn[ORC_MAX_ARR];     /* column-index bits, c(i) = 2^cbn(i)  */
  uint32_t clbs[ORC_MAX_RA];     /* LP-relative start offsets CL_bs(i) (Q6)     */
  uint32_t mangle_a, mangle_b;   /* affine mangling (Q3)                        */
  uint32_t bv_seed;              /* H_bv seed (Q4)                              */
  uint32_t va_seeds[ORC_MAX_VA]; /* H_j seeds (Q4)                              */
  int32_t theta_formula;         /* 0 = paper θ_bn, 1 = inverted Thm.2  */
  uint64_t tuple_cap;            /* cap on ∏|HC(i)| per CS              */
  int32_t direction;             /* 0 = normalized input, 1 = inner-prefix      */
  uint32_t n_prefix;
  uint32_t prefix[ORC_MAX_PREFIX], prefix_mask[ORC_MAX_PREFIX];
  int32_t union_threshold;       /* Alg. 3 threshold (Q20): 0 = θ_bn of Alg. 2,
                                    1 = union-specific θ_uc (Thm. 2 inverted)  */
} orc_config;

typedef struct {
  uint32_t ip;       /* original (unmangled) inner IP          */
  uint32_t cs;       /* CS index = RP                          */
  uint32_t lp;       /* restored left part                     */
  uint32_t z;        /* zero bits of the union column          */
  double estimate;   /* Thm. 2 corrected estimate              */
} orc_host;

typedef struct {
  uint64_t ztot;     /* zero bits in RA(0) of the CS           */
  double eta, eps, theta_bn;
  uint32_t zmax;     /* floor(θ_bn), clamped to [0, g]         */
  uint32_t n_hot[ORC_MAX_RA];
  uint64_t tuples;      /* ∏|HC(i)| (saturating)                 */
  uint64_t candidates;  /* tuples passing the CP check           */
  uint64_t hits;        /* tuples accepted by the union check    */
  int32_t overflow;     /* 1 if tuples > tuple_cap (skipped)     */
  uint32_t zmax_uc;     /* floor(θ_uc): Alg. 3 accepts Z ≤ this  */
  double theta_uc;      /* union-column threshold of Alg. 3      */
} orc_cs_stats;

/* ---------------------------------------------------------------- hashing */

/* mix32, S:224 (the paper leaves H_bv and H_j unspecified, Q4).
 * Pin: mix32 vectors in tests/golden/mix32.txt + bijection. */
uint32_t orc_mix32(uint32_t x) {
  uint32_t h = x;
  h ^= h >> 16;
  h = h * 0x45D9F3Bu;
  h ^= h >> 16;
  h = h * 0x45D9F3Bu;
  h ^= h >> 16;
  return h;
}

/* Mangling ("each IP will be hashed by a mangling operation";
 * affine reading Q3): m = A·x + B mod 2^32.  Pin: bijection. */
uint32_t orc_mangle(const orc_config* c, uint32_t x) { return c->mangle_a * x + c->mangle_b; }

/* Inverse of odd A modulo 2^32 by the extended Euclidean algorithm.
 * Pin: A·inv ≡ 1 and the stated inverse 0x0E8B2F51 of 0x9E3779B1 (Q3). */
uint32_t orc_inverse_mod32(uint32_t a) {
  int64_t t = 0, newt = 1;
  int64_t r = (int64_t)1 << 32, newr = a;
  while (newr != 0) {
    int64_t q = r / newr, tmp;
    tmp = t - q * newt; t = newt; newt = tmp;
    tmp = r - q * newr; r = newr; newr = tmp;
  }
  /* r == gcd == 1 for odd a */
  if (t < 0) t += (int64_t)1 << 32;
  return (uint32_t)t;
}

/* P:175 "we use the mangling operation again to acquire the origin IP". */
uint32_t orc_unmangle(const orc_config* c, uint32_t m) {
  return orc_inverse_mod32(c->mangle_a) * (m - c->mangle_b);
}

/* ------------------------------------------------------------ config */

/* |EP(i)| = CL_bs((i+1) mod |RA|) − CL_bs(i), taken mod L (Q6);
 * |CP(i)| = cbn(i) − |EP(i)| (Q18).  Pin: S:67 [10,10,8]/[2,2,4]. */
void orc_ep_cp(const orc_config* c, int32_t* ep, int32_t* cp) {
  int32_t L = 32 - (int32_t)c->r;
  for (uint32_t i = 0; i < c->num_ra; ++i) {
    int32_t nxt = (int32_t)c->clbs[(i + 1) % c->num_ra];
    int32_t cur = (int32_t)c->clbs[i];
    int32_t e = nxt - cur;
    while (e < 0) e += L;
    e %= L;
    ep[i] = e;
    cp[i] = (int32_t)c->cbn[i] - e;
  }
}

static int is_pow2(uint64_t x) { return x != 0 && (x & (x - 1)) == 0; }

/* Validate against S:37-41 (+ Q28/Q29).  Returns 0 if valid, otherwise the
 * number of the violated rule, and writes its text to err. */
int orc_validate(const orc_config* c, char* err, int errlen) {
#define FAIL(n, msg) do { if (err && errlen > 0) snprintf(err, (size_t)errlen, "%s", msg); return n; } while (0)
  if (c->r > 16) FAIL(1, "r must be <= 16");
  if (c->num_ra < 2 || c->num_ra > ORC_MAX_RA) FAIL(2, "num_ra must be in [2, 8] (a single RA has sum ep = 0 != L, S:66)");
  if (c->num_va > ORC_MAX_VA) FAIL(3, "num_va must be <= 8");
  if (!is_pow2(c->g) || c->g < 32) FAIL(4, "g must be a power of two >= 32 (S:40, Q28)");
  if ((c->mangle_a & 1u) == 0) FAIL(5, "mangle_a must be odd (S:40)");
  int32_t L = 32 - (int32_t)c->r;
  for (uint32_t i = 0; i < c->num_ra + c->num_va; ++i)
    if (c->cbn[i] < 1 || (int32_t)c->cbn[i] > L || c->cbn[i] > 24) FAIL(6, "cbn(i) must be in [1, min(L, 24)]");
  for (uint32_t i = 0; i < c->num_ra; ++i) {
    if ((int32_t)c->clbs[i] >= L) FAIL(7, "clbs(i) must be < L = 32 - r (Q6)");
    if (i > 0 && c->clbs[i] <= c->clbs[i - 1]) FAIL(8, "clbs must be strictly increasing (S:41)");
  }
  int32_t ep[ORC_MAX_RA], cp[ORC_MAX_RA];
  orc_ep_cp(c, ep, cp);
  int32_t sum = 0;
  for (uint32_t i = 0; i < c->num_ra; ++i) sum += ep[i];
  if (sum != L) FAIL(9, "sum of ep(i) must equal L = 32 - r (S:38)");
  for (uint32_t i = 0; i < c->num_ra; ++i) {
    if (cp[i] < 0) FAIL(10, "cp(i) = cbn(i) - ep(i) must be >= 0 (S:39)");
    if (cp[i] > ep[(i + 1) % c->num_ra]) FAIL(11, "cp(i) must be <= ep((i+1) mod num_ra) (S:39)");
  }
  if (c->theta_formula != 0 && c->theta_formula != 1) FAIL(12, "theta_formula must be 0 (paper) or 1 (inverted)");
  if (c->union_threshold != 0 && c->union_threshold != 1) FAIL(12, "union_threshold must be 0 (same as Alg. 2) or 1 (union)");
  if (c->direction != 0 && c->direction != 1) FAIL(13, "direction must be 0 (normalized) or 1 (inner prefix)");
  if (c->n_prefix > ORC_MAX_PREFIX) FAIL(14, "at most 16 inner prefixes");
  return 0;
#undef FAIL
}

/* Columns of array a: c(a) = 2^cbn(a). */
static uint64_t ncols(const orc_config* c, uint32_t a) { return (uint64_t)1 << c->cbn[a]; }

/* Bits in one CS: Σ_i c(i)·g.  Pin: 2^30 bits in the paper geometry. */
uint64_t orc_cs_bits(const orc_config* c) {
  uint64_t s = 0;
  for (uint32_t a = 0; a < c->num_ra + c->num_va; ++a) s += ncols(c, a) * c->g;
  return s;
}

uint64_t orc_cube_bytes(const orc_config* c) { return ((uint64_t)1 << c->r) * orc_cs_bits(c) / 8; }

/* Bit address of (cs, array a, column col, row) per S:116: cs ascending,
 * arrays RA(0..) then VA(0..), columns contiguous, rows inside a column. */
uint64_t orc_bit_address(const orc_config* c, uint32_t cs, uint32_t a, uint64_t col, uint32_t row) {
  uint64_t off = (uint64_t)cs * orc_cs_bits(c);
  for (uint32_t i = 0; i < a; ++i) off += ncols(c, i) * c->g;
  return off + col * c->g + row;
}

/* Row j is bit (j mod 8) of byte j/8, LSB first. */
static int get_bit(const uint8_t* cube, uint64_t addr) { return (cube[addr / 8] >> (addr % 8)) & 1; }
static void set_bit(uint8_t* cube, uint64_t addr) { cube[addr / 8] |= (uint8_t)(1u << (addr % 8)); }

/* ---------------------------------------------------------- ip mapping */

/* RP = right r bits, LP = left 32−r bits (Alg. 1). */
uint32_t orc_rp(const orc_config* c, uint32_t m) { return c->r == 0 ? 0 : (m & ((1u << c->r) - 1u)); }
uint32_t orc_lp(const orc_config* c, uint32_t m) { return c->r == 0 ? m : (m >> c->r); }

/* RA column, Alg. 1 P:235 "extract cbn(i) bits from CL_bs(i)": read the
 * bits at LP offsets clbs(i), clbs(i)+1, ..., clbs(i)+cbn(i)−1 (mod L, Q6)
 * of the MSB-first L-bit string of lp; the first bit read becomes the MSB
 * of the column index (Q7).  Pin: S:180 worked example (0xA57) + the
 * exhaustive LP round trip + the closed form rotl (tests). */
uint32_t orc_ra_col(const orc_config* c, uint32_t lp, uint32_t i) {
  uint32_t L = 32 - c->r;
  uint32_t col = 0;
  for (uint32_t t = 0; t < c->cbn[i]; ++t) {
    uint32_t pos = (c->clbs[i] + t) % L;         /* offset from the MSB of LP */
    uint32_t bit = (lp >> (L - 1 - pos)) & 1u;   /* offset 0 = bit L−1        */
    col = (col << 1) | bit;
  }
  return col;
}

/* VA column, Alg. 1 P:239 "CL(j) ⇐ H_j(LP)"; H_j = mix32(LP ⊕ seed_j) mod c (Q4, Q10). */
uint32_t orc_va_col(const orc_config* c, uint32_t lp, uint32_t j) {
  return orc_mix32(lp ^ c->va_seeds[j]) & (uint32_t)(ncols(c, c->num_ra + j) - 1);
}

/* Row, Alg. 1 P:230 "bvIdx ⇐ H_bv(oip)" on the mangled oip (Q2). */
uint32_t orc_row(const orc_config* c, uint32_t moip) { return orc_mix32(moip ^ c->bv_seed) & (c->g - 1); }

/* Alg. 1 per pair: cs, all |RA|+|VA| columns and the row.  Used by the unit
 * pins and by orc_update below. */
void orc_map_pair(const orc_config* c, uint32_t iip, uint32_t oip, uint32_t* cs, uint32_t* cols, uint32_t* row) {
  uint32_t mi = orc_mangle(c, iip);
  uint32_t mo = orc_mangle(c, oip);
  uint32_t lp = orc_lp(c, mi);
  *cs = orc_rp(c, mi);
  *row = orc_row(c, mo);
  for (uint32_t i = 0; i < c->num_ra; ++i) cols[i] = orc_ra_col(c, lp, i);
  for (uint32_t j = 0; j < c->num_va; ++j) cols[c->num_ra + j] = orc_va_col(c, lp, j);
}

/* Alg. 3: CP check, then LP = concatenation of the EPs.
 * CP(i) = low |CP(i)| bits of hc_i must equal the first |CP(i)| bits of
 * hc_{(i+1) mod |RA|} (Q19).  EP(i) = the high |EP(i)| bits of hc_i,
 * placed at LP offsets clbs(i).. (mod L).  Returns 1 and *lp, or 0 (the
 * "return −1" path).  Pin: round trip exhaustive over 2^28 LPs. */
int orc_lp_from_tuple(const orc_config* c, const uint32_t* cols, uint32_t* lp_out) {
  int32_t ep[ORC_MAX_RA], cp[ORC_MAX_RA];
  orc_ep_cp(c, ep, cp);
  uint32_t L = 32 - c->r;
  for (uint32_t i = 0; i < c->num_ra; ++i) {
    uint32_t nxt = (i + 1) % c->num_ra;
    for (int32_t t = 0; t < cp[i]; ++t) {
      /* t-th CP bit of hc_i (from its MSB side): column bit position ep[i]+t from the MSB */
      uint32_t a = (cols[i] >> (c->cbn[i] - 1 - (uint32_t)(ep[i] + t))) & 1u;
      /* t-th bit of hc_{i+1} from its MSB */
      uint32_t b = (cols[nxt] >> (c->cbn[nxt] - 1 - (uint32_t)t)) & 1u;
      if (a != b) return 0;
    }
  }
  uint32_t lp = 0;
  for (uint32_t i = 0; i < c->num_ra; ++i) {
    for (int32_t t = 0; t < ep[i]; ++t) {
      uint32_t bit = (cols[i] >> (c->cbn[i] - 1 - (uint32_t)t)) & 1u;
      uint32_t pos = (c->clbs[i] + (uint32_t)t) % L;
      lp |= bit << (L - 1 - pos);
    }
  }
  *lp_out = lp;
  return 1;
}

/* Direction normalisation (a0, Q25).  Returns 1 and the ⟨inner, outer⟩
 * pair, or 0 if the pair has zero or two inner endpoints (skipped). */
static int is_inner(const orc_config* c, uint32_t ip) {
  for (uint32_t k = 0; k < c->n_prefix; ++k)
    if ((ip & c->prefix_mask[k]) == c->prefix[k]) return 1;
  return 0;
}

int orc_normalize(const orc_config* c, uint32_t src, uint32_t dst, uint32_t* iip, uint32_t* oip) {
  if (c->direction == 0) { *iip = src; *oip = dst; return 1; }
  int si = is_inner(c, src), di = is_inner(c, dst);
  if (si && !di) { *iip = src; *oip = dst; return 1; }
  if (di && !si) { *iip = dst; *oip = src; return 1; }
  return 0;
}

/* ------------------------------------------------------------- update */

/* Alg. 1 over a stream: for every pair set |RA|+|VA| bits,
 * bvIdx-th row of column CL(i) in every array of the selected CS.
 * Pin: single-pair vector (golden/single_pair.txt), idempotence, order
 * independence, exactly |RA|+|VA| bits, shard-OR invariant. */
void orc_update(const orc_config* c, uint8_t* cube, const uint32_t* src, const uint32_t* dst, uint64_t n,
                uint64_t* skipped) {
  uint32_t cols[ORC_MAX_ARR];
  uint64_t skip = 0;
  for (uint64_t k = 0; k < n; ++k) {
    uint32_t iip, oip, cs, row;
    if (!orc_normalize(c, src[k], dst[k], &iip, &oip)) { ++skip; continue; }
    orc_map_pair(c, iip, oip, &cs, cols, &row);
    for (uint32_t a = 0; a < c->num_ra + c->num_va; ++a) set_bit(cube, orc_bit_address(c, cs, a, cols[a], row));
  }
  if (skipped) *skipped = skip;
}

/* Global merge: bitwise OR of local CBAs ("merges these CBA by bits
 * OR", Q1).  Pin: shard-OR invariant, identity, idempotence. */
void orc_merge(uint8_t* dst, const uint8_t* src, uint64_t nbytes) {
  for (uint64_t k = 0; k < nbytes; ++k) dst[k] |= src[k];
}

/* ------------------------------------------------------------ estimator */

/* Zero bits of one column, counted bit by bit (Alg. 2).
 * Pin: Z + popcount = g, brute force. */
uint32_t orc_zero_count(const orc_config* c, const uint8_t* cube, uint32_t cs, uint32_t a, uint64_t col) {
  uint32_t z = 0;
  uint64_t base = orc_bit_address(c, cs, a, col, 0);   /* row 0 of the column */
  for (uint32_t row = 0; row < c->g; ++row) z += get_bit(cube, base + row) ? 0u : 1u;
  return z;
}

/* Eq. 1: −g·ln(z/g); z = 0 → +∞.  Pin: closed forms. */
double orc_linear_estimate(double g, double z) {
  if (z <= 0.0) return INFINITY;
  return -g * log(z / g);
}

/* Theorem 1 (sign per the statement, Q13): ε = ∏_{i<|RA|+|VA|}
 * (1 − e^{−η/(c(i)·g)}) over all arrays with their own c(i) (Q14).
 * Capped at 1 − 2^−20.  Pin: ε(0)=0, single array at η = c·g. */
double orc_shared_bit_prob(const orc_config* c, double eta) {
  double eps = 1.0;
  for (uint32_t i = 0; i < c->num_ra + c->num_va; ++i) eps *= 1.0 - exp(-eta / ((double)ncols(c, i) * (double)c->g));
  double cap = 1.0 - ldexp(1.0, -20);
  return eps > cap ? cap : eps;
}

/* Theorem 2: −g·ln(Z/(g − g·ε)); Z = 0 → +∞; negative → 0 (Q21).
 * Pin: ε = 0 reduces to Eq. 1 bit for bit; Z = g(1−ε) → 0. */
double orc_corrected_estimate(double z, double eps, double g) {
  if (z <= 0.0) return INFINITY;
  double v = -g * log(z / (g - g * eps));
  return v < 0.0 ? 0.0 : v;
}

/* θ_bn: g(1+ε)e^{−θ/g} − gε, or the inverted Theorem 2
 * g(1−ε)e^{−θ/g} (Q15), clamped at 0.  Pin: ε = 0 closed form table. */
double orc_hot_threshold(double theta, double eps, double g, int formula) {
  double v;
  if (formula == 0) v = g * (1.0 + eps) * exp(-theta / g) - g * eps;
  else v = g * (1.0 - eps) * exp(-theta / g);
  return v < 0.0 ? 0.0 : v;
}

/* Union-column threshold of Alg. 3 (Q20 option).  P:309 rejects a tuple whose
 * union column UC has more than θ_bn zero bits, reusing Alg. 2's per-column
 * threshold although UC's noise differs.  Theorem 1
 * gives UC's shared-bit probability ε and Theorem 2 its estimator
 * −g·ln(Z/(g(1−ε))); solving estimate ≥ θ for Z gives
 *   θ_uc = g·(1−ε)·e^{−θ/g},
 * so with this option Alg. 3 accepts exactly the candidates whose Theorem 2
 * estimate is ≥ θ (Def. 1).  Clamped at 0.  Pin: ε = 0 closed form
 * (= Eq. 1 inverted), the golden ε ≠ 0 values, the round trip through
 * orc_corrected_estimate, and "output = candidates with estimate ≥ θ". */
double orc_union_threshold(double theta, double eps, double g) {
  double v = g * (1.0 - eps) * exp(-theta / g);
  return v < 0.0 ? 0.0 : v;
}

/* η of a CS by whole-array linear counting over RA(0) (Q12):
 * η = −c(0)·g·ln(Ztot/(c(0)·g)); Ztot = 0 → η = +∞ (ε then hits its cap). */
void orc_cs_load(const orc_config* c, const uint8_t* cube, uint32_t cs, uint64_t* ztot_out, double* eta_out,
                 double* eps_out) {
  uint64_t ztot = 0;
  for (uint64_t col = 0; col < ncols(c, 0); ++col) ztot += orc_zero_count(c, cube, cs, 0, col);
  double bits = (double)ncols(c, 0) * (double)c->g;
  double eta = ztot == 0 ? INFINITY : -bits * log((double)ztot / bits);
  *ztot_out = ztot;
  *eta_out = eta;
  *eps_out = orc_shared_bit_prob(c, eta);
}

/* zmax = ⌊θ_bn⌋ clamped to [0, g]: "no more than θ_bn zero bits" (Q16). */
uint32_t orc_zmax(double theta_bn, uint32_t g) {
  double f = floor(theta_bn);
  if (f < 0.0) return 0;
  if (f > (double)g) return g;
  return (uint32_t)f;
}

/* Zero counts of every RA column of every CS, in the order
 * cs → RA(i) → column (the layout the tests compare against). */
void orc_zero_counts_ra(const orc_config* c, const uint8_t* cube, uint32_t* zc) {
  uint64_t k = 0;
  for (uint32_t cs = 0; cs < (1u << c->r); ++cs)
    for (uint32_t i = 0; i < c->num_ra; ++i)
      for (uint64_t col = 0; col < ncols(c, i); ++col) zc[k++] = orc_zero_count(c, cube, cs, i, col);
}

/* ------------------------------------------------------------ recovery */

/* Alg. 2: HC(i) = ascending columns j ∈ [0, c(i)−1] (Q17) of
 * RA(i) whose zero count is no more than θ_bn.  hc[i] must hold c(i)
 * entries.  Pin: per-column brute force; planted-host recovery. */
void orc_hot_columns(const orc_config* c, const uint8_t* cube, uint32_t cs, uint32_t zmax, uint32_t** hc,
                     uint32_t* n_hc) {
  for (uint32_t i = 0; i < c->num_ra; ++i) {
    n_hc[i] = 0;
    for (uint64_t j = 0; j < ncols(c, i); ++j)
      if (orc_zero_count(c, cube, cs, i, j) <= zmax) hc[i][n_hc[i]++] = (uint32_t)j;
  }
}

/* Alg. 3 second half: UCol = AND of the tuple's RA columns and
 * of VA(j) column H_j(LP); returns the zero bits of UCol, bit by bit. */
uint32_t orc_union_zeros(const orc_config* c, const uint8_t* cube, uint32_t cs, const uint32_t* ra_cols,
                         uint32_t lp) {
  uint64_t base[ORC_MAX_ARR];   /* row 0 of each of the |RA|+|VA| columns */
  for (uint32_t i = 0; i < c->num_ra; ++i) base[i] = orc_bit_address(c, cs, i, ra_cols[i], 0);
  for (uint32_t j = 0; j < c->num_va; ++j)
    base[c->num_ra + j] = orc_bit_address(c, cs, c->num_ra + j, orc_va_col(c, lp, j), 0);
  uint32_t z = 0;
  for (uint32_t row = 0; row < c->g; ++row) {
    int u = 1;
    for (uint32_t a = 0; a < c->num_ra + c->num_va; ++a) u &= get_bit(cube, base[a] + row);
    z += u ? 0u : 1u;
  }
  return z;
}

static int host_cmp(const void* pa, const void* pb) {
  const orc_host* a = (const orc_host*)pa;
  const orc_host* b = (const orc_host*)pb;
  if (a->estimate > b->estimate) return -1;   /* estimate descending */
  if (a->estimate < b->estimate) return 1;
  if (a->ip < b->ip) return -1;               /* then ip ascending            */
  if (a->ip > b->ip) return 1;
  return 0;
}

/* recoverAll: per CS, load → θ_bn → Alg. 2 → the full Cartesian
 * product of HC(0)×…×HC(|RA|−1) ("test them one by one") → Alg. 3
 * → ip = unmangle((lp << r) | cs) with its Thm. 2 estimate.
 * A CS whose ∏|HC(i)| exceeds tuple_cap is skipped and flagged.
 * Returns 0; 1 if any CS overflowed; 2 if more than cap hosts (out holds
 * the first cap after sorting, *n_out the full count). */
int orc_detect(const orc_config* c, const uint8_t* cube, double theta, orc_host* out, uint64_t cap,
               uint64_t* n_out, orc_cs_stats* stats) {
  uint64_t n_cs = (uint64_t)1 << c->r;
  uint64_t total = 0, alloc = 1024;
  orc_host* hosts = (orc_host*)malloc(alloc * sizeof(orc_host));
  uint32_t* hc[ORC_MAX_RA];
  uint32_t n_hc[ORC_MAX_RA];
  for (uint32_t i = 0; i < c->num_ra; ++i) hc[i] = (uint32_t*)malloc(ncols(c, i) * sizeof(uint32_t));
  int any_overflow = 0;
  for (uint32_t cs = 0; cs < n_cs; ++cs) {
    orc_cs_stats st;
    memset(&st, 0, sizeof st);
    orc_cs_load(c, cube, cs, &st.ztot, &st.eta, &st.eps);
    st.theta_bn = orc_hot_threshold(theta, st.eps, (double)c->g, c->theta_formula);
    st.zmax = orc_zmax(st.theta_bn, c->g);
    /* Alg. 3's threshold: the same θ_bn as written, or θ_uc (Q20) */
    st.theta_uc = c->union_threshold ? orc_union_threshold(theta, st.eps, (double)c->g) : st.theta_bn;
    st.zmax_uc = orc_zmax(st.theta_uc, c->g);
    orc_hot_columns(c, cube, cs, st.zmax, hc, n_hc);
    uint64_t prod = 1;
    for (uint32_t i = 0; i < c->num_ra; ++i) {
      st.n_hot[i] = n_hc[i];
      if (n_hc[i] != 0 && prod > UINT64_MAX / n_hc[i]) prod = UINT64_MAX;  /* saturate */
      else prod *= n_hc[i];
    }
    st.tuples = prod;
    if (prod > c->tuple_cap) {
      st.overflow = 1;
      any_overflow = 1;
    } else {
      /* odometer over the Cartesian product, last index fastest */
      uint32_t idx[ORC_MAX_RA];
      for (uint32_t i = 0; i < c->num_ra; ++i) idx[i] = 0;
      for (uint64_t t = 0; t < prod; ++t) {
        uint32_t cols[ORC_MAX_RA];
        for (uint32_t i = 0; i < c->num_ra; ++i) cols[i] = hc[i][idx[i]];
        uint32_t lp;
        if (orc_lp_from_tuple(c, cols, &lp)) {
          st.candidates++;
          uint32_t z = orc_union_zeros(c, cube, cs, cols, lp);
          if (z <= st.zmax_uc) {   /* P:309 reject iff zeros > θ_bn (Q16), or θ_uc (Q20) */
            st.hits++;
            if (total == alloc) { alloc *= 2; hosts = (orc_host*)realloc(hosts, alloc * sizeof(orc_host)); }
            uint32_t m = c->r == 0 ? lp : ((lp << c->r) | cs);
            hosts[total].ip = orc_unmangle(c, m);
            hosts[total].cs = cs;
            hosts[total].lp = lp;
            hosts[total].z = z;
            hosts[total].estimate = orc_corrected_estimate((double)z, st.eps, (double)c->g);
            total++;
          }
        }
        for (int i = (int)c->num_ra - 1; i >= 0; --i) {
          if (++idx[i] < n_hc[i]) break;
          idx[i] = 0;
        }
      }
    }
    if (stats) stats[cs] = st;
  }
  qsort(hosts, total, sizeof(orc_host), host_cmp);
  uint64_t ncopy = total < cap ? total : cap;
  if (out && ncopy) memcpy(out, hosts, ncopy * sizeof(orc_host));
  *n_out = total;
  free(hosts);
  for (uint32_t i = 0; i < c->num_ra; ++i) free(hc[i]);
  if (total > cap) return 2;
  return any_overflow ? 1 : 0;
}

/* Candidate LPs of one CS (tuples passing the CP check), in odometer order;
 * test hook for comparing candidate sets.  Returns the count (≤ cap written). */
uint64_t orc_candidates(const orc_config* c, const uint8_t* cube, uint32_t cs, uint32_t zmax, uint32_t* lps,
                        uint64_t cap) {
  uint32_t* hc[ORC_MAX_RA];
  uint32_t n_hc[ORC_MAX_RA];
  for (uint32_t i = 0; i < c->num_ra; ++i) hc[i] = (uint32_t*)malloc(ncols(c, i) * sizeof(uint32_t));
  orc_hot_columns(c, cube, cs, zmax, hc, n_hc);
  uint64_t prod = 1, count = 0;
  for (uint32_t i = 0; i < c->num_ra; ++i) prod *= n_hc[i];
  uint32_t idx[ORC_MAX_RA] = {0};
  for (uint64_t t = 0; t < prod && prod <= c->tuple_cap; ++t) {
    uint32_t cols[ORC_MAX_RA], lp;
    for (uint32_t i = 0; i < c->num_ra; ++i) cols[i] = hc[i][idx[i]];
    if (orc_lp_from_tuple(c, cols, &lp)) {
      if (count < cap) lps[count] = lp;
      count++;
    }
    for (int i = (int)c->num_ra - 1; i >= 0; --i) {
      if (++idx[i] < n_hc[i]) break;
      idx[i] = 0;
    }
  }
  for (uint32_t i = 0; i < c->num_ra; ++i) free(hc[i]);
  return count;
}

/* Pin loop (tests only): for every lp in [lo, hi) rebuild the RA tuple with
 * orc_ra_col and invert it with orc_lp_from_tuple (S:213 round trip).  With
 * flip_cp != 0 it instead flips the first CP bit of the tuple (when a CP bit
 * exists) and counts tuples that are NOT rejected.  Returns the
 * number of failures. */
uint64_t orc_lp_roundtrip_failures(const orc_config* c, uint64_t lo, uint64_t hi, int flip_cp) {
  int32_t ep[ORC_MAX_RA], cp[ORC_MAX_RA];
  orc_ep_cp(c, ep, cp);
  int first = -1;
  for (uint32_t i = 0; i < c->num_ra; ++i)
    if (cp[i] > 0) { first = (int)i; break; }
  uint64_t fails = 0;
  for (uint64_t v = lo; v < hi; ++v) {
    uint32_t lp = (uint32_t)v, cols[ORC_MAX_RA], back = 0;
    for (uint32_t i = 0; i < c->num_ra; ++i) cols[i] = orc_ra_col(c, lp, i);
    if (!flip_cp) {
      if (!orc_lp_from_tuple(c, cols, &back) || back != lp) ++fails;
    } else if (first >= 0) {
      cols[first] ^= 1u;   /* lowest column bit lies in CP(first) */
      if (orc_lp_from_tuple(c, cols, &back)) ++fails;
    }
  }
  return fails;
}

/* ------------------------------------------------- sparse SketchFile "CBA2"
 * The optional sparse/compressed form of the cross-router transfer (S:479
 * "optionally sparse").  This build's format:
 * the cube's bits are cut into blocks of 2^15 bits (4 KiB; bit 8j+k of the
 * cube = bit k of byte j); a block is the ascending list of its set-bit
 * positions p_0 < p_1 < …, written as the gaps p_0, p_1 − p_0 − 1, … in
 * LEB128 (7 bits per byte, low group first, bit 7 = "more").  Plain per-bit
 * loops: one call per block. */
#define ORC_SPARSE_BLOCK_BITS 32768u

static uint64_t orc_leb128_len(uint32_t v) {
  uint64_t n = 1;
  while (v >= 128) { v >>= 7; ++n; }
  return n;
}

/* Bytes of block b's varint stream (the last block may be short: nbits). */
uint64_t orc_sparse_block_bytes(const uint8_t* cube, uint64_t nbytes, uint64_t b) {
  uint64_t first = b * ORC_SPARSE_BLOCK_BITS, end = first + ORC_SPARSE_BLOCK_BITS, bytes = 0;
  if (end > nbytes * 8) end = nbytes * 8;
  int64_t prev = -1;
  for (uint64_t i = first; i < end; ++i) {
    if ((cube[i >> 3] >> (i & 7)) & 1u) {
      int64_t pos = (int64_t)(i - first);
      bytes += orc_leb128_len((uint32_t)(pos - prev - 1));
      prev = pos;
    }
  }
  return bytes;
}

/* Writes block b's varint stream to out; returns the bytes written. */
uint64_t orc_sparse_block_encode(const uint8_t* cube, uint64_t nbytes, uint64_t b, uint8_t* out) {
  uint64_t first = b * ORC_SPARSE_BLOCK_BITS, end = first + ORC_SPARSE_BLOCK_BITS, k = 0;
  if (end > nbytes * 8) end = nbytes * 8;
  int64_t prev = -1;
  for (uint64_t i = first; i < end; ++i) {
    if ((cube[i >> 3] >> (i & 7)) & 1u) {
      int64_t pos = (int64_t)(i - first);
      uint32_t gap = (uint32_t)(pos - prev - 1);
      while (gap >= 128) { out[k++] = (uint8_t)(0x80u | (gap & 0x7Fu)); gap >>= 7; }
      out[k++] = (uint8_t)gap;
      prev = pos;
    }
  }
  return k;
}

/* ORs block b's set bits, read from len bytes at in, into cube; returns 0, or 1 on a malformed
 * stream (a varint past the end, a position past the block). */
int orc_sparse_block_decode(const uint8_t* in, uint64_t len, uint8_t* cube, uint64_t nbytes, uint64_t b) {
  uint64_t first = b * ORC_SPARSE_BLOCK_BITS, k = 0;
  int64_t prev = -1;
  while (k < len) {
    uint64_t gap = 0;
    int shift = 0;
    for (;;) {
      if (k >= len || shift > 28) return 1;
      uint8_t byte = in[k++];
      gap |= (uint64_t)(byte & 0x7Fu) << shift;
      shift += 7;
      if (!(byte & 0x80u)) break;
    }
    int64_t pos = prev + 1 + (int64_t)gap;
    if (pos >= (int64_t)ORC_SPARSE_BLOCK_BITS || first + (uint64_t)pos >= nbytes * 8) return 1;
    cube[(first + pos) >> 3] |= (uint8_t)(1u << ((first + pos) & 7));
    prev = pos;
  }
  return 0;
}
