/*
 * TEST INFRASTRUCTURE ONLY — the CPU checker.  Never linked into or called by
 * the product (paper_1405_5483_b200/libmag_b200.so); only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline/reference arm load it.
 *
 * Plain-C restatement of the reference's search phase for the pieces whose
 * bodies the reference does NOT ship: the FilterMachine
 * constructor, the verifier, the engine's strided/overlapping search and the
 * tuner.  Everything that DOES ship (naive/AC oracles, maps, encode_text,
 * superimposition) is pinned against the compiled reference in
 * oracle/_ref/libmagref.so by tests/test_oracle.py, and the result set of
 * mo_search() is pinned against the reference's own naive_search/ac_search
 * (result sets are parameter-invariant).
 *
 * Citations are /root/reference/ paths.
 */
#include "mag_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- maps --
 * alphabet_map.cpp:42-50  by_count_desc: stable sort, descending count,
 *                          ties by ascending byte.
 * alphabet_map.cpp:54-66  greedy LPT: item into the lightest bin, ties to
 *                          the lowest bin index.
 * alphabet_map.cpp:70-114 identity / frequency / balanced / lowbits.      */
static void order_by_count(const uint64_t counts[256], int order[256]) {
  for (int i = 0; i < 256; ++i) order[i] = i;
  /* insertion sort is stable and 256 items is nothing */
  for (int i = 1; i < 256; ++i) {
    int v = order[i], j = i - 1;
    while (j >= 0 && counts[order[j]] < counts[v]) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = v;
  }
}

int mo_map_build(int strategy, const uint64_t counts[256], uint32_t sigma_prime,
                 unsigned lowbits, uint8_t table[256], uint32_t* sigma_out) {
  int order[256];
  switch (strategy) {
    case MO_MAP_IDENTITY:
      for (int c = 0; c < 256; ++c) table[c] = (uint8_t)c;
      *sigma_out = 256;
      return 0;
    case MO_MAP_FREQUENCY:
      if (sigma_prime < 2 || sigma_prime > 256) return MO_ERR_CONFIG;
      order_by_count(counts, order);
      for (uint32_t rank = 0; rank < 256; ++rank)
        table[order[rank]] = (uint8_t)(rank < sigma_prime - 1 ? rank : sigma_prime - 1);
      *sigma_out = sigma_prime;
      return 0;
    case MO_MAP_BALANCED: {
      if (sigma_prime < 2 || sigma_prime > 256) return MO_ERR_CONFIG;
      order_by_count(counts, order);
      uint64_t load[256] = {0};
      for (int i = 0; i < 256; ++i) {
        uint32_t best = 0;
        for (uint32_t b = 1; b < sigma_prime; ++b)
          if (load[b] < load[best]) best = b;
        table[order[i]] = (uint8_t)best;
        load[best] += counts[order[i]];
      }
      *sigma_out = sigma_prime;
      return 0;
    }
    case MO_MAP_LOWBITS:
      if (lowbits < 1 || lowbits > 8) return MO_ERR_CONFIG;
      for (unsigned c = 0; c < 256; ++c) table[c] = (uint8_t)(c & ((1u << lowbits) - 1));
      *sigma_out = 1u << lowbits;
      return 0;
  }
  return MO_ERR_CONFIG;
}

/* ------------------------------------------------------------- q-grams --
 * qgram.hpp:30-36  little-endian Horner: sum map(p[i]) * sigma'^i.
 * qgram.cpp:9-19   1 <= q <= 8, sigma'^q <= 2^24.                         */
uint32_t mo_encode_gram(const uint8_t table[256], uint32_t sigma_prime, unsigned q,
                        const uint8_t* p) {
  uint32_t code = table[p[q - 1]];
  for (unsigned i = q - 1; i-- > 0;) code = code * sigma_prime + table[p[i]];
  return code;
}

void mo_encode_text(const uint8_t table[256], uint32_t sigma_prime, unsigned q,
                    const uint8_t* text, size_t n, uint32_t* out) {
  size_t nq = n / q;
  for (size_t u = 0; u < nq; ++u) out[u] = mo_encode_gram(table, sigma_prime, q, text + u * q);
}

/* Hashed q-gram alphabet (the paper's §3.3 q-gram-alphabet mapping by
 * hashing; GPU extension, documented in DESIGN.md):
 * the q raw bytes (q <= 16) are read as four little-endian words (bytes past
 * q are zero) and mixed; the top `bits` bits index the mask table.  Must stay
 * bit-identical to hash_gram() in paper_1405_5483_b200/csrc/mag_common.h.  */
uint32_t mo_gram_hash(const uint8_t* p, unsigned q) {
  uint32_t x[4] = {0, 0, 0, 0};
  for (unsigned i = 0; i < q; ++i) x[i >> 2] |= (uint32_t)p[i] << (8 * (i & 3));
  uint32_t h = x[0] * 0x9E3779B1u + x[1] * 0x85EBCA77u + x[2] * 0xC2B2AE3Du +
               x[3] * 0x27D4EB2Fu;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  return h;
}

/* Multi-probe hashed grams (GPU extension; paper_1405_5483_b200/csrc/
 * mag_common.h bloom_block/bloom_bit): `probes` entries of one 64-entry
 * block, admitted only where all of them are admitted. */
static inline uint32_t probe_entry(const mo_params* P, uint32_t h, unsigned i) {
  uint32_t blk = (uint32_t)(((uint64_t)h * P->blocks) >> 32);
  uint64_t g = (uint64_t)h * 0x9E3779B97F4A7C15ull;
  uint32_t bit = (uint32_t)(g >> (58 - 6 * i)) & 63u;
  return blk * 64u + bit;
}

static inline int multi_probe(const mo_params* P) {
  return P->gram_mode == MO_GRAM_HASHED && P->probes > 1;
}

static inline uint32_t gram_index(const mo_params* P, const uint8_t* g) {
  if (P->gram_mode == MO_GRAM_EXACT) return mo_encode_gram(P->map, P->sigma_prime, P->q, g);
  if (P->table_bits == 0) return 0;
  return mo_gram_hash(g, P->q) >> (32 - P->table_bits);
}

/* ------------------------------------------------------------ machine --
 * filter.hpp:27-31  k Shift-Or automata in one word; alignment j holds class
 *                   positions j, j+k, j+2k, ... (SPEC.md:306 P^j[i]=P[j+ik])
 *                   truncated to m' = min(floor(L/k), floor(w/k)); bit
 *                   j*m'+i of a mask is 0 iff the code is admitted there.
 * superimpose.hpp:33-47 admissions: strided = all q shifts x L_q grams of
 *                   the first m bytes; overlapping = m-q+1 grams.
 * superimpose.cpp:11-21 L_q = floor((m-q+1)/q) needs m >= 2q-1; L = m-q+1
 *                   needs m >= q.                                          */
int mo_machine_shape(const mo_params* P, size_t m, mo_shape* S) {
  unsigned q = P->q;
  int og = P->variant == MO_VARIANT_OG;
  if (q < 1) return MO_ERR_CONFIG;
  if (P->gram_mode == MO_GRAM_EXACT) {
    if (q > 8) return MO_ERR_CONFIG;
    uint64_t space = 1;
    for (unsigned i = 0; i < q; ++i) {
      space *= P->sigma_prime;
      if (space > (1u << 24)) return MO_ERR_CONFIG;
    }
    S->entries = space;
  } else {
    if (q > 16 || P->table_bits > 26) return MO_ERR_CONFIG;
    S->entries = P->probes > 1 ? (uint64_t)P->blocks * 64 : (uint64_t)1 << P->table_bits;
  }
  if (og) {
    if (m < q) return MO_ERR_CONFIG;
    S->L = m - q + 1;
    S->k = 1;
  } else {
    if (m < 2 * (size_t)q - 1) return MO_ERR_CONFIG;
    S->L = (m - q + 1) / q;
    S->k = P->k;
  }
  unsigned w = P->word_bits ? P->word_bits : 64;
  if (w > 64) w = 64;
  if (S->k < 1 || S->k > S->L || S->k > w) return MO_ERR_CONFIG;
  size_t mp = S->L / S->k;
  if (mp > w / S->k) mp = w / S->k;
  S->m_prime = (unsigned)mp;
  if (multi_probe(P) && (S->m_prime != 1 || S->k != 1 || P->blocks < 1 || P->probes > 8))
    return MO_ERR_CONFIG;
  S->match_mask = 0;
  S->boundary_keep = ~0ull;
  for (unsigned j = 0; j < S->k; ++j) {
    S->match_mask |= 1ull << (j * S->m_prime + S->m_prime - 1);
    S->boundary_keep &= ~(1ull << (j * S->m_prime));
  }
  return 0;
}

int mo_build_masks(const mo_params* P, const uint8_t* pat_bytes, const size_t* lens, size_t r,
                   const mo_shape* S, uint64_t* masks) {
  unsigned q = P->q;
  int og = P->variant == MO_VARIANT_OG;
  for (uint64_t e = 0; e < S->entries; ++e) masks[e] = ~0ull;
  size_t off = 0;
  for (size_t i = 0; i < r; ++i) {
    const uint8_t* p = pat_bytes + off;
    off += lens[i];
    unsigned shifts = og ? 1 : q;
    for (unsigned s = 0; s < shifts; ++s) {
      for (size_t j = 0; j < S->L; ++j) {
        const uint8_t* g = og ? p + j : p + s + j * q;
        size_t align = j % S->k, pos = j / S->k;
        if (pos >= S->m_prime) continue;
        if (multi_probe(P)) {
          uint32_t h = mo_gram_hash(g, q);
          for (unsigned i = 0; i < P->probes; ++i) masks[probe_entry(P, h, i)] &= ~1ull;
          continue;
        }
        masks[gram_index(P, g)] &= ~(1ull << (align * S->m_prime + pos));
      }
    }
  }
  return 0;
}

/* ------------------------------------------------------------- search --*/
typedef struct {
  uint64_t* off;
  uint32_t* pid;
  size_t n, cap;
} occ_vec;

static int occ_push(occ_vec* v, uint64_t off, uint32_t pid) {
  if (v->n == v->cap) {
    size_t nc = v->cap ? v->cap * 2 : 256;
    uint64_t* o = (uint64_t*)realloc(v->off, nc * 8);
    if (!o) return -1;
    v->off = o;
    uint32_t* p = (uint32_t*)realloc(v->pid, nc * 4);
    if (!p) return -1;
    v->pid = p;
    v->cap = nc;
  }
  v->off[v->n] = off;
  v->pid[v->n] = pid;
  v->n++;
  return 0;
}

/* verify.hpp:28-31 / SPEC.md:376-380: every pattern at every start of the
 * window; a match needs a + len <= n and byte equality.  `bucket` is an
 * optional speed index (patterns grouped by their first byte) — it only
 * skips patterns whose first byte differs, so the set compared is the same. */
typedef struct {
  const uint8_t* bytes;
  const size_t* lens;
  const size_t* offs;
  size_t r;
  uint32_t* by_first; /* pattern ids sorted by first byte */
  size_t first_lo[257];
} pat_index;

static int verify_start(const pat_index* I, const uint8_t* text, size_t n, size_t a,
                        occ_vec* out) {
  uint8_t c = text[a];
  for (size_t x = I->first_lo[c]; x < I->first_lo[c + 1]; ++x) {
    uint32_t i = I->by_first[x];
    size_t len = I->lens[i];
    if (a + len <= n && memcmp(text + a, I->bytes + I->offs[i], len) == 0)
      if (occ_push(out, a, i)) return -1;
  }
  return 0;
}

static int cmp_occ(const void* A, const void* B) {
  const uint64_t* a = (const uint64_t*)A;
  const uint64_t* b = (const uint64_t*)B;
  if (a[0] != b[0]) return a[0] < b[0] ? -1 : 1;
  if (a[1] != b[1]) return a[1] < b[1] ? -1 : 1;
  return 0;
}

/* verify.hpp:37-38 sort_dedup: sort by (offset, pattern_index), drop dups. */
static int sort_dedup(occ_vec* v) {
  if (v->n < 2) return 0;
  uint64_t* tmp = (uint64_t*)malloc(v->n * 16);
  if (!tmp) return -1;
  for (size_t i = 0; i < v->n; ++i) {
    tmp[2 * i] = v->off[i];
    tmp[2 * i + 1] = v->pid[i];
  }
  qsort(tmp, v->n, 16, cmp_occ);
  size_t w = 0;
  for (size_t i = 0; i < v->n; ++i) {
    if (w && tmp[2 * i] == v->off[w - 1] && tmp[2 * i + 1] == v->pid[w - 1]) continue;
    v->off[w] = tmp[2 * i];
    v->pid[w] = (uint32_t)tmp[2 * i + 1];
    ++w;
  }
  v->n = w;
  free(tmp);
  return 0;
}

int mo_search(const uint8_t* text, size_t n, const uint8_t* pat_bytes, const size_t* lens,
              size_t r, const mo_params* P, uint64_t** offs_out, uint32_t** pids_out,
              size_t* count, uint64_t* reads_out, uint64_t* cands_out) {
  if (r == 0) return MO_ERR_EMPTY_SET;
  size_t m = lens[0];
  for (size_t i = 0; i < r; ++i) {
    if (lens[i] == 0) return MO_ERR_EMPTY_PATTERN;
    if (lens[i] < m) m = lens[i];
  }
  mo_shape S;
  int rc = mo_machine_shape(P, m, &S);
  if (rc) return rc;
  uint64_t* masks = (uint64_t*)malloc(S.entries * 8);
  size_t* poffs = (size_t*)malloc(r * sizeof(size_t));
  pat_index I;
  I.by_first = (uint32_t*)malloc(r * 4);
  if (!masks || !poffs || !I.by_first) return MO_ERR_NOMEM;
  mo_build_masks(P, pat_bytes, lens, r, &S, masks);
  size_t o = 0;
  size_t cnt[257] = {0};
  for (size_t i = 0; i < r; ++i) {
    poffs[i] = o;
    cnt[pat_bytes[o] + 1]++;
    o += lens[i];
  }
  for (int c = 0; c < 256; ++c) cnt[c + 1] += cnt[c];
  memcpy(I.first_lo, cnt, sizeof(cnt));
  for (size_t i = 0; i < r; ++i) I.by_first[cnt[pat_bytes[poffs[i]]]++] = (uint32_t)i;
  I.bytes = pat_bytes;
  I.lens = lens;
  I.offs = poffs;
  I.r = r;

  const unsigned q = P->q, k = S.k, mp = S.m_prime;
  const int og = P->variant == MO_VARIANT_OG;
  /* read budget: floor(floor(n/q)/k) strided (filter.hpp:44-45), n-q+1
   * overlapping grams (k forced to 1) */
  uint64_t T = og ? (n >= q ? n - q + 1 : 0) : (n / q) / k;
  uint64_t reads = 0, cands = 0;
  occ_vec out = {0, 0, 0, 0};
  uint64_t d = ~0ull;
  /* filter.hpp:58-73: d = ((d << 1) & boundary_keep) | masks[code(u)];
   * every 0 bit of d under match_mask is a Candidate with super_start
   * u - j - (m'-1)k. */
  for (uint64_t t = 0; t < T; ++t) {
    uint64_t u = og ? t : (t + 1) * k - 1;
    const uint8_t* g = text + (og ? u : u * q);
    ++reads;
    uint64_t mv;
    if (multi_probe(P)) {
      uint32_t h = mo_gram_hash(g, q);
      mv = 0;
      for (unsigned i = 0; i < P->probes; ++i) mv |= masks[probe_entry(P, h, i)] & 1ull;
      mv |= ~1ull;
    } else {
      mv = masks[gram_index(P, g)];
    }
    d = ((d << 1) & S.boundary_keep) | mv;
    if ((d & S.match_mask) == S.match_mask) continue;
    uint64_t hits = ~d & S.match_mask;
    while (hits) {
      unsigned bit = (unsigned)__builtin_ctzll(hits);
      hits &= hits - 1;
      unsigned j = bit / mp;
      ++cands;
      uint64_t ss = u - j - (uint64_t)(mp - 1) * k;
      /* windows: og_candidate_window verify.hpp:25-26 pins the start;
       * candidate_window verify.hpp:21-23 / SPEC.md:371 spans
       * [q*ss-(q-1), q*ss+(q-1)] clipped to [0, n-m]; MO_WINDOW_Q narrows it
       * to the q starts [q*ss-(q-1), q*ss] that can hold an occurrence. */
      if (n < m) continue;
      int64_t lo, hi, last = (int64_t)(n - m);
      if (og) {
        lo = (int64_t)ss;
        hi = (int64_t)ss;
      } else {
        lo = (int64_t)(q * ss) - (int64_t)(q - 1);
        hi = (int64_t)(q * ss) + (P->window_rule == MO_WINDOW_Q ? 0 : (int64_t)(q - 1));
      }
      if (lo < 0) lo = 0;
      if (hi > last) hi = last;
      for (int64_t a = lo; a <= hi; ++a)
        if (verify_start(&I, text, n, (size_t)a, &out)) return MO_ERR_NOMEM;
    }
  }
  free(masks);
  free(poffs);
  free(I.by_first);
  if (sort_dedup(&out)) return MO_ERR_NOMEM;
  if (!out.off) {
    out.off = (uint64_t*)malloc(8);
    out.pid = (uint32_t*)malloc(4);
  }
  *offs_out = out.off;
  *pids_out = out.pid;
  *count = out.n;
  if (reads_out) *reads_out = reads;
  if (cands_out) *cands_out = cands;
  return 0;
}

/* naive_search restated (oracles.cpp:9-21), for the CPU suite when the
 * compiled reference is absent. */
int mo_naive_search(const uint8_t* text, size_t n, const uint8_t* pat_bytes, const size_t* lens,
                    size_t r, uint64_t** offs_out, uint32_t** pids_out, size_t* count) {
  occ_vec out = {0, 0, 0, 0};
  size_t m = r ? lens[0] : 0;
  for (size_t i = 0; i < r; ++i)
    if (lens[i] < m) m = lens[i];
  size_t* po = (size_t*)malloc((r ? r : 1) * sizeof(size_t));
  size_t o = 0;
  for (size_t i = 0; i < r; ++i) {
    po[i] = o;
    o += lens[i];
  }
  if (n >= m) {
    for (size_t a = 0; a + m <= n; ++a)
      for (size_t i = 0; i < r; ++i)
        if (a + lens[i] <= n && memcmp(text + a, pat_bytes + po[i], lens[i]) == 0)
          occ_push(&out, a, (uint32_t)i);
  }
  free(po);
  if (!out.off) {
    out.off = (uint64_t*)malloc(8);
    out.pid = (uint32_t*)malloc(4);
  }
  *offs_out = out.off;
  *pids_out = out.pid;
  *count = out.n;
  return 0;
}

void mo_free(void* p) { free(p); }

/* -------------------------------------------------------------- tuner --
 * Restated from tuner.hpp:8-66 and SPEC.md:427-492 (no body ships).     */
double mo_expected_class_size(double sigma_eff, double n_super) {
  if (sigma_eff <= 0) return 0;
  return sigma_eff * (1.0 - pow(1.0 - 1.0 / sigma_eff, n_super));
}

double mo_match_probability(double sigma_eff, double n_super) {
  if (sigma_eff <= 0) return 1;
  return 1.0 - pow(1.0 - 1.0 / sigma_eff, n_super);
}

/* tuner.hpp:38-40: user override wins; observed sigma when <= 64; else 256.
 * sigma' >= 2 is required by the maps (alphabet_map.cpp:37-40). */
uint32_t mo_resolve_sigma_prime(uint32_t sigma_observed, uint32_t user_choice) {
  if (user_choice) return user_choice;
  if (sigma_observed <= 64) return sigma_observed < 2 ? 2 : sigma_observed;
  return 256;
}

static double log_base(double x, double b) { return log(x) / log(b); }

static int q_feasible(uint32_t sp, uint64_t m, unsigned q) {
  if (q < 1 || q > 8) return 0;
  if (m < 2ull * q - 1) return 0;
  double space = pow((double)sp, (double)q);
  return space <= (double)(1u << 24);
}

unsigned mo_max_feasible_q(const mo_tuning_input* ti) {
  for (unsigned q = 8; q >= 1; --q)
    if (q_feasible(ti->sigma_prime, ti->m, q)) return q;
  return 1;
}

unsigned mo_choose_q(const mo_tuning_input* ti) {
  double rm = (double)ti->r * (double)ti->m;
  double lq = rm > 1 ? log_base(rm, ti->sigma_prime) : 0;
  long q = lround(lq);
  if (q < 1) q = 1;
  if (q > 8) q = 8;
  while (q > 1 && !q_feasible(ti->sigma_prime, ti->m, (unsigned)q)) --q;
  return (unsigned)q;
}

double mo_strided_k_seed(const mo_tuning_input* ti, unsigned q) {
  (void)q;
  double rm = (double)ti->r * (double)ti->m;
  double L = log_base(rm, ti->sigma_prime);
  if (L <= 0) return 1;
  double rho = L / (double)ti->m;
  double l = log_base(1.0 / rho, ti->sigma_prime);
  if (L + l <= 0) return 1;
  return (double)ti->m / L * l / (L + l);
}

static unsigned alignment_len(const mo_tuning_input* ti, unsigned q, unsigned k) {
  uint64_t Lq = (ti->m - q + 1) / q;
  unsigned w = ti->word_bits ? ti->word_bits : 64;
  uint64_t mp = Lq / k;
  if (mp > w / k) mp = w / k;
  return (unsigned)mp;
}

double mo_predicted_cost(const mo_tuning_input* ti, unsigned q, unsigned k) {
  double nq = (double)(ti->n / q);
  double p = mo_match_probability(pow((double)ti->sigma_prime, (double)q), (double)q * ti->r);
  unsigned mp = alignment_len(ti, q, k);
  return nq / k + nq * pow(p, (double)mp) * (2.0 * q - 1) * (double)ti->r * (double)ti->m;
}

unsigned mo_choose_k(const mo_tuning_input* ti, unsigned q) {
  uint64_t Lq = (ti->m - q + 1) / q;
  if (Lq < 1) Lq = 1;
  unsigned w = ti->word_bits ? ti->word_bits : 64;
  long k0 = lround(mo_strided_k_seed(ti, q));
  if (k0 < 1) k0 = 1;
  if ((uint64_t)k0 > Lq) k0 = (long)Lq;
  long lo = k0 - 2 < 1 ? 1 : k0 - 2;
  long hi = (uint64_t)(k0 + 2) > Lq ? (long)Lq : k0 + 2;
  unsigned best = (unsigned)k0;
  double bc = INFINITY;
  for (long k = lo; k <= hi; ++k) {
    if ((unsigned)k > w) continue;
    double c = mo_predicted_cost(ti, q, (unsigned)k);
    if (c < bc) {
      bc = c;
      best = (unsigned)k;
    }
  }
  return best;
}

int mo_tune(const mo_tuning_input* in, int fixed_q, int fixed_k, mo_tuning_result* out) {
  mo_tuning_input ti = *in;
  if (ti.r < 1 || ti.m < 1 || ti.sigma < 1) return MO_ERR_CONFIG;
  if (!ti.word_bits) ti.word_bits = 64;
  ti.sigma_prime = mo_resolve_sigma_prime(ti.sigma, ti.sigma_prime);
  if (ti.sigma_prime < 2 || ti.sigma_prime > 256) return MO_ERR_CONFIG;
  unsigned q0 = fixed_q > 0 ? (unsigned)fixed_q : mo_choose_q(&ti);
  if (!q_feasible(ti.sigma_prime, ti.m, q0)) return MO_ERR_CONFIG;
  unsigned qlo = q0, qhi = q0;
  if (fixed_q <= 0) {
    qlo = q0 > 2 ? q0 - 2 : 1;
    qhi = q0 + 2;
  }
  unsigned bq = q0, bk = 1;
  double bc = INFINITY;
  for (unsigned q = qlo; q <= qhi; ++q) {
    if (!q_feasible(ti.sigma_prime, ti.m, q)) continue;
    unsigned k;
    if (fixed_k > 0) {
      uint64_t Lq = (ti.m - q + 1) / q;
      if ((uint64_t)fixed_k > Lq || (unsigned)fixed_k > ti.word_bits) continue;
      k = (unsigned)fixed_k;
    } else {
      k = mo_choose_k(&ti, q);
    }
    double c = mo_predicted_cost(&ti, q, k);
    if (c < bc) {
      bc = c;
      bq = q;
      bk = k;
    }
  }
  if (bc == INFINITY) return MO_ERR_CONFIG;
  double rm = (double)ti.r * (double)ti.m;
  out->q = bq;
  out->k = bk;
  out->sigma_prime = ti.sigma_prime;
  out->rho = (rm > 1 ? log_base(rm, ti.sigma_prime) : 0) / (double)ti.m;
  out->predicted_p = mo_match_probability(pow((double)ti.sigma_prime, (double)bq), (double)bq * ti.r);
  out->predicted_cost = bc;
  return 0;
}

/* ------------------------------------------------------------ sampling --
 * sampling.hpp:10-14 (no body ships): seeded uniform offsets in [0, n-m].
 * Generator: splitmix64, offset = next() % (n-m+1).  Must match
 * paper_1405_5483_b200/csrc/host_engine.cpp sample_offsets().             */
static uint64_t splitmix64(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int mo_sample_offsets(size_t corpus_len, size_t count, size_t length, uint64_t seed,
                      uint64_t* out) {
  if (length == 0 || length > corpus_len) return MO_ERR_CONFIG;
  uint64_t s = seed;
  uint64_t span = corpus_len - length + 1;
  for (size_t i = 0; i < count; ++i) out[i] = splitmix64(&s) % span;
  return 0;
}
