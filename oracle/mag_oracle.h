/* TEST INFRASTRUCTURE ONLY — CPU checker for the GPU search path.
 * See mag_oracle.c for what is restated and where it is pinned.          */
#ifndef MAG_ORACLE_H
#define MAG_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { MO_MAP_IDENTITY = 0, MO_MAP_FREQUENCY = 1, MO_MAP_BALANCED = 2, MO_MAP_LOWBITS = 3 };
enum { MO_VARIANT_MAG = 0, MO_VARIANT_SMAG = 1, MO_VARIANT_OG = 2 };
enum { MO_GRAM_EXACT = 0, MO_GRAM_HASHED = 1 };
enum { MO_WINDOW_REF = 0, MO_WINDOW_Q = 1 };
enum {
  MO_ERR_CONFIG = -2,
  MO_ERR_NOMEM = -3,
  MO_ERR_EMPTY_SET = -4,
  MO_ERR_EMPTY_PATTERN = -5
};

typedef struct mo_params {
  int variant;          /* MO_VARIANT_* */
  int gram_mode;        /* MO_GRAM_* */
  unsigned q, k;        /* k ignored (forced 1) for the overlapping variant */
  unsigned word_bits;   /* w; 0 = 64 */
  unsigned table_bits;  /* hashed: 2^table_bits mask entries */
  uint32_t sigma_prime; /* exact: map size */
  int window_rule;      /* MO_WINDOW_* */
  unsigned probes;      /* hashed, m' = k = 1: entries probed per gram (0/1 = one) */
  unsigned blocks;      /* probes >= 2: 64-entry blocks (table = 64 * blocks entries) */
  uint8_t map[256];     /* exact: byte -> code */
} mo_params;

typedef struct mo_shape {
  uint64_t entries;
  size_t L;
  unsigned k, m_prime;
  uint64_t match_mask, boundary_keep;
} mo_shape;

typedef struct mo_tuning_input {
  uint32_t sigma, sigma_prime;
  uint64_t r, m, n;
  uint32_t word_bits;
} mo_tuning_input;

typedef struct mo_tuning_result {
  int q, k, sigma_prime;
  double rho, predicted_p, predicted_cost;
} mo_tuning_result;

int mo_map_build(int strategy, const uint64_t counts[256], uint32_t sigma_prime,
                 unsigned lowbits, uint8_t table[256], uint32_t* sigma_out);
uint32_t mo_encode_gram(const uint8_t table[256], uint32_t sigma_prime, unsigned q,
                        const uint8_t* p);
void mo_encode_text(const uint8_t table[256], uint32_t sigma_prime, unsigned q,
                    const uint8_t* text, size_t n, uint32_t* out);
uint32_t mo_gram_hash(const uint8_t* p, unsigned q);
int mo_machine_shape(const mo_params* P, size_t m, mo_shape* S);
int mo_build_masks(const mo_params* P, const uint8_t* pat_bytes, const size_t* lens, size_t r,
                   const mo_shape* S, uint64_t* masks);
int mo_search(const uint8_t* text, size_t n, const uint8_t* pat_bytes, const size_t* lens,
              size_t r, const mo_params* P, uint64_t** offs, uint32_t** pids, size_t* count,
              uint64_t* reads, uint64_t* cands);
int mo_naive_search(const uint8_t* text, size_t n, const uint8_t* pat_bytes, const size_t* lens,
                    size_t r, uint64_t** offs, uint32_t** pids, size_t* count);
void mo_free(void* p);

double mo_expected_class_size(double sigma_eff, double n_super);
double mo_match_probability(double sigma_eff, double n_super);
uint32_t mo_resolve_sigma_prime(uint32_t sigma_observed, uint32_t user_choice);
unsigned mo_max_feasible_q(const mo_tuning_input* ti);
unsigned mo_choose_q(const mo_tuning_input* ti);
double mo_strided_k_seed(const mo_tuning_input* ti, unsigned q);
unsigned mo_choose_k(const mo_tuning_input* ti, unsigned q);
double mo_predicted_cost(const mo_tuning_input* ti, unsigned q, unsigned k);
int mo_tune(const mo_tuning_input* in, int fixed_q, int fixed_k, mo_tuning_result* out);
int mo_sample_offsets(size_t corpus_len, size_t count, size_t length, uint64_t seed,
                      uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif
