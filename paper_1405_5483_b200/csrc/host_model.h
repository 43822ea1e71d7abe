// Host-side model of the search: pattern set, alphabet maps, the
// reference's tuner, the GPU planner and the table builders.  No CUDA here;
// everything is deterministic host code that runs at engine creation.
#pragma once

#include <stddef.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "mag_common.h"

namespace magb {

// core.hpp:44-62 PatternSet: input order kept, duplicates kept, m = min length.
struct PatternData {
  std::vector<uint8_t> bytes;     // each pattern at a 16-byte aligned offset, zero padded
  std::vector<uint64_t> off;
  std::vector<uint32_t> len;
  size_t r = 0, m = 0, maxlen = 0;
  const uint8_t* pattern(size_t i) const { return bytes.data() + off[i]; }
};

// alphabet_map.hpp:19-26 Histogram.
struct Histogram {
  uint64_t counts[256] = {0};
  uint64_t total = 0;
  void add(const uint8_t* p, size_t n) {
    for (size_t i = 0; i < n; ++i) ++counts[p[i]];
    total += n;
  }
  uint32_t distinct() const {
    uint32_t d = 0;
    for (int i = 0; i < 256; ++i) d += counts[i] > 0;
    return d;
  }
};

enum MapStrategy : int { kMapIdentity = 0, kMapFrequency = 1, kMapBalanced = 2, kMapLowbits = 3 };

// alphabet_map.cpp:70-114.  Returns false (config error) on a bad sigma' or ell.
bool build_map(int strategy, const Histogram& h, uint32_t sigma_prime, unsigned lowbits,
               uint8_t table[256], uint32_t* sigma_out, std::string* err);

// ---- tuner (tuner.hpp:8-66, restated: the reference ships no body)
struct TuningInput {
  uint32_t sigma = 256, sigma_prime = 0;
  uint64_t r = 1, m = 1, n = 1u << 20;
  unsigned word_bits = 64;
};
struct TuningResult {
  unsigned q = 1, k = 1;
  uint32_t sigma_prime = 256;
  double rho = 0, predicted_p = 0, predicted_cost = 0;
};
double expected_class_size(double sigma_eff, double n_super);
double match_probability(double sigma_eff, double n_super);
uint32_t resolve_sigma_prime(uint32_t sigma_observed, uint32_t user_choice);
unsigned choose_q(const TuningInput& ti);
double strided_k_seed(const TuningInput& ti, unsigned q);
unsigned choose_k(const TuningInput& ti, unsigned q);
double predicted_cost(const TuningInput& ti, unsigned q, unsigned k);
bool tune(const TuningInput& ti, int fixed_q, int fixed_k, TuningResult* out, std::string* err);

// ---- plan
struct PlanRequest {
  int variant = 0;           // mag_variant
  int mapping = -1;          // mag_mapping
  int lowbits = 0;
  int q = 0, k = 0, sigma_prime = 0;
  int gram_mode = -1;        // mag_gram_mode
  int table_bits = 0;        // hashed: 0 auto, -1 verify-all
  int word_bits = 0;
  int tile_bytes = 0, warps = 0, stages = 0;  // tile_bytes: chunk bytes target; stages: ring
  int probes = 0;            // hashed: 0 auto
  int kernel = 0;            // mag_scan_kernel: 0 auto, 1 staged, 2 direct, 3 roll
  int cluster = 0;           // direct: 0 auto, 1 never, 8 force the cluster-shared table
  size_t smem_limit = 232448;  // sm_100 max dynamic shared memory per CTA
};

struct Plan {
  ScanPlan sp{};
  int variant = 0;
  int mapping = 0;           // mag_mapping in effect
  uint8_t map[256] = {0};
  // kernel geometry (scan_launch.h ScanArgs)
  uint32_t chunk_target = 0;   // planner's chunk size (gram bytes), 0 = default
  uint32_t chunk_samples = 0;  // samples per ring slot
  uint64_t slice_samples = 0;  // samples per warp work item
  uint32_t back = 0;           // staged bytes after a chunk's last gram
  uint32_t full_bytes = 0;     // staged bytes of an interior chunk
  uint32_t slot_bytes = 0;
  uint32_t ring = 0, nwarps = 0;
  double pred_cand_per_byte = 0;
  // planner's cost (thread-instructions per text byte) and its derivative in
  // the candidate rate: a measured rate re-prices the plan as
  // pred_cost + cost_slope * (measured - predicted)
  double pred_cost = 0, cost_slope = 0;
  // survivors: candidates whose verification key is a pattern's (true gram
  // matches of repetitive text); direct plans price them separately.  Each
  // survivor walks every table entry sharing its key, one dependent L2 round
  // trip per entry in a single lane: repetitive text whose grams occur in
  // hundreds of patterns (SURVEY.md §7 hard part 2)
  double pred_surv_per_byte = 0, surv_slope = 0, meas_surv_per_byte = -1;
  double meas_walk_per_byte = -1;
  // measured on a text sample (mag_options.histogram_sample): -1 = no sample
  double meas_cand_per_byte = -1, meas_cost = 0;
  uint64_t meas_sample_bytes = 0;
  uint32_t meas_plans = 0;  // finalist plans whose filters ran over the sample
};

size_t plan_smem(const Plan& p);

// Errors: returns a mag_status value (0 ok) and fills *err.
int make_plan(const PatternData& pd, const Histogram& h, const PlanRequest& rq, Plan* plan,
              std::string* err);

// GPU-aware parameter choice with measured candidate rates (
// replaces the uniform-text estimate of tuner.hpp:58-66 where a text sample
// is given): make_plan, then the analytic best plan of every kernel family
// has its real filter table built and run over `sample`; the measured
// candidates per byte re-price each plan and the cheapest one is returned.
// Plans the caller pinned (reference parameters, a forced kernel) are
// measured but not replaced.
int make_plan_measured(const PatternData& pd, const Histogram& h, const PlanRequest& rq,
                       const uint8_t* sample, size_t sample_len, Plan* plan, std::string* err);

// The plan's own filter and verification keys over text[0, n), per text
// byte: candidates as the kernels count mag_metrics.candidates; survivors =
// candidates whose verification key is a pattern's; walked = the table entries
// those survivors visit (all entries sharing the key).
struct FilterRates {
  double candidates = 0, survivors = 0, walked = 0;
};
FilterRates measure_filter(const Plan& plan, const PatternData& pd, const std::vector<uint8_t>& table,
                           const uint8_t* text, size_t n);

// Packed mask table (bit j*m'+i of entry c is 0 iff c admitted at alignment
// j position i; filter.hpp:27-31), table_bytes long.
void build_masks(const Plan& plan, const PatternData& pd, std::vector<uint8_t>* table);
uint64_t mask_entry(const Plan& plan, const std::vector<uint8_t>& table, uint64_t idx);

// Verification tables: prefilter bitmap, buckets, entries {key, pid}.
struct PatternTable {
  std::vector<uint32_t> prefilter;
  std::vector<uint32_t> l2map;
  std::vector<uint32_t> bucket_start;
  std::vector<uint32_t> entries;  // interleaved key, pid
  // roll plans: open-addressing verification table, 8 words per slot
  // {len | F << 31, pid (0xffffffff = empty), key, pattern offset / 16, first 16 bytes};
  // F: patterns whose home slot this is live further along the probe run
  std::vector<uint32_t> vtab;
  uint32_t vmask = 0;
  uint32_t vbits = 0;  // pack2: log2 slots
};
void build_pattern_table(const Plan& plan, const PatternData& pd, PatternTable* pt);

// Analytic read budget (filter.hpp:44-45; n-q+1 for the overlapping scan).
uint64_t filter_reads(const Plan& plan, uint64_t n);

// Seeded offsets for mag_sample_patterns (splitmix64, offset = next % span).
void sample_offsets(size_t corpus_len, size_t count, size_t length, uint64_t seed,
                    std::vector<uint64_t>* out);

}  // namespace magb
