/*
 * mag_b200.h — GPU additions to the mag.h ABI (libmag_b200.so).
 *
 * Nothing here changes the reference entry points in mag.h; these calls only
 * expose what a GPU caller needs beyond them: text that already lives in HBM,
 * stream-ordered (asynchronous) searches, the search plan the engine chose
 * and a few introspection hooks used by the parity tests.
 */
#ifndef MAG_B200_H
#define MAG_B200_H

#include "mag.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Gram modes of the filter's q-gram stage. */
typedef enum mag_gram_mode {
  MAG_GRAM_AUTO = -1,
  MAG_GRAM_EXACT = 0,  /* reference code: sum map(p[i]) * sigma'^i, sigma'^q entries */
  MAG_GRAM_HASHED = 1  /* raw q bytes hashed to 2^table_bits entries (paper §3.3) */
} mag_gram_mode;

/* Extended options.  mag_engine_create(opts) == mag_engine_create_ex with
 * every extra field left at its default. */
typedef struct mag_options_ex {
  mag_options base;
  int gram_mode;   /* mag_gram_mode */
  int table_bits;  /* hashed: log2 mask entries; 0 = auto; -1 = no filter (verify all) */
  int word_bits;   /* w of the reference machine (filter.hpp:34); 0 = 64 */
  int tile_bytes;  /* 0 = auto */
  int warps;       /* warps per scan CTA, 0 = auto (15 staged / W=16 direct, 16 W=8 direct / roll;
                      up to 24 for the roll kernel's equal-length short-set path) */
  int stages;      /* TMA ring depth, 0 = auto */
  int device;      /* CUDA device ordinal, -1 = current */
  int probes;      /* hashed: table entries probed per gram, 0 = auto */
  int scan_kernel; /* mag_scan_kernel: which scan the planner may pick, 0 = auto */
  int cluster;     /* 0 or 1 (kept for ABI stability; the cluster-shared table of round 1 was retired) */
} mag_options_ex;

/* Scan kernels of hashed plans (mag_options_ex.scan_kernel). */
typedef enum mag_scan_kernel {
  MAG_KERNEL_AUTO = 0,
  MAG_KERNEL_STAGED = 1, /* TMA-staged strided / overlapping machine (every plan shape) */
  MAG_KERNEL_DIRECT = 2, /* q = 16 aligned-sample stream + L2 screen (m >= 31) */
  MAG_KERNEL_ROLL = 3,   /* dense rolling-hash prefix Bloom scan (m >= 8) */
  MAG_KERNEL_PACK2 = 4   /* dense 2-bit exact-code scan (<= 4 pattern symbols, m >= 10) */
} mag_scan_kernel;

MAG_API void mag_options_ex_init(mag_options_ex* opts);
MAG_API mag_status mag_engine_create_ex(const uint8_t* const* patterns,
                                        const size_t* pattern_lens, size_t count,
                                        const mag_options_ex* opts, mag_engine** out);

/* The plan the engine runs (all fields are what the kernels use). */
typedef struct mag_plan_info {
  int variant;          /* mag_variant */
  int gram_mode;        /* mag_gram_mode in effect */
  int q, k, m_prime;
  int sigma_prime;
  int verify_all;       /* 1: the table admits everything; every start is verified */
  uint32_t table_bits;  /* hashed: log2 entries */
  uint32_t entry_bits;  /* bits per mask entry */
  uint64_t table_bytes;
  int table_in_smem;
  uint32_t key_len;     /* verification key bytes */
  uint32_t prefilter_bits;
  uint32_t bucket_bits;
  uint32_t tile_bytes, halo, warps, stages;
  size_t smem_bytes;
  double predicted_candidates_per_byte;
  uint32_t probes;      /* hashed, m' = k = 1: table entries probed per gram */
  uint32_t blocks;      /* probes >= 2: 64-entry table blocks */
  int direct;           /* q = 16 stream kernel */
  int roll;             /* dense rolling-hash scan (every position, q-byte prefix Bloom) */
  int cluster;          /* always 0 (kept for ABI stability) */
  int pack2;            /* dense 2-bit exact-code scan (sigma' = 4 codes, two levels) */
  /* Measured selectivity (mag_options.histogram_sample given, >= 4 KiB): the
   * plan's own filter, with its real tables, run over up to 1 MiB of that
   * sample at engine creation.  Replaces the uniform-text estimate of the
   * reference's cost model (tuner.hpp:58-66) when plans are compared. */
  double measured_candidates_per_byte; /* -1: no sample was given */
  uint64_t measured_sample_bytes;
  double predicted_cost;  /* planner cost, thread-instructions per text byte (analytic rate) */
  double measured_cost;   /* the same cost re-priced with the measured rate */
  uint32_t measured_plans; /* finalist plans (one per kernel family) measured on the sample */
  /* direct plans: filter hits per byte that also pass the L2 screen, and the
   * bucket entries those survivors walk (entries sharing their key); -1 otherwise */
  double measured_survivors_per_byte;
  double measured_walk_per_byte;
} mag_plan_info;

MAG_API mag_status mag_engine_get_plan(const mag_engine* engine, mag_plan_info* out);

/* Text already in device memory (caller-owned, must outlive the handle). */
MAG_API mag_status mag_prepare_device_text(const mag_engine* engine, const uint8_t* d_text,
                                           size_t len, mag_prepared** out);

/* Enqueue a search on `cuda_stream` (a cudaStream_t; NULL = legacy default)
 * and return at once.  The handle materialises (waits, copies the sorted
 * matches to the host) on first use by mag_matches_count/get/metrics or by
 * mag_matches_sync; destroying it unmaterialised is allowed.  The prepared
 * text (and the device memory behind mag_prepare_device_text) must outlive
 * the handle's materialisation: a slice that overflowed its staging is
 * searched again then. */
MAG_API mag_status mag_search_prepared_async(const mag_engine* engine,
                                             const mag_prepared* prepared, void* cuda_stream,
                                             mag_matches** out);
MAG_API mag_status mag_matches_sync(mag_matches* matches);

/* Bulk read of the sorted matches (after materialisation). */
MAG_API mag_status mag_matches_copy(const mag_matches* matches, uint64_t* offsets,
                                    uint32_t* pattern_indices, size_t capacity);

/* Introspection for tests. */
MAG_API mag_status mag_prepared_copy_codes(const mag_prepared* prepared, uint32_t* out,
                                           size_t count);
MAG_API mag_status mag_engine_copy_masks(const mag_engine* engine, uint64_t* out,
                                         size_t count);
MAG_API uint64_t mag_kernel_launches(void);

/* Device timing of a search's kernels: when enabled, every scan launch is
 * bracketed by CUDA events on its stream; read() waits for and sums them.
 * on = 1: the scan kernel and the finish grid that follows it (one search);
 * on = 2: the scan kernel alone (the end event is recorded between the two,
 * so the finish grid no longer overlaps the scan's tail: timing runs only). */
MAG_API void mag_scan_timer_enable(int on);
MAG_API mag_status mag_scan_timer_read(double* total_ms, uint64_t* launches);

#ifdef __cplusplus
}
#endif

#endif /* MAG_B200_H */
