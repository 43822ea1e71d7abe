// Host-side view of the device search kernels (scan_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include "mag_common.h"

namespace magb {

// Everything one scan launch needs.  Device pointers only.
//
// Work decomposition: the filter's samples t in [0, samples) are cut into
// slices of slice_samples; a slice is owned by one warp (dynamic ticket) and
// produces the matches of exactly the candidate windows its samples raise,
// in (offset, pattern) order, into staging + slice * slice_cap.  A slice is
// streamed through the warp's ring of shared-memory slots in chunks of
// chunk_samples samples (TMA bulk copies, one mbarrier per slot).
struct ScanArgs {
  ScanPlan plan;
  const uint8_t* text;          // 16-byte aligned
  uint64_t n;
  const uint32_t* codes;        // SMAG: per-gram mask index, n/q entries
  const void* table;            // packed mask table (global copy)
  const uint32_t* prefilter;    // 2^pf_bits bits
  const uint32_t* bucket_start; // 2^bucket_bits + 1
  const uint32_t* l2map;        // 2^l2_bits-bit key bitmap (window keys)
  const uint2* bucket_entries;  // {key hash, pattern id}, r entries
  const uint8_t* pat_bytes;     // 16-byte aligned, zero padded per pattern
  const uint64_t* pat_off;
  const uint32_t* pat_len;
  const uint8_t* map;           // 256-byte alphabet map (exact grams)
  const uint4* vtab;            // roll: verification slots (2 x uint4 each), vmask + 1 of them
  uint32_t vmask;
  uint32_t zero;                // always 0; opaque to the compiler (orders slot reads before TMA refills)
  uint64_t samples;             // T: floor(n_q/k) strided, n-q+1 overlapping, n verify-all
  uint64_t slice_samples;       // multiple of chunk_samples
  uint32_t chunk_samples;       // samples per chunk (iterations * advance)
  uint32_t back;                // staged bytes after the last gram (pattern reach)
  uint32_t full_bytes;          // staged bytes of an interior chunk (multiple of 16)
  uint32_t slot_bytes;          // one ring slot (multiple of 16, >= full_bytes + 32)
  uint32_t ring;                // slots per warp
  uint32_t nwarps;              // warps per CTA
  uint64_t slice_begin, slice_end;  // slices of this launch
  uint64_t num_slices;
  uint64_t* staging;            // num_slices * slice_cap packed matches
  uint32_t slice_cap;
  uint32_t* slice_count;        // exact per-slice counts (even past slice_cap)
  unsigned long long* counters; // [1] candidates [2] matches [3] max slice count
  unsigned long long* ticket;   // slice ticket of this launch (zeroed)
  unsigned long long* reset;    // compaction zeroes reset[0..reset_words) (next search's counters)
  uint32_t reset_words;
};

struct LaunchShape {
  size_t smem_bytes;
  unsigned threads;
};

LaunchShape scan_shape(const ScanArgs& a);

// Enqueues the fused filter + verify kernel (persistent, `grid` CTAs).
cudaError_t launch_scan(const ScanArgs& a, cudaStream_t stream, int grid);

// Gathers the staged slices into the sorted output (out[0..total)) and
// writes counters[2] (total) and counters[3] (largest slice count).
cudaError_t launch_compact(const ScanArgs& a, uint64_t* out, uint64_t out_cap, cudaStream_t stream,
                           int grid);

// SMAG prepare: codes[u] = mask index of gram u, for u < n/q.
cudaError_t launch_encode(const ScanPlan& plan, const uint8_t* text, uint64_t n,
                          const uint8_t* map, uint32_t* codes, cudaStream_t stream);

// Number of kernels this library has enqueued (process lifetime).
unsigned long long kernel_launch_count();

}  // namespace magb
