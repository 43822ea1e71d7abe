// Host-side view of the device search kernels (scan_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include "mag_common.h"

namespace magb {

// Everything one scan launch needs.  Device pointers only.
struct ScanArgs {
  ScanPlan plan;
  const uint8_t* text;          // 16-byte aligned
  uint64_t n;
  const uint32_t* codes;        // SMAG: per-gram mask index, n/q entries
  const void* table;            // packed mask table (global copy)
  const uint32_t* prefilter;    // 2^pf_bits bits
  const uint32_t* bucket_start; // 2^bucket_bits + 1
  const uint2* bucket_entries;  // {key hash, pattern id}, r entries
  const uint8_t* pat_bytes;     // 16-byte aligned, zero padded per pattern
  const uint64_t* pat_off;
  const uint32_t* pat_len;
  const uint8_t* map;           // 256-byte alphabet map (exact grams)
  uint64_t samples;             // T: floor(n_q/k) strided, n-q+1 overlapping
  uint64_t tile_bytes;          // multiple of 16 and of the gram step
  uint64_t tile_begin, tile_end;  // tiles this launch owns
  uint64_t num_tiles;           // tiles of the whole search (status array)
  uint32_t halo;                // extra staged bytes after a tile
  uint32_t nwarps, stages, mbuf;
  uint64_t* out;                // packed (offset, pid) keys
  uint64_t out_cap;
  unsigned long long* status;   // num_tiles look-back words (zeroed per search)
  unsigned long long* counters; // [1] candidates, [2] matches
  unsigned long long* ticket;   // tile ticket of this launch (zeroed)
};

struct LaunchShape {
  size_t smem_bytes;
  unsigned threads;
};

// Computes the dynamic shared memory and block size of launch_scan().
LaunchShape scan_shape(const ScanArgs& a);

// Enqueues the fused filter+verify+ordered-output kernel.
cudaError_t launch_scan(const ScanArgs& a, cudaStream_t stream, int grid);

// SMAG prepare: codes[u] = mask index of gram u, for u < n/q.
cudaError_t launch_encode(const ScanPlan& plan, const uint8_t* text, uint64_t n,
                          const uint8_t* map, uint32_t* codes, cudaStream_t stream);

// Number of kernels this library has enqueued (process lifetime).
unsigned long long kernel_launch_count();

}  // namespace magb
