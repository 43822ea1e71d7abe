// Host-side view of the device search kernels (scan_*.cu).
#pragma once

#include <cuda_runtime.h>

#include "mag_common.h"

namespace magb {

// Everything one scan launch needs.  Device pointers only.
//
// Work decomposition: the filter's samples t in [0, samples) are cut into
// slices of slice_samples.  A slice is owned by one warp (dynamic ticket)
// and produces the matches of exactly the candidate windows its samples
// raise, in (offset, pattern) order, into staging + slice * slice_cap.  A
// slice is streamed through the warp's ring of shared-memory slots in chunks
// of chunk_samples samples (TMA bulk copies, one mbarrier per slot).
//
// Ordered gather (concurrent, no second pass).  Slices form groups of 32
// (kGroup).  At the end of a slice its owner stores the count in
// slice_count[] and adds (1 << 40 | count) to its group's word.  A gather
// grid of one-warp CTAs runs beside the scan (programmatic dependent launch
// into the registers a 15-warp scan CTA leaves free): under a lock, one
// gather warp at a time advances the watermark
// (counters[kCtrWatermark], in groups) over complete groups, writing their
// inclusive prefix counts into group_incl[]; every gather warp claims one
// group at a time below the watermark, places its slices (a warp scan of
// their counts) and copies their staged matches to out[prefix..].  The last
// gather warp of the final launch of a search writes the counters to
// host_ctr (mapped pinned host memory) and zeroes the next search's control
// words.
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
  uint32_t nwarps;              // warps per scan CTA (the gather grid: one warp per CTA)
  uint64_t slice_begin, slice_end;  // slices of this launch (whole groups except at the text end)
  uint64_t num_slices;
  uint64_t* staging;            // num_slices * slice_cap packed matches
  uint32_t slice_cap;           // multiple of 16 (slices never share a 128-byte line)
  uint32_t* slice_count;        // per slice: exact match count (even past slice_cap)
  uint64_t* group_word;         // per group: completed slices << 40 | match count (zeroed after its copy)
  uint64_t* group_incl;         // per group: inclusive prefix of counts (valid below the watermark)
  uint64_t* out;                // sorted output
  uint64_t out_cap;
  unsigned long long* counters; // control words (kCtr*)
  unsigned long long* ticket;   // slice ticket of this launch (zeroed)
  unsigned long long* exits;    // warps of this launch that have left (zeroed)
  unsigned long long* copy_cursor;  // gather warps' copy claims of this launch (zeroed)
  uint32_t final_launch;        // 1: the search's last launch publishes the counters
  unsigned long long* host_ctr; // mapped pinned host words: [1] candidates [2] matches [3] max slice count
  unsigned long long* reset;    // zeroed by the final launch's last warp (next search's control words)
  uint32_t reset_words;
};

// Slice geometry (host and device).
constexpr unsigned kGroup = 32;  // slices per gather group
MAG_HD uint64_t slice_t0(const ScanArgs& a, uint64_t x) { return x * a.slice_samples; }
MAG_HD uint64_t slice_t1(const ScanArgs& a, uint64_t x) {
  const uint64_t t = (x + 1) * a.slice_samples;
  return t < a.samples ? t : a.samples;
}

// Control words of one search (a half of the workspace's ctrl array).
// Each group has its own 128-byte line, so the scanning warps' ticket
// atomics never share a line with the gather warps' polls.
constexpr unsigned kCtrWatermark = 0;  // gather watermark (groups)
constexpr unsigned kCtrTotal = 1;      // total matches (set when the watermark reaches the end)
constexpr unsigned kCtrLock = 16;      // watermark-advance lock
constexpr unsigned kCtrCands = 32;     // filter candidates
constexpr unsigned kCtrMax = 48;       // largest slice count
constexpr unsigned kCtrLaunch = 64;    // launch li: ticket at kCtrLaunch + kCtrPerLaunch * li, exits +16, copies +32
constexpr unsigned kCtrPerLaunch = 48;
constexpr unsigned kMaxLaunches = 64;
constexpr unsigned kCtrWords = kCtrLaunch + kCtrPerLaunch * kMaxLaunches;

struct LaunchShape {
  size_t smem_bytes;
  unsigned threads;
};

// Enqueues the fused filter + verify kernel (persistent, `grid` CTAs) and
// beside it, as its programmatic dependent, the gather grid (`grid` one-warp
// CTAs) that places the slices' matches in order.
cudaError_t launch_scan(const ScanArgs& a, cudaStream_t stream, int grid);

// SMAG prepare: codes[u] = mask index of gram u, for u < n/q.
cudaError_t launch_encode(const ScanPlan& plan, const uint8_t* text, uint64_t n,
                          const uint8_t* map, uint32_t* codes, cudaStream_t stream);

// Number of kernels this library has enqueued (process lifetime).
unsigned long long kernel_launch_count();

// ---- internal: per-family launchers (scan_*.cu)
cudaError_t launch_direct(const ScanArgs& a, cudaStream_t stream, int grid);
cudaError_t launch_roll(const ScanArgs& a, cudaStream_t stream, int grid);
cudaError_t launch_staged_exact(const ScanArgs& a, cudaStream_t stream, int grid);
cudaError_t launch_staged_hashed(const ScanArgs& a, cudaStream_t stream, int grid);
cudaError_t launch_staged_codes(const ScanArgs& a, cudaStream_t stream, int grid);
void count_launch();
// Raises a kernel's dynamic shared-memory limit to `need` on the current
// device when it is lower (per (kernel, device); thread-safe).
cudaError_t allow_max_smem(const void* kernel, size_t need);

}  // namespace magb
