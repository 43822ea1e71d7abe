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
// Ordered output.  Slices form groups of 32 (kGroup).  At the end of a slice
// its owner stores the count in slice_count[] and, when nonzero, adds it to
// its group's sum (one atomic; no fence: the finish grid reads them after
// the scan grid has completed).  The finish grid (scan_dispatch.cu), launched
// as the scan's programmatic dependent so its CTAs are resident and waiting
// when the scan's last CTA leaves, places every group: exclusive prefix of
// the group sums before it, a warp scan of its slice counts, a flat copy of
// the staged matches to out[].  Its last CTA writes the counters to host_ctr
// (mapped pinned host memory) and zeroes the next search's control words.
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
  unsigned long long* group_sum;       // per group: match count (this search's half, zero at its start)
  unsigned long long* group_sum_next;  // the other half: zeroed by the finish grid for the next search
  uint64_t group_sum_words;     // words per half
  uint64_t* out;                // sorted output
  uint64_t out_cap;
  unsigned long long* counters; // control words (kCtr*)
  unsigned long long* ticket;   // slice ticket of this launch (zeroed)
  unsigned long long* exits;    // finish CTAs that have left (zeroed)
  uint32_t final_launch;        // 1: the search's last launch; the finish grid follows it
  uint32_t finish_grid;         // CTAs of the finish grid (>= 1)
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
// atomics never share a line with the finish grid's counters.
constexpr unsigned kCtrTotal = 1;      // total matches (finish grid)
constexpr unsigned kCtrExits = 16;     // finish CTAs that have left
constexpr unsigned kCtrCands = 32;     // filter candidates
constexpr unsigned kCtrMax = 48;       // largest slice count
constexpr unsigned kCtrLaunch = 64;    // launch li: slice ticket at kCtrLaunch + kCtrPerLaunch * li
constexpr unsigned kCtrPerLaunch = 16;
constexpr unsigned kMaxLaunches = 64;
constexpr unsigned kCtrWords = kCtrLaunch + kCtrPerLaunch * kMaxLaunches;

struct LaunchShape {
  size_t smem_bytes;
  unsigned threads;
};

// Enqueues the fused filter + verify kernel (persistent, `grid` CTAs); after
// the search's final launch, the finish grid (programmatic dependent) that
// places the slices' matches in order and publishes the counters.
// `after_scan` (timing only) is recorded between the scan kernel and the
// finish grid; the finish grid then starts after the scan has completed.
cudaError_t launch_scan(const ScanArgs& a, cudaStream_t stream, int grid, cudaEvent_t after_scan = nullptr);

// SMAG prepare: codes[u] = mask index of gram u, for u < n/q.
cudaError_t launch_encode(const ScanPlan& plan, const uint8_t* text, uint64_t n,
                          const uint8_t* map, uint32_t* codes, cudaStream_t stream);

// Number of kernels this library has enqueued (process lifetime).
unsigned long long kernel_launch_count();

// ---- internal: per-family launchers (scan_*.cu)
cudaError_t launch_direct(const ScanArgs& a, cudaStream_t stream, int grid);
cudaError_t launch_roll(const ScanArgs& a, cudaStream_t stream, int grid);
cudaError_t launch_pack2(const ScanArgs& a, cudaStream_t stream, int grid);
cudaError_t launch_staged_exact(const ScanArgs& a, cudaStream_t stream, int grid);
cudaError_t launch_staged_hashed(const ScanArgs& a, cudaStream_t stream, int grid);
cudaError_t launch_staged_codes(const ScanArgs& a, cudaStream_t stream, int grid);
void count_launch();
// Raises a kernel's dynamic shared-memory limit to `need` on the current
// device when it is lower (per (kernel, device); thread-safe).
cudaError_t allow_max_smem(const void* kernel, size_t need);

}  // namespace magb
