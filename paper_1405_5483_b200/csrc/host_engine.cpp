// C ABI of libmag_b200.so (include/mag.h + include/mag_b200.h).
//
// Host side of the drop-in: validation and error convention of the
// reference (core.cpp:7-23, mag.h:6-7,156-157), engine construction (host
// preprocessing + one upload of masks / prefilter / pattern table to HBM),
// and the search orchestration around the device kernels in
// scan_kernels.cu.  No CPU search path exists: without a GPU every search
// entry point fails with MAG_ERR_INTERNAL.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/mag_b200.h"
#include "host_model.h"
#include "scan_launch.h"

using namespace magb;

namespace {

thread_local std::string tl_error;

mag_status fail(mag_status s, const std::string& msg) {
  tl_error = msg;
  return s;
}

mag_status cuda_fail(cudaError_t e, const char* what) {
  return fail(e == cudaErrorMemoryAllocation ? MAG_ERR_NO_MEMORY : MAG_ERR_INTERNAL,
              std::string(what) + ": " + cudaGetErrorString(e));
}

#define MAG_CUDA(call)                                   \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);  \
  } while (0)

template <class T>
cudaError_t upload(const std::vector<T>& v, T** out) {
  *out = nullptr;
  if (v.empty()) return cudaSuccess;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(out), v.size() * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*out, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
}

// Per-search device scratch, pooled per engine.  `done` orders reuse on the
// device (a later search waits for it with cudaStreamWaitEvent).
struct Workspace {
  // two halves of kCtrWords control words (scan_launch.h): a
  // search uses half `parity` and the last warp of its final launch zeroes
  // the other half for the next search on this workspace (no memset launch
  // per search).  `dirty`: a search failed half-way; both halves are
  // cleared before the next one.
  unsigned long long* ctrl = nullptr;
  uint32_t parity = 0;
  bool dirty = false;
  uint32_t* slice_count = nullptr;     // per slice: match count
  unsigned long long* group_sum = nullptr;  // two halves (parity) of per-group match counts
  size_t slices_cap = 0;
  uint64_t* staging = nullptr;         // num_slices * slice_cap staged matches
  uint64_t* out = nullptr;             // sorted matches (same capacity)
  size_t out_cap = 0;
  unsigned long long* h_ctr = nullptr;  // mapped pinned [1] candidates [2] matches [3] max, written by the kernel
  unsigned long long* d_hctr = nullptr; // its device alias
  uint8_t* text = nullptr;              // device copy of host text (mag_search)
  size_t text_cap = 0;
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> chunk_ev;
  cudaEvent_t done = nullptr;
  int device = 0;
  // geometry of the last enqueued search
  uint64_t num_slices = 0, slice_cap = 0, slice_samples = 0;

  ~Workspace() {
    cudaSetDevice(device);
    if (ctrl) cudaFree(ctrl);
    if (slice_count) cudaFree(slice_count);
    if (group_sum) cudaFree(group_sum);
    if (staging) cudaFree(staging);
    if (out) cudaFree(out);
    if (h_ctr) cudaFreeHost(h_ctr);
    if (text) cudaFree(text);
    for (auto ev : chunk_ev) cudaEventDestroy(ev);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (done) cudaEventDestroy(done);
  }
};

constexpr size_t kMaxLaunch = kMaxLaunches;

// Optional device timing of the scan kernel launches (bench/profiling only):
// CUDA events around every launch_scan, read back by mag_scan_timer_read.
struct ScanTimer {
  std::mutex mu;
  bool on = false;
  bool scan_only = false;  // mode 2: the end event sits between the scan kernel and the finish grid
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> spare;
  double total_ms = 0;
  uint64_t launches = 0;
};
ScanTimer g_timer;

cudaError_t timed_launch(const ScanArgs& a, cudaStream_t st, int grid) {
  if (!g_timer.on) return launch_scan(a, st, grid);
  std::pair<cudaEvent_t, cudaEvent_t> ev;
  {
    std::lock_guard<std::mutex> g(g_timer.mu);
    if (!g_timer.spare.empty()) {
      ev = g_timer.spare.back();
      g_timer.spare.pop_back();
    } else {
      cudaEventCreate(&ev.first);
      cudaEventCreate(&ev.second);
    }
  }
  cudaEventRecord(ev.first, st);
  const bool scan_only = g_timer.scan_only;
  cudaError_t e = launch_scan(a, st, grid, scan_only ? ev.second : nullptr);
  if (!scan_only) cudaEventRecord(ev.second, st);
  std::lock_guard<std::mutex> g(g_timer.mu);
  g_timer.pending.push_back(ev);
  return e;
}

}  // namespace

struct mag_engine {
  PatternData pd;
  Histogram hist;
  Plan plan;
  std::vector<uint8_t> table;  // packed masks (host copy)
  PatternTable ptab;
  int device = -1;  // -2: host-only engine (no upload)
  int sm_count = 148;
  // device tables
  void* d_table = nullptr;
  uint32_t* d_prefilter = nullptr;
  uint32_t* d_l2map = nullptr;
  uint32_t* d_bucket_start = nullptr;
  uint32_t* d_entries = nullptr;
  uint32_t* d_vtab = nullptr;
  uint8_t* d_pat_bytes = nullptr;
  uint64_t* d_pat_off = nullptr;
  uint32_t* d_pat_len = nullptr;
  uint8_t* d_map = nullptr;
  // learned output density: max matches per slice seen so far, per sample
  mutable double slice_density = 0;
  // pool
  mutable std::mutex mu;
  mutable std::vector<std::unique_ptr<Workspace>> pool;

  ~mag_engine() {
    pool.clear();
    if (device >= 0) {
      cudaSetDevice(device);
      cudaFree(d_table);
      cudaFree(d_prefilter);
      cudaFree(d_l2map);
      cudaFree(d_bucket_start);
      cudaFree(d_entries);
      cudaFree(d_vtab);
      cudaFree(d_pat_bytes);
      cudaFree(d_pat_off);
      cudaFree(d_pat_len);
      cudaFree(d_map);
    }
  }
};

struct mag_prepared {
  const mag_engine* engine = nullptr;
  const uint8_t* host_text = nullptr;
  const uint8_t* d_text = nullptr;  // what the kernels read
  uint8_t* d_owned = nullptr;       // our copy, if any
  uint32_t* d_codes = nullptr;      // SMAG gram indices
  size_t len = 0;
  ~mag_prepared() {
    if (engine && engine->device >= 0) {
      cudaSetDevice(engine->device);
      if (d_owned) cudaFree(d_owned);
      if (d_codes) cudaFree(d_codes);
    }
  }
};

struct mag_matches {
  const mag_engine* engine = nullptr;
  std::vector<uint64_t> keys;
  mag_metrics metrics{0, 0};
  // pending (asynchronous) state
  bool pending = false;
  std::unique_ptr<Workspace> ws;
  cudaStream_t stream = nullptr;
  const uint8_t* d_text = nullptr;
  const uint32_t* d_codes = nullptr;
  size_t n = 0;
  mag_status sticky = MAG_OK;
  std::string sticky_msg;
  ~mag_matches();
};

struct mag_patterns {
  std::vector<std::vector<uint8_t>> items;
};

namespace {

std::unique_ptr<Workspace> acquire(const mag_engine* e) {
  std::lock_guard<std::mutex> g(e->mu);
  if (!e->pool.empty()) {
    auto w = std::move(e->pool.back());
    e->pool.pop_back();
    return w;
  }
  auto w = std::make_unique<Workspace>();
  w->device = e->device;
  return w;
}

void release(const mag_engine* e, std::unique_ptr<Workspace> w) {
  if (!w) return;
  std::lock_guard<std::mutex> g(e->mu);
  e->pool.push_back(std::move(w));
}

constexpr size_t kCounters = 8;
constexpr size_t kCtrlWords = kCtrWords;

struct SearchGeometry {
  uint64_t samples, slice_samples, num_slices, slice_cap;
  uint32_t bps;  // text bytes per sample
};

uint64_t bytes_per_sample(const Plan& P) {
  return P.sp.verify_all || P.sp.overlapping ? 1 : static_cast<uint64_t>(P.sp.q) * P.sp.k;
}

uint64_t step_unit(const Plan& P) {
  if (P.sp.pack2) return kPack2Step;
  return P.sp.roll ? P.sp.roll_step : (P.sp.direct ? direct_step_bytes(P.sp.q) / P.sp.q : P.chunk_samples);
}

// Slices are the warps' work items: the plan's size, but small texts get
// smaller slices (whole kernel steps) so that every warp of the grid has
// one (direct plans) or two of them: each slice costs a ticket, a TMA ramp
// and an exposed screen round trip at its end.
uint64_t slice_samples_for(const mag_engine* e, uint64_t samples) {
  const Plan& P = e->plan;
  const uint64_t unit = step_unit(P);
  // B200, slices per warp 4 / 2 / 1: cfg1 (16 MiB, direct) 420 / 489 / 539 GB/s per step,
  // cfg2 at 64 MiB 1,572 / 1,613 / 1,734; cfg5 at 32 MiB (roll) 438 / 449 / 405
  const uint64_t per_warp = P.sp.direct ? 1 : 2;
  const uint64_t warps = static_cast<uint64_t>(e->sm_count) * P.nwarps * per_warp;
  uint64_t want = (samples + warps - 1) / warps;
  want = (want + unit - 1) / unit * unit;
  return std::max<uint64_t>(unit, std::min<uint64_t>(P.slice_samples, want));
}

SearchGeometry geometry(const mag_engine* e, uint64_t n, uint64_t cap_override) {
  const Plan& P = e->plan;
  SearchGeometry g;
  g.samples = filter_reads(P, n);
  g.bps = static_cast<uint32_t>(bytes_per_sample(P));
  g.slice_samples = slice_samples_for(e, g.samples);
  g.num_slices = (g.samples + g.slice_samples - 1) / g.slice_samples;
  if (cap_override) {
    g.slice_cap = cap_override;
  } else {
    double dens;
    {
      std::lock_guard<std::mutex> lk(e->mu);
      dens = e->slice_density;
    }
    // until a search has been seen: 1 match per 128 text bytes of a slice
    const double bytes = static_cast<double>(g.slice_samples) *
                         (P.sp.verify_all || P.sp.overlapping ? 1 : P.sp.q * P.sp.k);
    const double guess = std::max(dens * static_cast<double>(g.slice_samples) * 1.25, bytes / 128);
    g.slice_cap = std::max<uint64_t>(64, static_cast<uint64_t>(guess) + 32);
  }
  g.slice_cap = (g.slice_cap + 15) / 16 * 16;  // slices never share a 128-byte line
  return g;
}

ScanArgs geometry_args(const SearchGeometry& g) {
  ScanArgs a{};
  a.samples = g.samples;
  a.slice_samples = g.slice_samples;
  a.num_slices = g.num_slices;
  return a;
}

// Slices [0, k) whose last sample ends at most `bytes` bytes into the text.
uint64_t slices_ending_by(const SearchGeometry& g, uint64_t bytes) {
  const ScanArgs a = geometry_args(g);
  uint64_t lo = 0, hi = g.num_slices;  // answer in [lo, hi]
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo + 1) / 2;  // is slice mid-1 covered?
    if (slice_t1(a, mid - 1) * g.bps <= bytes)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

mag_status ensure_ws(Workspace* w, const SearchGeometry& g, cudaStream_t st) {
  if (!w->done) MAG_CUDA(cudaEventCreateWithFlags(&w->done, cudaEventDisableTiming));
  if (!w->h_ctr) {
    MAG_CUDA(cudaHostAlloc(&w->h_ctr, kCounters * sizeof(unsigned long long), cudaHostAllocMapped));
    std::memset(w->h_ctr, 0, kCounters * sizeof(unsigned long long));
    MAG_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&w->d_hctr), w->h_ctr, 0));
  }
  if (!w->ctrl) {
    MAG_CUDA(cudaMalloc(&w->ctrl, 2 * kCtrlWords * sizeof(unsigned long long)));
    w->dirty = true;
  }
  if (w->dirty) {  // new, or a search failed half-way: control words and group words from zero
    MAG_CUDA(cudaMemsetAsync(w->ctrl, 0, 2 * kCtrlWords * sizeof(unsigned long long), st));
    if (w->group_sum) MAG_CUDA(cudaMemsetAsync(w->group_sum, 0, 2 * w->slices_cap / kGroup * sizeof(uint64_t), st));
    w->parity = 0;
    w->dirty = false;
  }
  if (w->slices_cap < std::max<uint64_t>(1, g.num_slices)) {
    if (w->slice_count) MAG_CUDA(cudaFree(w->slice_count));
    if (w->group_sum) MAG_CUDA(cudaFree(w->group_sum));
    w->slice_count = nullptr;
    w->group_sum = nullptr;
    w->slices_cap = 0;
    const size_t cap = (std::max<uint64_t>(1, g.num_slices) + kGroup - 1) / kGroup * kGroup;
    MAG_CUDA(cudaMalloc(&w->slice_count, cap * sizeof(uint32_t)));
    MAG_CUDA(cudaMalloc(&w->group_sum, 2 * cap / kGroup * sizeof(uint64_t)));
    MAG_CUDA(cudaMemsetAsync(w->group_sum, 0, 2 * cap / kGroup * sizeof(uint64_t), st));
    w->slices_cap = cap;
  }
  const size_t cap = std::max<size_t>(1, g.num_slices * g.slice_cap);
  if (w->out_cap < cap) {
    if (w->out) MAG_CUDA(cudaFree(w->out));
    if (w->staging) MAG_CUDA(cudaFree(w->staging));
    w->out = w->staging = nullptr;
    w->out_cap = 0;
    MAG_CUDA(cudaMalloc(&w->staging, cap * sizeof(uint64_t)));
    MAG_CUDA(cudaMalloc(&w->out, cap * sizeof(uint64_t)));
    w->out_cap = cap;
  }
  return MAG_OK;
}

struct SliceRange {
  uint64_t begin, end;
  cudaEvent_t wait;  // may be null
};

// Enqueue one complete search over device text: the fused kernel over the
// slice ranges (one launch per range, each after its range's wait event);
// after the final launch, the finish grid places the matches in order,
// leaves the counters in the mapped host copy and clears the next search's
// control words; record ws->done.  All on `st`.
mag_status enqueue_search(const mag_engine* e, Workspace* w, const uint8_t* d_text, uint64_t n,
                          const uint32_t* d_codes, cudaStream_t st,
                          const std::vector<SliceRange>& ranges, uint64_t cap_override = 0) {
  const Plan& P = e->plan;
  const SearchGeometry g = geometry(e, n, cap_override);
  mag_status s = ensure_ws(w, g, st);
  if (s != MAG_OK) return s;
  w->dirty = true;  // until every launch of this search is enqueued
  w->num_slices = g.num_slices;
  w->slice_cap = g.slice_cap;
  w->slice_samples = g.slice_samples;
  unsigned long long* counters = w->ctrl + w->parity * kCtrlWords;
  unsigned long long* next_ctrl = w->ctrl + (w->parity ^ 1u) * kCtrlWords;
  ScanArgs a = geometry_args(g);
  a.plan = P.sp;
#ifdef MAG_B200_DIAGNOSTICS
  if (const char* d = std::getenv("MAG_B200_DIAG")) a.plan.diag = std::atoi(d);  // profiling builds only
#else
  a.plan.diag = 0;
#endif
  a.text = d_text;
  a.n = n;
  a.codes = d_codes;
  a.table = e->d_table;
  a.prefilter = e->d_prefilter;
  a.bucket_start = e->d_bucket_start;
  a.l2map = e->d_l2map;
  a.bucket_entries = reinterpret_cast<const uint2*>(e->d_entries);
  a.vtab = reinterpret_cast<const uint4*>(e->d_vtab);
  a.vmask = e->ptab.vmask;
  a.pat_bytes = e->d_pat_bytes;
  a.pat_off = e->d_pat_off;
  a.pat_len = e->d_pat_len;
  a.map = e->d_map;
  a.chunk_samples = P.chunk_samples;
  a.back = P.back;
  a.slot_bytes = P.slot_bytes;
  a.full_bytes = P.full_bytes;
  a.ring = P.ring;
  a.nwarps = P.nwarps;
  a.staging = w->staging;
  a.slice_cap = static_cast<uint32_t>(std::min<uint64_t>(g.slice_cap, 0xfffffff0u));
  a.slice_count = w->slice_count;
  a.group_sum_words = w->slices_cap / kGroup;
  a.group_sum = w->group_sum + w->parity * a.group_sum_words;
  a.group_sum_next = w->group_sum + (w->parity ^ 1u) * a.group_sum_words;
  a.out = w->out;
  a.out_cap = w->out_cap;
  a.counters = counters;
  a.host_ctr = w->d_hctr;
  a.reset = next_ctrl;
  a.reset_words = static_cast<uint32_t>(kCtrlWords);
  // the last non-empty range is the final launch (an empty search still
  // launches once, so the counters get published)
  size_t last = ranges.size();
  for (size_t i = 0; i < ranges.size(); ++i)
    if (ranges[i].end > ranges[i].begin) last = i;
  size_t li = 0;
  auto launch = [&](uint64_t begin, uint64_t end, bool final_launch) -> mag_status {
    if (li >= kMaxLaunch) return fail(MAG_ERR_INTERNAL, "too many scan launches for one search");
    a.slice_begin = begin;
    a.slice_end = end;
    a.ticket = counters + kCtrLaunch + kCtrPerLaunch * li;
    a.exits = counters + kCtrExits;
    ++li;
    const uint64_t ctas = std::max<uint64_t>(1, (end - begin + P.nwarps - 1) / P.nwarps);
    const int grid = static_cast<int>(std::min<uint64_t>(ctas, static_cast<uint64_t>(e->sm_count)));
    a.final_launch = final_launch ? 1u : 0u;
    a.finish_grid = static_cast<uint32_t>(std::max<uint64_t>(
        1, std::min<uint64_t>((g.num_slices + kGroup - 1) / kGroup, static_cast<uint64_t>(e->sm_count))));
    MAG_CUDA(timed_launch(a, st, grid));
    return MAG_OK;
  };
  for (size_t i = 0; i < ranges.size(); ++i) {
    const SliceRange& r = ranges[i];
    if (r.wait) MAG_CUDA(cudaStreamWaitEvent(st, r.wait, 0));
    if (r.end <= r.begin) continue;
    s = launch(r.begin, r.end, i == last);
    if (s != MAG_OK) return s;
  }
  if (last == ranges.size()) {
    s = launch(0, 0, true);
    if (s != MAG_OK) return s;
  }
  MAG_CUDA(cudaEventRecord(w->done, st));
  w->parity ^= 1u;
  w->dirty = false;
  return MAG_OK;
}

uint64_t analytic_candidates(const Plan& P, uint64_t n) {
  // verify-all plans admit every code: every sample t (q = k = m' = 1) fires.
  return filter_reads(P, n);
}

// Waits for a pending search, reruns it if a slice overflowed its staging
// capacity (counts are exact even then), copies the sorted keys to the host.
mag_status materialize(mag_matches* m) {
  if (!m->pending) return m->sticky;
  const mag_engine* e = m->engine;
  cudaSetDevice(e->device);
  Workspace* w = m->ws.get();
  MAG_CUDA(cudaEventSynchronize(w->done));
  volatile unsigned long long* hc = w->h_ctr;  // written by the kernel (mapped)
  unsigned long long total = hc[2], maxc = hc[3];
  if (maxc > w->slice_cap) {
    const uint64_t slices = w->num_slices;
    mag_status s = enqueue_search(e, w, m->d_text, m->n, m->d_codes, m->stream,
                                  {SliceRange{0, slices, nullptr}}, maxc);
    if (s != MAG_OK) return s;
    MAG_CUDA(cudaEventSynchronize(w->done));
    total = hc[2];
    maxc = hc[3];
  }
  {
    const double dens = static_cast<double>(maxc) / static_cast<double>(std::max<uint64_t>(1, w->slice_samples));
    std::lock_guard<std::mutex> lk(e->mu);
    e->slice_density = std::max(e->slice_density, dens);
  }
  m->keys.resize(total);
  if (total)
    MAG_CUDA(cudaMemcpy(m->keys.data(), w->out, total * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  m->metrics.filter_reads = filter_reads(e->plan, m->n);
  m->metrics.candidates = e->plan.sp.verify_all ? analytic_candidates(e->plan, m->n) : hc[1];
#ifdef MAG_B200_DIAGNOSTICS
  if (std::getenv("MAG_B200_TIMELINE"))
    std::fprintf(stderr, "timeline_ns last_scan_end=%llu watermark_end=%llu last_gather_exit=%llu last_gather_start=%llu\n",
                 hc[4], hc[5], hc[6], hc[7]);
#endif
  m->pending = false;
  release(e, std::move(m->ws));
  return MAG_OK;
}

mag_status validate_patterns(const uint8_t* const* patterns, const size_t* lens, size_t count,
                             PatternData* pd) {
  if (!patterns || !lens) return fail(MAG_ERR_NULL_ARGUMENT, "patterns / pattern_lens is NULL");
  if (count == 0) return fail(MAG_ERR_EMPTY_PATTERN_SET, "pattern set is empty");  // core.cpp:8
  size_t total = 0;
  for (size_t i = 0; i < count; ++i) {
    if (lens[i] == 0)  // core.cpp:9-12
      return fail(MAG_ERR_EMPTY_PATTERN, "pattern " + std::to_string(i) + " is empty");
    if (!patterns[i]) return fail(MAG_ERR_NULL_ARGUMENT, "pattern " + std::to_string(i) + " is NULL");
    total += align16(lens[i]);
  }
  pd->r = count;
  pd->off.resize(count);
  pd->len.resize(count);
  pd->bytes.assign(total + 16, 0);
  size_t o = 0;
  pd->m = lens[0];
  pd->maxlen = lens[0];
  for (size_t i = 0; i < count; ++i) {
    if (lens[i] > 0xffffffffull) return fail(MAG_ERR_INVALID_ARGUMENT, "pattern longer than 4 GiB");
    pd->off[i] = o;
    pd->len[i] = static_cast<uint32_t>(lens[i]);
    std::memcpy(pd->bytes.data() + o, patterns[i], lens[i]);
    o += align16(lens[i]);
    pd->m = std::min(pd->m, lens[i]);
    pd->maxlen = std::max(pd->maxlen, lens[i]);
  }
  return MAG_OK;
}

mag_status upload_engine(mag_engine* e) {
  MAG_CUDA(cudaSetDevice(e->device));
  MAG_CUDA(cudaDeviceGetAttribute(&e->sm_count, cudaDevAttrMultiProcessorCount, e->device));
  MAG_CUDA(upload(e->table, reinterpret_cast<uint8_t**>(&e->d_table)));
  MAG_CUDA(upload(e->ptab.prefilter, &e->d_prefilter));
  MAG_CUDA(upload(e->ptab.l2map, &e->d_l2map));
  MAG_CUDA(upload(e->ptab.bucket_start, &e->d_bucket_start));
  MAG_CUDA(upload(e->ptab.entries, &e->d_entries));
  MAG_CUDA(upload(e->ptab.vtab, &e->d_vtab));
  MAG_CUDA(upload(e->pd.bytes, &e->d_pat_bytes));
  MAG_CUDA(upload(e->pd.off, &e->d_pat_off));
  MAG_CUDA(upload(e->pd.len, &e->d_pat_len));
  std::vector<uint8_t> map(e->plan.map, e->plan.map + 256);
  MAG_CUDA(upload(map, &e->d_map));
  // Keep freed stream-ordered memory cached (no re-allocation per search).
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, e->device) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  return MAG_OK;
}

mag_status device_guard(const mag_engine* e) {
  if (e->device < 0)
    return fail(MAG_ERR_INTERNAL, "engine has no CUDA device (created host-only or no GPU)");
  MAG_CUDA(cudaSetDevice(e->device));
  return MAG_OK;
}

mag_status encode_codes(const mag_engine* e, mag_prepared* p, cudaStream_t st) {
  const Plan& P = e->plan;
  if (!P.sp.smag || P.sp.verify_all) return MAG_OK;
  const uint64_t nq = p->len / P.sp.q;
  if (!nq) return MAG_OK;
  MAG_CUDA(cudaMalloc(&p->d_codes, nq * sizeof(uint32_t)));
  MAG_CUDA(launch_encode(P.sp, p->d_text, p->len, e->d_map, p->d_codes, st));
  return MAG_OK;
}

}  // namespace

mag_matches::~mag_matches() {
  if (ws && engine) {
    // Unmaterialised: the device may still be using the workspace; its
    // `done` event orders the next user, so it can go back to the pool.
    release(engine, std::move(ws));
  }
}

// =====================================================================
extern "C" {

MAG_API void mag_options_init(mag_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->variant = MAG_VARIANT_MAG;
  o->mapping = MAG_MAPPING_AUTO;
  o->threads = 1;
}

MAG_API void mag_options_ex_init(mag_options_ex* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  mag_options_init(&o->base);
  o->gram_mode = MAG_GRAM_AUTO;
  o->device = -1;
}

MAG_API mag_status mag_engine_create_ex(const uint8_t* const* patterns, const size_t* lens,
                                        size_t count, const mag_options_ex* opts_in,
                                        mag_engine** out) {
  if (!out) return fail(MAG_ERR_NULL_ARGUMENT, "out is NULL");
  *out = nullptr;
  mag_options_ex opts;
  if (opts_in)
    opts = *opts_in;
  else
    mag_options_ex_init(&opts);
  try {
    auto e = std::make_unique<mag_engine>();
    mag_status s = validate_patterns(patterns, lens, count, &e->pd);
    if (s != MAG_OK) return s;
    for (size_t i = 0; i < count; ++i) e->hist.add(patterns[i], lens[i]);
    if (opts.base.histogram_sample && opts.base.histogram_sample_len)
      e->hist.add(opts.base.histogram_sample,
                  std::min<size_t>(opts.base.histogram_sample_len, size_t(1) << 20));
    PlanRequest rq;
    rq.variant = opts.base.variant;
    rq.mapping = opts.base.mapping;
    rq.lowbits = opts.base.lowbits;
    rq.q = opts.base.q;
    rq.k = opts.base.k;
    rq.sigma_prime = opts.base.sigma_prime;
    rq.gram_mode = opts.gram_mode;
    rq.table_bits = opts.table_bits;
    rq.word_bits = opts.word_bits;
    rq.tile_bytes = opts.tile_bytes;
    rq.warps = opts.warps;
    rq.stages = opts.stages;
    rq.probes = opts.probes;
    rq.cluster = opts.cluster;
    if (opts.cluster != 0 && opts.cluster != 1)
      return fail(MAG_ERR_BAD_CONFIG, "cluster must be 0 (auto) or 1 (the cluster-shared table was retired)");
    rq.kernel = opts.scan_kernel;
    if (opts.scan_kernel < 0 || opts.scan_kernel > 4)
      return fail(MAG_ERR_BAD_CONFIG, "unknown scan kernel " + std::to_string(opts.scan_kernel));
    if (opts.base.q < 0 || opts.base.k < 0 || opts.base.sigma_prime < 0)
      return fail(MAG_ERR_BAD_CONFIG, "q, k and sigma' must be >= 0 (0 = auto)");
    if (opts.base.mapping < -1 || opts.base.mapping > 3)
      return fail(MAG_ERR_BAD_CONFIG, "unknown mapping " + std::to_string(opts.base.mapping));
    std::string err;
    // a text sample also prices the finalist plans by their measured candidate rates
    int ps = make_plan_measured(e->pd, e->hist, rq, opts.base.histogram_sample,
                                opts.base.histogram_sample ? opts.base.histogram_sample_len : 0, &e->plan, &err);
    if (ps != 0) return fail(static_cast<mag_status>(ps), err);
    build_masks(e->plan, e->pd, &e->table);
    build_pattern_table(e->plan, e->pd, &e->ptab);
    e->plan.sp.vbits = e->ptab.vbits;
    if (opts.device == -2) {
      e->device = -2;
    } else {
      int dev = opts.device;
      if (dev < 0) {
        cudaError_t ce = cudaGetDevice(&dev);
        if (ce != cudaSuccess) {
          cudaGetLastError();
          return fail(MAG_ERR_INTERNAL, std::string("no CUDA device: ") + cudaGetErrorString(ce));
        }
      }
      int ndev = 0;
      if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(MAG_ERR_INTERNAL, "no CUDA device available (this library has no CPU path)");
      }
      e->device = dev;
      s = upload_engine(e.get());
      if (s != MAG_OK) return s;
    }
    *out = e.release();
    return MAG_OK;
  } catch (const std::bad_alloc&) {
    return fail(MAG_ERR_NO_MEMORY, "out of host memory");
  } catch (const std::exception& ex) {
    return fail(MAG_ERR_INTERNAL, ex.what());
  }
}

MAG_API mag_status mag_engine_create(const uint8_t* const* patterns, const size_t* lens,
                                     size_t count, const mag_options* opts, mag_engine** out) {
  mag_options_ex ex;
  mag_options_ex_init(&ex);
  if (opts) ex.base = *opts;
  return mag_engine_create_ex(patterns, lens, count, &ex, out);
}

MAG_API void mag_engine_destroy(mag_engine* e) { delete e; }

MAG_API mag_status mag_engine_get_info(const mag_engine* e, mag_engine_info* out) {
  if (!e || !out) return fail(MAG_ERR_NULL_ARGUMENT, "engine / out is NULL");
  out->variant = e->plan.variant;
  out->r = static_cast<uint32_t>(e->pd.r);
  out->m = e->pd.m;
  out->q = static_cast<int>(e->plan.sp.q);
  out->k = static_cast<int>(e->plan.sp.k);
  out->sigma_prime = static_cast<int>(e->plan.sp.sigma_prime);
  out->mapping = e->plan.mapping;
  return MAG_OK;
}

MAG_API mag_status mag_engine_get_plan(const mag_engine* e, mag_plan_info* out) {
  if (!e || !out) return fail(MAG_ERR_NULL_ARGUMENT, "engine / out is NULL");
  const Plan& P = e->plan;
  // the machine that runs: mag may be planned onto the overlapping scan
  out->variant = P.sp.overlapping ? MAG_VARIANT_SHIFTOR_OG : P.variant;
  out->gram_mode = P.sp.gram_mode;
  out->q = static_cast<int>(P.sp.q);
  out->k = static_cast<int>(P.sp.k);
  out->m_prime = static_cast<int>(P.sp.m_prime);
  out->sigma_prime = static_cast<int>(P.sp.sigma_prime);
  out->verify_all = P.sp.verify_all;
  out->table_bits = P.sp.table_bits;
  out->entry_bits = 1u << P.sp.entry_log2;
  out->table_bytes = P.sp.table_bytes;
  out->table_in_smem = P.sp.table_in_smem;
  out->key_len = P.sp.key_len;
  out->prefilter_bits = P.sp.pf_bits;
  out->bucket_bits = P.sp.bucket_bits;
  out->tile_bytes = static_cast<uint32_t>(
      P.chunk_samples * (P.sp.verify_all || P.sp.overlapping ? 1 : P.sp.q * P.sp.k));
  out->halo = P.back;
  out->warps = P.nwarps;
  out->stages = P.ring;
  out->smem_bytes = plan_smem(P);
  out->predicted_candidates_per_byte = P.pred_cand_per_byte;
  out->probes = P.sp.probes;
  out->blocks = P.sp.blocks;
  out->direct = P.sp.direct;
  out->roll = P.sp.roll;
  out->cluster = 0;
  out->pack2 = P.sp.pack2;
  out->measured_candidates_per_byte = P.meas_cand_per_byte;
  out->measured_sample_bytes = P.meas_sample_bytes;
  out->predicted_cost = P.pred_cost;
  out->measured_cost = P.meas_cand_per_byte < 0 ? P.pred_cost : P.meas_cost;
  out->measured_plans = P.meas_plans;
  out->measured_survivors_per_byte = P.meas_surv_per_byte;
  out->measured_walk_per_byte = P.meas_walk_per_byte;
  return MAG_OK;
}

MAG_API mag_status mag_engine_copy_alphabet(const mag_engine* e, uint8_t table[256],
                                            uint32_t* sigma_prime) {
  if (!e || !table || !sigma_prime) return fail(MAG_ERR_NULL_ARGUMENT, "NULL argument");
  std::memcpy(table, e->plan.map, 256);
  *sigma_prime = e->plan.sp.sigma_prime;
  return MAG_OK;
}

MAG_API mag_status mag_engine_copy_masks(const mag_engine* e, uint64_t* out, size_t count) {
  if (!e || (!out && count)) return fail(MAG_ERR_NULL_ARGUMENT, "NULL argument");
  if (count > e->plan.sp.entries) return fail(MAG_ERR_OUT_OF_RANGE, "more entries than the table");
  for (size_t i = 0; i < count; ++i) out[i] = mask_entry(e->plan, e->table, i);
  return MAG_OK;
}

MAG_API mag_status mag_prepare_text(const mag_engine* e, const uint8_t* text, size_t len,
                                    mag_prepared** out) {
  if (!e || !out || (!text && len)) return fail(MAG_ERR_NULL_ARGUMENT, "NULL argument");
  *out = nullptr;
  if (len >= kMaxText) return fail(MAG_ERR_INVALID_ARGUMENT, "text longer than 2^40 bytes");
  mag_status s = device_guard(e);
  if (s != MAG_OK) return s;
  auto p = std::make_unique<mag_prepared>();
  p->engine = e;
  p->host_text = text;
  p->len = len;
  MAG_CUDA(cudaMalloc(&p->d_owned, align16(len) + 64));
  if (len) MAG_CUDA(cudaMemcpy(p->d_owned, text, len, cudaMemcpyHostToDevice));
  p->d_text = p->d_owned;
  s = encode_codes(e, p.get(), cudaStreamPerThread);
  if (s != MAG_OK) return s;
  MAG_CUDA(cudaStreamSynchronize(cudaStreamPerThread));
  *out = p.release();
  return MAG_OK;
}

MAG_API mag_status mag_prepare_device_text(const mag_engine* e, const uint8_t* d_text,
                                           size_t len, mag_prepared** out) {
  if (!e || !out || (!d_text && len)) return fail(MAG_ERR_NULL_ARGUMENT, "NULL argument");
  *out = nullptr;
  if (len >= kMaxText) return fail(MAG_ERR_INVALID_ARGUMENT, "text longer than 2^40 bytes");
  mag_status s = device_guard(e);
  if (s != MAG_OK) return s;
  auto p = std::make_unique<mag_prepared>();
  p->engine = e;
  p->len = len;
  if (reinterpret_cast<uintptr_t>(d_text) % 16 != 0) {
    // the TMA stages need 16-byte aligned sources: keep an aligned copy
    MAG_CUDA(cudaMalloc(&p->d_owned, align16(len) + 64));
    if (len) MAG_CUDA(cudaMemcpy(p->d_owned, d_text, len, cudaMemcpyDeviceToDevice));
    p->d_text = p->d_owned;
  } else {
    p->d_text = d_text;
  }
  s = encode_codes(e, p.get(), cudaStreamPerThread);
  if (s != MAG_OK) return s;
  MAG_CUDA(cudaStreamSynchronize(cudaStreamPerThread));
  *out = p.release();
  return MAG_OK;
}

MAG_API void mag_prepared_destroy(mag_prepared* p) { delete p; }

MAG_API mag_status mag_prepared_copy_codes(const mag_prepared* p, uint32_t* out, size_t count) {
  if (!p || (!out && count)) return fail(MAG_ERR_NULL_ARGUMENT, "NULL argument");
  const uint64_t nq = p->engine->plan.sp.q ? p->len / p->engine->plan.sp.q : 0;
  if (!p->d_codes) return fail(MAG_ERR_INVALID_ARGUMENT, "prepared text has no gram codes (not smag)");
  if (count > nq) return fail(MAG_ERR_OUT_OF_RANGE, "count exceeds n/q");
  cudaSetDevice(p->engine->device);
  MAG_CUDA(cudaMemcpy(out, p->d_codes, count * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return MAG_OK;
}

MAG_API mag_status mag_search_prepared_async(const mag_engine* e, const mag_prepared* p,
                                             void* stream, mag_matches** out) {
  if (!e || !p || !out) return fail(MAG_ERR_NULL_ARGUMENT, "NULL argument");
  *out = nullptr;
  if (p->engine != e) return fail(MAG_ERR_INVALID_ARGUMENT, "prepared text belongs to another engine");
  mag_status s = device_guard(e);
  if (s != MAG_OK) return s;
  try {
    auto m = std::make_unique<mag_matches>();
    m->engine = e;
    m->ws = acquire(e);
    m->stream = static_cast<cudaStream_t>(stream);
    m->d_text = p->d_text;
    m->d_codes = p->d_codes;
    m->n = p->len;
    if (m->ws->done) MAG_CUDA(cudaStreamWaitEvent(m->stream, m->ws->done, 0));
    const uint64_t slices = geometry(e, p->len, 1).num_slices;
    s = enqueue_search(e, m->ws.get(), p->d_text, p->len, p->d_codes, m->stream,
                       {SliceRange{0, slices, nullptr}});
    if (s != MAG_OK) return s;
    m->pending = true;
    *out = m.release();
    return MAG_OK;
  } catch (const std::bad_alloc&) {
    return fail(MAG_ERR_NO_MEMORY, "out of host memory");
  }
}

MAG_API mag_status mag_search_prepared(const mag_engine* e, const mag_prepared* p,
                                       mag_matches** out) {
  mag_matches* m = nullptr;
  mag_status s = mag_search_prepared_async(e, p, cudaStreamPerThread, &m);
  if (s != MAG_OK) return s;
  s = materialize(m);
  if (s != MAG_OK) {
    delete m;
    return s;
  }
  *out = m;
  return MAG_OK;
}

// prepare + search with the host->device copy pipelined against the scan:
// the text goes up in chunks on a copy stream and each scan launch covers
// the tiles whose bytes (and halo) have arrived.
MAG_API mag_status mag_search(const mag_engine* e, const uint8_t* text, size_t len,
                              mag_matches** out) {
  if (!e || !out || (!text && len)) return fail(MAG_ERR_NULL_ARGUMENT, "NULL argument");
  *out = nullptr;
  if (len >= kMaxText) return fail(MAG_ERR_INVALID_ARGUMENT, "text longer than 2^40 bytes");
  mag_status s = device_guard(e);
  if (s != MAG_OK) return s;
  if (e->plan.sp.smag) {
    // SMAG needs the whole text encoded first (prepare).
    mag_prepared* p = nullptr;
    s = mag_prepare_text(e, text, len, &p);
    if (s != MAG_OK) return s;
    s = mag_search_prepared(e, p, out);
    mag_prepared_destroy(p);
    return s;
  }
  try {
    auto m = std::make_unique<mag_matches>();
    m->engine = e;
    m->ws = acquire(e);
    Workspace* w = m->ws.get();
    cudaStream_t st = cudaStreamPerThread;
    m->stream = st;
    m->n = len;
    if (w->done) MAG_CUDA(cudaStreamWaitEvent(st, w->done, 0));
    if (w->text_cap < len + 64) {
      if (w->text) MAG_CUDA(cudaFree(w->text));
      w->text = nullptr;
      MAG_CUDA(cudaMalloc(&w->text, align16(len) + 64));
      w->text_cap = align16(len) + 64;
    }
    if (!w->copy_stream) MAG_CUDA(cudaStreamCreateWithFlags(&w->copy_stream, cudaStreamNonBlocking));
    // the copy stream must not overwrite text a previous search still reads
    if (w->done) MAG_CUDA(cudaStreamWaitEvent(w->copy_stream, w->done, 0));
    const Plan& P = e->plan;
    const SearchGeometry sg = geometry(e, len, 1);
    const uint64_t slices = sg.num_slices;
    // bytes past a slice's last sample that its scan may read: the staged
    // halo, and verification compares of whole patterns (global reads up to
    // a + maxlen + 32, a up to a sample width past the slice end)
    const uint64_t reach = static_cast<uint64_t>(P.back) + e->pd.maxlen +
                           2 * std::max<uint64_t>(16, sg.bps) + 96;
    const uint64_t chunk = std::max<uint64_t>(uint64_t(64) << 20, (len + 31) / 32);
    std::vector<SliceRange> ranges;
    uint64_t copied = 0, slices_done = 0;
    size_t ci = 0;
    while (copied < len) {
      const uint64_t nb = std::min<uint64_t>(chunk, len - copied);
      MAG_CUDA(cudaMemcpyAsync(w->text + copied, text + copied, nb, cudaMemcpyHostToDevice,
                               w->copy_stream));
      copied += nb;
      if (w->chunk_ev.size() <= ci) {
        cudaEvent_t ev;
        MAG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        w->chunk_ev.push_back(ev);
      }
      MAG_CUDA(cudaEventRecord(w->chunk_ev[ci], w->copy_stream));
      // slices whose bytes (plus the pattern reach) have fully arrived
      const uint64_t ready = copied == len ? slices : (copied > reach ? slices_ending_by(sg, copied - reach) : 0);
      ranges.push_back(SliceRange{slices_done, ready, w->chunk_ev[ci]});
      slices_done = std::max(slices_done, ready);
      ++ci;
    }
    m->d_text = w->text;
    s = enqueue_search(e, w, w->text, len, nullptr, st, ranges);
    if (s != MAG_OK) return s;
    m->pending = true;
    s = materialize(m.get());
    if (s != MAG_OK) return s;
    *out = m.release();
    return MAG_OK;
  } catch (const std::bad_alloc&) {
    return fail(MAG_ERR_NO_MEMORY, "out of host memory");
  }
}

MAG_API mag_status mag_matches_sync(mag_matches* m) {
  if (!m) return fail(MAG_ERR_NULL_ARGUMENT, "matches is NULL");
  return materialize(m);
}

MAG_API size_t mag_matches_count(const mag_matches* m) {
  if (!m) return 0;
  mag_matches* mm = const_cast<mag_matches*>(m);
  if (mm->pending) {
    mag_status s = materialize(mm);
    if (s != MAG_OK) {
      mm->sticky = s;
      mm->pending = false;
      return 0;
    }
  }
  return m->keys.size();
}

MAG_API mag_status mag_matches_get(const mag_matches* m, size_t index, uint32_t* pid,
                                   size_t* offset) {
  if (!m || !pid || !offset) return fail(MAG_ERR_NULL_ARGUMENT, "NULL argument");
  const size_t n = mag_matches_count(m);
  if (m->sticky != MAG_OK) return m->sticky;
  if (index >= n)
    return fail(MAG_ERR_OUT_OF_RANGE, "match index " + std::to_string(index) + " >= " +
                                          std::to_string(n));
  const uint64_t k = m->keys[index];
  *pid = static_cast<uint32_t>(k & ((1u << kPidBits) - 1));
  *offset = static_cast<size_t>(k >> kPidBits);
  return MAG_OK;
}

MAG_API mag_status mag_matches_copy(const mag_matches* m, uint64_t* offsets, uint32_t* pids,
                                    size_t capacity) {
  if (!m) return fail(MAG_ERR_NULL_ARGUMENT, "matches is NULL");
  const size_t n = mag_matches_count(m);
  if (m->sticky != MAG_OK) return m->sticky;
  if (capacity < n) return fail(MAG_ERR_OUT_OF_RANGE, "capacity below match count");
  for (size_t i = 0; i < n; ++i) {
    const uint64_t k = m->keys[i];
    if (offsets) offsets[i] = k >> kPidBits;
    if (pids) pids[i] = static_cast<uint32_t>(k & ((1u << kPidBits) - 1));
  }
  return MAG_OK;
}

MAG_API mag_status mag_matches_metrics(const mag_matches* m, mag_metrics* out) {
  if (!m || !out) return fail(MAG_ERR_NULL_ARGUMENT, "NULL argument");
  mag_matches_count(m);
  if (m->sticky != MAG_OK) return m->sticky;
  *out = m->metrics;
  return MAG_OK;
}

MAG_API void mag_matches_destroy(mag_matches* m) { delete m; }

MAG_API mag_status mag_tune(const mag_tuning_input* in, mag_tuning_result* out) {
  if (!in || !out) return fail(MAG_ERR_NULL_ARGUMENT, "NULL argument");
  TuningInput ti;
  ti.sigma = in->sigma;
  ti.sigma_prime = in->sigma_prime;
  ti.r = in->r;
  ti.m = in->m;
  ti.n = in->n;
  ti.word_bits = in->word_bits ? in->word_bits : 64;
  if (ti.r == 0 || ti.m == 0 || ti.sigma == 0)
    return fail(MAG_ERR_INVALID_ARGUMENT, "sigma, r and m must be >= 1");
  if (ti.word_bits > 64) return fail(MAG_ERR_BAD_CONFIG, "word_bits must be <= 64");
  TuningResult tr;
  std::string err;
  if (!tune(ti, 0, 0, &tr, &err)) return fail(MAG_ERR_BAD_CONFIG, err);
  out->q = static_cast<int>(tr.q);
  out->k = static_cast<int>(tr.k);
  out->sigma_prime = static_cast<int>(tr.sigma_prime);
  out->rho = tr.rho;
  out->predicted_p = tr.predicted_p;
  out->predicted_cost = tr.predicted_cost;
  return MAG_OK;
}

MAG_API mag_status mag_sample_patterns(const uint8_t* corpus, size_t corpus_len, size_t count,
                                       size_t length, uint64_t seed, mag_patterns** out) {
  if (!out || (!corpus && corpus_len)) return fail(MAG_ERR_NULL_ARGUMENT, "NULL argument");
  *out = nullptr;
  if (length == 0) return fail(MAG_ERR_INVALID_ARGUMENT, "pattern length must be >= 1");
  if (length > corpus_len)
    return fail(MAG_ERR_INVALID_ARGUMENT, "pattern length exceeds the corpus");
  try {
    auto p = std::make_unique<mag_patterns>();
    std::vector<uint64_t> offs;
    sample_offsets(corpus_len, count, length, seed, &offs);
    p->items.reserve(count);
    for (uint64_t o : offs) p->items.emplace_back(corpus + o, corpus + o + length);
    *out = p.release();
    return MAG_OK;
  } catch (const std::bad_alloc&) {
    return fail(MAG_ERR_NO_MEMORY, "out of host memory");
  }
}

MAG_API size_t mag_patterns_count(const mag_patterns* p) { return p ? p->items.size() : 0; }

MAG_API mag_status mag_patterns_get(const mag_patterns* p, size_t index, const uint8_t** bytes,
                                    size_t* len) {
  if (!p || !bytes || !len) return fail(MAG_ERR_NULL_ARGUMENT, "NULL argument");
  if (index >= p->items.size()) return fail(MAG_ERR_OUT_OF_RANGE, "pattern index out of range");
  *bytes = p->items[index].data();
  *len = p->items[index].size();
  return MAG_OK;
}

MAG_API void mag_patterns_destroy(mag_patterns* p) { delete p; }

MAG_API const char* mag_status_string(mag_status s) {
  switch (s) {
    case MAG_OK: return "ok";
    case MAG_ERR_NULL_ARGUMENT: return "null argument";
    case MAG_ERR_INVALID_ARGUMENT: return "invalid argument";
    case MAG_ERR_EMPTY_PATTERN_SET: return "empty pattern set";
    case MAG_ERR_EMPTY_PATTERN: return "empty pattern";
    case MAG_ERR_BAD_CONFIG: return "bad configuration";
    case MAG_ERR_OUT_OF_RANGE: return "out of range";
    case MAG_ERR_NO_MEMORY: return "out of memory";
    case MAG_ERR_INTERNAL: return "internal error";
  }
  return "unknown status";
}

MAG_API const char* mag_last_error(void) { return tl_error.c_str(); }

MAG_API const char* mag_version(void) { return "mag-b200 0.1.0 (sm_100a)"; }

MAG_API uint64_t mag_kernel_launches(void) { return kernel_launch_count(); }

MAG_API void mag_scan_timer_enable(int on) {
  std::lock_guard<std::mutex> g(g_timer.mu);
  g_timer.on = on != 0;
  g_timer.scan_only = on == 2;
  g_timer.total_ms = 0;
  g_timer.launches = 0;
  for (auto& ev : g_timer.pending) g_timer.spare.push_back(ev);
  g_timer.pending.clear();
}

MAG_API mag_status mag_scan_timer_read(double* total_ms, uint64_t* launches) {
  if (!total_ms || !launches) return fail(MAG_ERR_NULL_ARGUMENT, "NULL argument");
  std::lock_guard<std::mutex> g(g_timer.mu);
  for (auto& ev : g_timer.pending) {
    MAG_CUDA(cudaEventSynchronize(ev.second));
    float ms = 0;
    MAG_CUDA(cudaEventElapsedTime(&ms, ev.first, ev.second));
    g_timer.total_ms += ms;
    g_timer.launches++;
    g_timer.spare.push_back(ev);
  }
  g_timer.pending.clear();
  *total_ms = g_timer.total_ms;
  *launches = g_timer.launches;
  return MAG_OK;
}

}  // extern "C"
