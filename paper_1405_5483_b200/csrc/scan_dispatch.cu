// Kernel-family dispatch, the SMAG prepare kernel and launch bookkeeping.
#include <atomic>
#include <mutex>
#include <map>
#include <utility>

#include "kern_common.cuh"

namespace magb {
namespace {

std::atomic<unsigned long long> g_launches{0};

// The finish grid: places every slice's staged matches at its final
// offset once the search's scan grid has completed (griddepcontrol.wait: it
// is launched as the scan's programmatic dependent, so its CTAs are resident
// and waiting as the scan's CTAs leave).  CTA b owns groups [g0, g1): the
// sum of the group sums before g0 (a coalesced pass over at most a few
// thousand words) and a block scan of its own give each group's base; a warp
// per group scans the group's 32 slice counts and copies the group's matches
// as one flat run, 16 loads in flight per lane.  The CTA of the last groups
// publishes the counters and clears the next search's control words.
constexpr int kFinishThreads = 512;
__global__ void __launch_bounds__(kFinishThreads) mag_finish_kernel(const __grid_constant__ ScanArgs A) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) diag_time(A, 2, true);
  __shared__ unsigned long long red[kFinishThreads / 32];
  __shared__ unsigned long long s_base[kFinishThreads];  // inclusive sums of the owned groups (this chunk)
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int kW = kFinishThreads / 32;
  const uint64_t G = (A.num_slices + kGroup - 1) / kGroup;
  const uint64_t g0 = blockIdx.x * G / gridDim.x, g1 = (blockIdx.x + 1) * G / gridDim.x;
  // clear the other half of the group sums for the next search
  for (uint64_t i = blockIdx.x * kFinishThreads + tid; i < A.group_sum_words; i += uint64_t(gridDim.x) * kFinishThreads)
    A.group_sum_next[i] = 0;
  // Requested before the prefix is known (independent loads, one round trip
  // together with the prefix's): the first chunk's group sums and this warp's
  // first group's slice counts.
  const unsigned long long gs_first = g0 + tid < g1 ? A.group_sum[g0 + tid] : 0ull;
  uint32_t cnt_first = 0;
  if (g0 + wid < g1) {
    const uint64_t x = (g0 + wid) * kGroup + lane;
    cnt_first = x < A.num_slices ? A.slice_count[x] : 0u;
  }
  // matches before g0
  unsigned long long acc = 0;
  for (uint64_t i = tid; i < g0; i += kFinishThreads) acc += A.group_sum[i];
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
  if (lane == 0) red[wid] = acc;
  __syncthreads();
  unsigned long long base = 0;
  for (int w = 0; w < kW; ++w) base += red[w];
  __syncthreads();
  for (uint64_t c0 = g0; c0 < g1; c0 += kFinishThreads) {
    // block scan of this chunk's group sums
    const uint64_t g = c0 + tid;
    const unsigned long long gs = c0 == g0 ? gs_first : (g < g1 ? A.group_sum[g] : 0ull);
    unsigned long long v = gs;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(kFull, v, o);
      if (lane >= o) v += y;
    }
    if (lane == 31) red[wid] = v;
    __syncthreads();
    unsigned long long wbase = 0;
    for (int w = 0; w < wid; ++w) wbase += red[w];
    unsigned long long ctot = 0;
    for (int w = 0; w < kW; ++w) ctot += red[w];
    s_base[tid] = base + wbase + v - gs;  // exclusive base of group g
    __syncthreads();
    // a warp per group: slice counts -> offsets -> flat copy
    const uint64_t nchunk = g1 - c0 < kFinishThreads ? g1 - c0 : kFinishThreads;
    for (uint64_t k = wid; k < nchunk; k += kW) {
      const uint64_t grp = c0 + k;
      const unsigned long long gb = s_base[k];
      const uint64_t x = grp * kGroup + lane;
      const uint32_t cnt = (c0 == g0 && k == static_cast<uint64_t>(wid)) ? cnt_first
                                                                         : (x < A.num_slices ? A.slice_count[x] : 0u);
      uint32_t u = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, u, o);
        if (lane >= o) u += y;
      }
      const uint32_t excl = u - cnt, tot = __shfl_sync(kFull, u, 31);
      if (!tot) continue;
      constexpr int kU = 16;  // loads in flight per lane (8 -> 16: cfg5 finish 0.15 -> ? ms)
      if (!__any_sync(kFull, cnt > A.slice_cap)) {
        // element e belongs to the last slice whose exclusive prefix is <= e
        for (uint32_t e0 = 0; e0 < tot; e0 += 32 * kU) {
          uint64_t val[kU];
#pragma unroll
          for (int j = 0; j < kU; ++j) {
            const uint32_t e = e0 + 32 * j + lane;
            int sl = 0;
#pragma unroll
            for (int step = 16; step; step >>= 1) {
              const uint32_t t = __shfl_sync(kFull, excl, sl + step);
              if (t <= e) sl += step;
            }
            const uint32_t off = e - __shfl_sync(kFull, excl, sl);
            val[j] = e < tot ? A.staging[(grp * kGroup + sl) * A.slice_cap + off] : 0ull;
          }
#pragma unroll
          for (int j = 0; j < kU; ++j) {
            const uint32_t e = e0 + 32 * j + lane;
            if (e < tot && gb + e < A.out_cap) A.out[gb + e] = val[j];
          }
        }
      } else {
        // a slice overflowed its staging (the host searches again with a
        // larger capacity): copy what fits, slice by slice
        for (unsigned m = __ballot_sync(kFull, cnt != 0); m; m &= m - 1) {
          const int sl = __ffs(m) - 1;
          const uint32_t n = __shfl_sync(kFull, cnt, sl);
          const unsigned long long dst = gb + __shfl_sync(kFull, excl, sl);
          const uint32_t cc = n < A.slice_cap ? n : A.slice_cap;
          const uint64_t* src = A.staging + (grp * kGroup + sl) * A.slice_cap;
          for (uint32_t i = lane; i < cc; i += 32)
            if (dst + i < A.out_cap) A.out[dst + i] = src[i];
        }
      }
    }
    base += ctot;
    __syncthreads();
  }
  // The CTA of the last groups knows the total.  It publishes the counters
  // and clears the NEXT search's control words (the other parity half, which
  // no CTA of this search reads), so it need not wait for the other CTAs:
  // the kernel's completion orders everything before the next search.
  if (blockIdx.x != gridDim.x - 1) return;
  if (tid == 0) {
    const volatile unsigned long long* c = A.counters;
    volatile unsigned long long* h = A.host_ctr;
    h[1] = c[kCtrCands];
    h[2] = base;
    h[3] = c[kCtrMax];
  }
  if ((A.plan.diag & 2048) && tid < 4) {  // diagnostics timeline
    const volatile unsigned long long* c = A.counters;
    const uint64_t t0 = ~c[kCtrTime];
    const uint64_t t = tid == 2 ? global_ns() : (tid == 1 ? ~c[kCtrTime + 2] : c[kCtrTime + 1 + tid]);
    A.host_ctr[4 + tid] = t - t0;
  }
  for (uint32_t i = tid; i < A.reset_words; i += kFinishThreads) A.reset[i] = 0;
}

// SMAG prepare (encode_text qgram.cpp:29-37) on the device.
__global__ void mag_encode_kernel(const ScanPlan P, const uint8_t* __restrict__ text, uint64_t nq,
                                  const uint8_t* __restrict__ map, uint32_t* __restrict__ codes) {
  __shared__ uint8_t smap[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) smap[i] = map ? map[i] : 0;
  __syncthreads();
  const uint32_t q = P.q;
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < nq; u += (uint64_t)gridDim.x * blockDim.x) {
    const uint8_t* g = text + u * q;
    uint32_t v;
    if (P.gram_mode == kGramExact) {
      v = smap[g[q - 1]];
      for (int i = static_cast<int>(q) - 2; i >= 0; --i) v = v * P.sigma_prime + smap[g[i]];
    } else {
      uint32_t x[4] = {0, 0, 0, 0};
      for (uint32_t i = 0; i < q; ++i) x[i >> 2] |= static_cast<uint32_t>(g[i]) << (8 * (i & 3));
      v = gram_slot(hash_gram_words(x[0], x[1], x[2], x[3]), P.table_bits);
    }
    codes[u] = v;
  }
}

}  // namespace

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

unsigned long long kernel_launch_count() { return g_launches.load(); }

cudaError_t allow_max_smem(const void* kernel, size_t need) {
  // The limit only ever grows to what a launch needs (not the device's
  // opt-in maximum): the driver sizes the shared-memory carveout, hence what
  // is left for L1, from it.
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> set;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  size_t& cur = set[{kernel, dev}];
  if (cur >= need) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(need));
  if (e != cudaSuccess) return e;
  cur = need;
  return cudaSuccess;
}

namespace {
cudaError_t launch_scan_only(const ScanArgs& a, cudaStream_t stream, int grid) {
  if (a.plan.direct) return launch_direct(a, stream, grid);
  if (a.plan.roll) return launch_roll(a, stream, grid);
  if (a.plan.pack2) return launch_pack2(a, stream, grid);
  if (a.plan.smag) return launch_staged_codes(a, stream, grid);
  if (a.plan.gram_mode == kGramHashed) return launch_staged_hashed(a, stream, grid);
  return launch_staged_exact(a, stream, grid);
}
}  // namespace

cudaError_t launch_scan(const ScanArgs& a, cudaStream_t stream, int grid, cudaEvent_t after_scan) {
  cudaError_t e = launch_scan_only(a, stream, grid);
  if (after_scan) cudaEventRecord(after_scan, stream);
  if (e != cudaSuccess || !a.final_launch) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.finish_grid);
  cfg.blockDim = dim3(kFinishThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, mag_finish_kernel, a);
  if (e != cudaSuccess) return e;
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_encode(const ScanPlan& plan, const uint8_t* text, uint64_t n, const uint8_t* map,
                          uint32_t* codes, cudaStream_t stream) {
  const uint64_t nq = n / plan.q;
  if (nq == 0) return cudaSuccess;
  const int threads = 256;
  uint64_t blocks = (nq + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  (void)cudaGetLastError();
  mag_encode_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(plan, text, nq, map, codes);
  count_launch();
  return cudaGetLastError();
}

}  // namespace magb
