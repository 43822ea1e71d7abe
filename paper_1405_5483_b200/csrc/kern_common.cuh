// Device helpers shared by the scan kernels (scan_staged.cuh, scan_direct.cu,
// scan_roll.cu): PTX wrappers (mbarrier, 1-D TMA bulk copies, L2 policy),
// warp scans, exact compares against the text, the window-key bucket walk,
// and the in-kernel ordered gather (slice publication, gather warp, exit).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "scan_launch.h"

namespace magb {
namespace {

constexpr unsigned kFull = 0xffffffffu;

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "MAG_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra MAG_WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// Text is read once: stream it through L2 with an evict-first policy so it
// does not push the pattern tables and the screen bitmap out of L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_1d_stream(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                                   uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, int lane) {
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  return x - v;
}

// Coherent (L2) 64-bit load/store for words other warps write in this launch.
__device__ __forceinline__ uint64_t ld_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Fences at GPU scope.  An acquire (fence.acq_rel, ld.acquire) invalidates the
// SM's whole L1 (CCTL.IVALL), which the scanning warps' screen and pattern
// loads rely on: the scanning warps only ever release (MEMBAR, no IVALL);
// the gather warps acquire once per lock or copy claim.
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_release() { asm volatile("fence.release.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Exact compare of pattern pid against text[a, a + len) in global memory:
// 16 pattern bytes at a time against two aligned 16-byte text loads
// (independent, one round trip per piece) realigned with funnel shifts.
__device__ __forceinline__ uint32_t fsr(uint32_t lo, uint32_t hi, uint32_t b) { return __funnelshift_r(lo, hi, b); }
__device__ bool equal_text(const ScanArgs& A, unsigned long long a, uint32_t pid, uint32_t len) {
  const uint8_t* p = A.pat_bytes + __ldg(A.pat_off + pid);
  if (a + len + 32 > A.n) {  // near the end of the text: bytewise (no over-read)
    const uint8_t* t = A.text + a;
    for (uint32_t i = 0; i < len; ++i)
      if (__ldg(t + i) != __ldg(p + i)) return false;
    return true;
  }
  for (uint32_t i = 0; i < len; i += 16) {
    const unsigned long long x = a + i;
    const uint4* c = reinterpret_cast<const uint4*>(A.text + (x & ~15ull));
    const uint4 t0 = __ldg(c), t1 = __ldg(c + 1);
    const uint4 pv = __ldg(reinterpret_cast<const uint4*>(p + i));
    const uint32_t sh = static_cast<uint32_t>(x & 15), b = (sh & 3u) * 8u;
    uint32_t w0, w1, w2, w3, w4;
    switch (sh >> 2) {
      case 0: w0 = t0.x; w1 = t0.y; w2 = t0.z; w3 = t0.w; w4 = t1.x; break;
      case 1: w0 = t0.y; w1 = t0.z; w2 = t0.w; w3 = t1.x; w4 = t1.y; break;
      case 2: w0 = t0.z; w1 = t0.w; w2 = t1.x; w3 = t1.y; w4 = t1.z; break;
      default: w0 = t0.w; w1 = t1.x; w2 = t1.y; w3 = t1.z; w4 = t1.w; break;
    }
    const uint32_t rem = len - i;  // bytes of this piece that count
    const uint32_t d0 = fsr(w0, w1, b) ^ pv.x, d1 = fsr(w1, w2, b) ^ pv.y;
    const uint32_t d2 = fsr(w2, w3, b) ^ pv.z, d3 = fsr(w3, w4, b) ^ pv.w;
    auto keep = [&](uint32_t word) -> uint32_t {
      const uint32_t lo = 4u * word;
      if (rem >= lo + 4) return 0xffffffffu;
      if (rem <= lo) return 0u;
      return (1u << (8 * (rem - lo))) - 1u;
    };
    if ((d0 & keep(0)) | (d1 & keep(1)) | (d2 & keep(2)) | (d3 & keep(3))) return false;
  }
  return true;
}

// Window-key bucket walk: a candidate window's key (read at its gram
// boundary a0) against the (pattern, shift) index; entry shift s names the
// start a0 - s.  Entries come in (shift descending, pattern ascending) order
// = text order.  Counted, or written (dst != nullptr) from dst[idx].
__device__ uint32_t window_probe(const ScanArgs& A, unsigned long long a0, uint32_t key, uint64_t* dst,
                                 uint32_t idx) {
  const uint32_t b = key & ((1u << A.plan.bucket_bits) - 1u);
  const uint32_t lo = __ldg(A.bucket_start + b), hi = __ldg(A.bucket_start + b + 1);
  uint32_t c = 0;
  for (uint32_t e = lo; e < hi; ++e) {
    const uint2 ent = __ldg(A.bucket_entries + e);
    if (ent.x != key) continue;
    const uint32_t s = ent.y >> kPidBits, pid = ent.y & ((1u << kPidBits) - 1u);
    if (s > a0) continue;
    const unsigned long long a = a0 - s;
    const uint32_t len = __ldg(A.pat_len + pid);
    if (a + len > A.n || !equal_text(A, a, pid, len)) continue;
    if (dst && idx + c < A.slice_cap) dst[idx + c] = pack_match(a, pid);
    ++c;
  }
  return c;
}

// Screen + verify a probe queue {key, start - pbase} (staged and direct
// kernels).  Keys are screened 4 per lane (independent L2 loads, one round
// trip per 128); the survivors — true matches and ~0.5% strays — are
// compacted in queue order (reusing the queue's own storage) so each
// bucket-walk round serves up to 32 of them.  Output is ordered: queue order
// = text order.
__device__ __noinline__ uint32_t flush_queue(const ScanArgs& A, uint2* pq, uint32_t pqn, unsigned long long pbase,
                                             uint64_t* out, uint32_t fill, int lane, bool screened) {
  __syncwarp();
  const uint32_t lb = A.plan.l2_bits;
  uint32_t nlive = screened ? pqn : 0;
  for (uint32_t b0 = 0; !screened && b0 < pqn; b0 += 4 * 32) {
    const uint32_t i0 = b0 + 4 * lane;
    uint2 e[4];
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      e[j] = i0 + j < pqn ? pq[i0 + j] : make_uint2(0u, 0xffffffffu);
      w[j] = ~0u;
      if (lb && e[j].y != 0xffffffffu) w[j] = __ldg(A.l2map + (screen_bit(e[j].x, lb) >> 5));
    }
    uint32_t live = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (e[j].y != 0xffffffffu && (!lb || ((w[j] >> (screen_bit(e[j].x, lb) & 31u)) & 1u))) live |= 1u << j;
    const uint32_t cnt = __popc(live);
    const uint32_t excl = warp_excl_scan(cnt, lane);
    const uint32_t total = __shfl_sync(kFull, excl + cnt, 31);
    __syncwarp();
    uint32_t r = nlive + excl;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (live & (1u << j)) pq[r++] = e[j];
    __syncwarp();
    nlive += total;
  }
  for (uint32_t i0 = 0; i0 < nlive; i0 += 32) {
    const uint32_t i = i0 + lane;
    uint2 e = make_uint2(0u, 0xffffffffu);
    uint32_t c = 0;
    if (i < nlive) {
      e = pq[i];
      c = window_probe(A, pbase + e.y, e.x, nullptr, 0);
    }
    if (!__any_sync(kFull, c != 0)) continue;
    const uint32_t excl = warp_excl_scan(c, lane);
    const uint32_t total = __shfl_sync(kFull, excl + c, 31);
    if (c) window_probe(A, pbase + e.y, e.x, out, fill + excl);
    fill += total;
  }
  __syncwarp();
  return fill;
}

// ------------------------------------------------------------ ordered gather
// Slice end (whole warp): the slice's staged matches and its count become
// visible before its group word says "one more slice done".  slice_count is
// zero between searches (the copier clears it), so an empty slice stores
// nothing and needs no fence (a fence waits ~1 us for the store
// acknowledgements; most slices of a sparse search are empty).  The largest
// slice count (staging overflow check, learned density) is a fire-and-forget
// reduction.
__device__ __forceinline__ void publish_slice(const ScanArgs& A, uint64_t slice, uint32_t count, int lane) {
  if (A.plan.diag & 512) return;  // diagnostics: no publication (no gather)
  if (count) {
    if (lane == 0) A.slice_count[slice] = count;
    fence_release();  // every lane's staged matches (and the count) before the group word
  }
  __syncwarp();
  if (lane == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(A.group_word + slice / kGroup), (1ull << 40) | count);
    if (count) atomicMax(A.counters + kCtrMax, static_cast<unsigned long long>(count));
  }
  __syncwarp();
}

// Diagnostics builds (MAG_B200_DIAG bit 2048): a timeline of the search in
// spare control words, ns since the first scan CTA started (the host prints
// it): [kCtrTime] ~first scan start, +1 last scan warp end, +2 watermark at
// the end, +3 last gather warp exit, +4 last gather warp start.
constexpr unsigned kCtrTime = 56;
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void diag_time(const ScanArgs& A, unsigned slot) {
  if (!(A.plan.diag & 2048)) return;
  const uint64_t t = global_ns();
  atomicMax(A.counters + kCtrTime + slot, static_cast<unsigned long long>(slot == 0 ? ~t : t));
}

// A scanning warp leaves the kernel: its candidate count joins the counters.
__device__ __forceinline__ void scan_exit(const ScanArgs& A, unsigned long long cands, int lane) {
#pragma unroll
  for (int o = 16; o; o >>= 1) cands += __shfl_xor_sync(kFull, cands, o);
  if (lane == 0 && cands) atomicAdd(A.counters + kCtrCands, cands);
  if (lane == 0) diag_time(A, 1);
}

// Let the search's gather kernel start now (programmatic dependent launch):
// its one-warp CTAs run beside the scan on the registers a 15-warp CTA
// leaves free, and place slices while the scan goes on.
__device__ __forceinline__ void allow_gather(const ScanArgs& A) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) diag_time(A, 0);
}

// Watermark advance (one gather warp at a time, under the advance lock):
// lane l takes the 32 groups W + 32 l ... W + 32 l + 31, so the run of
// complete groups right above W (up to 1024 groups = 32768 slices) is found
// and prefix-summed with per-lane serial sums and one warp scan; the
// inclusive prefix counts go to group_incl[] and the new watermark is stored
// after them.  Returns the new W (groups).
__device__ __forceinline__ uint64_t advance_watermark(const ScanArgs& A, uint64_t W, uint64_t gend, int lane) {
  constexpr int kPer = 32;
  const uint64_t g0 = W + static_cast<uint64_t>(kPer) * lane;
  uint64_t wd[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) wd[i] = g0 + i < gend ? ld_gpu(A.group_word + g0 + i) : 0ull;
  const unsigned long long base = W == 0 ? 0ull : ld_gpu(A.group_incl + W - 1);
  int lead = kPer;
#pragma unroll
  for (int i = kPer - 1; i >= 0; --i) {
    const uint64_t g = g0 + i;
    const uint64_t want = g < gend ? min(static_cast<uint64_t>(kGroup), A.num_slices - g * kGroup) : ~0ull;
    if ((wd[i] >> 40) != want) lead = i;
  }
  unsigned long long sum = 0;
#pragma unroll
  for (int i = 0; i < kPer; ++i)
    if (i < lead) sum += wd[i] & ((1ull << 40) - 1);
  const unsigned partial = __ballot_sync(kFull, lead < kPer);
  const int stop = partial ? __ffs(partial) - 1 : 32;
  if (lane > stop) {
    lead = 0;
    sum = 0;
  }
  const uint64_t j = static_cast<uint64_t>(kPer) * stop + (stop < 32 ? __shfl_sync(kFull, lead, stop) : 0);
  if (j == 0) return W;
  unsigned long long v = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += y;
  }
  const unsigned long long end = base + __shfl_sync(kFull, v, 31);
  unsigned long long run = base + v - sum;
#pragma unroll
  for (int i = 0; i < kPer; ++i)
    if (i < lead) {
      run += wd[i] & ((1ull << 40) - 1);
      st_gpu(A.group_incl + g0 + i, run);
    }
  W += j;
  fence_release();  // every lane's prefix stores before the new watermark
  __syncwarp();
  if (lane == 0) {
    if (W * kGroup >= A.num_slices) st_gpu(reinterpret_cast<uint64_t*>(A.counters) + kCtrTotal, end);
    fence_release();
    st_gpu(reinterpret_cast<uint64_t*>(A.counters) + kCtrWatermark, W);
  }
  __syncwarp();
  return W;
}

// Place group c (below the watermark): its slices' offsets are the group's
// exclusive prefix plus a warp scan of their counts; copy their staged
// matches; clear the group word for the next search.
__device__ __forceinline__ void copy_group(const ScanArgs& A, uint64_t c, int lane) {
  const uint64_t x = c * kGroup + lane;
  const unsigned long long base = c == 0 ? 0ull : ld_gpu(A.group_incl + c - 1);
  const uint32_t cnt = x < A.num_slices ? __ldcg(A.slice_count + x) : 0u;
  unsigned long long v = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += y;
  }
  const unsigned long long mine = base + v - cnt;
  constexpr int kU = 8;  // loads in flight per lane
  if (!__any_sync(kFull, cnt > A.slice_cap)) {
    // the group's matches as one flat run: element e belongs to the last
    // slice whose exclusive prefix is <= e (binary search over the lanes)
    const uint32_t excl = static_cast<uint32_t>(v) - cnt;
    const uint32_t tot = static_cast<uint32_t>(__shfl_sync(kFull, v, 31));
    for (uint32_t e0 = 0; e0 < tot; e0 += 32 * kU) {
      uint64_t val[kU];
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        const uint32_t e = e0 + 32 * k + lane;
        int sl = 0;
#pragma unroll
        for (int step = 16; step; step >>= 1) {
          const uint32_t t = __shfl_sync(kFull, excl, sl + step);
          if (t <= e) sl += step;
        }
        const uint32_t off = e - __shfl_sync(kFull, excl, sl);
        val[k] = e < tot ? __ldcg(A.staging + (c * kGroup + sl) * A.slice_cap + off) : 0ull;
      }
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        const uint32_t e = e0 + 32 * k + lane;
        if (e < tot && base + e < A.out_cap) A.out[base + e] = val[k];
      }
    }
  } else {
    // a slice overflowed its staging (the host searches again with a larger
    // capacity): copy what fits, slice by slice
    for (unsigned m = __ballot_sync(kFull, cnt != 0); m; m &= m - 1) {
      const int sl = __ffs(m) - 1;
      const uint32_t n = __shfl_sync(kFull, cnt, sl);
      const unsigned long long dst = __shfl_sync(kFull, mine, sl);
      const uint32_t cc = n < A.slice_cap ? n : A.slice_cap;
      const uint64_t* src = A.staging + (c * kGroup + sl) * A.slice_cap;
      for (uint32_t i = lane; i < cc; i += 32)
        if (dst + i < A.out_cap) A.out[dst + i] = __ldcg(src + i);
    }
  }
  // zero between searches: the group word and the nonzero slice counts
  if (cnt) A.slice_count[x] = 0;
  if (lane == 0) st_gpu(A.group_word + c, 0ull);
}

// A gather warp (scan_dispatch.cu mag_gather_kernel: one per CTA, grid
// beside the scan).  Two jobs: advancing the watermark (the warp that takes
// the advance lock keeps advancing while groups complete), and copying: each
// gather warp claims one group at a time (a cursor per launch) and places it
// once the watermark has passed it.  The scan never waits for the gather, and
// the gather only waits for slices the scan's running warps have claimed, so
// nothing can deadlock whether or not the two grids are co-resident.
__device__ __noinline__ void gather_warp_run(const ScanArgs& A, int lane) {
  if (lane == 0) diag_time(A, 4);
  if (A.plan.diag & 256) return;  // diagnostics: no gather warp
  unsigned long long* lock = A.counters + kCtrLock;
  const uint64_t gbeg = A.slice_begin / kGroup;
  const uint64_t gend = (A.slice_end + kGroup - 1) / kGroup;  // launches end on group boundaries
  uint64_t claim = ~0ull;
  bool claims_done = false, advancer = false;
  uint32_t idle = 0;
  while (true) {
    uint64_t W = ld_gpu(reinterpret_cast<const uint64_t*>(A.counters) + kCtrWatermark);
    bool progress = false;
    bool ready = false;  // the lock is only tried when the group at the watermark is complete
    if (lane == 0 && !advancer && W < gend)
      ready = (ld_gpu(A.group_word + W) >> 40) == min(static_cast<uint64_t>(kGroup), A.num_slices - W * kGroup);
    if (!advancer && __shfl_sync(kFull, ready, 0)) {
      unsigned long long got = 1;
      if (lane == 0) got = atomicCAS(lock, 0ull, 1ull);
      got = __shfl_sync(kFull, got, 0);
      if (got == 0) {
        // this warp is the advancer until the launch's last group: it polls
        // the group words itself (one warp spinning on one SM), so the
        // watermark follows the scan by about one poll
        fence_gpu();
        W = ld_gpu(reinterpret_cast<const uint64_t*>(A.counters) + kCtrWatermark);
        uint32_t spins = 0;
        while (W < gend) {
          bool next = false;  // the group at W complete?  (one load before a full advance)
          if (lane == 0)
            next = (ld_gpu(A.group_word + W) >> 40) == min(static_cast<uint64_t>(kGroup), A.num_slices - W * kGroup);
          const uint64_t W2 = __shfl_sync(kFull, next, 0) ? advance_watermark(A, W, gend, lane) : W;
          if (W2 == W) {
            __nanosleep(spins < 64 ? 32 : 128);
            ++spins;
          } else {
            spins = 0;
            progress = true;
            W = W2;
            // place a claimed group as soon as the watermark passes it
            if (claim != ~0ull && claim < W) {
              fence_gpu();
              copy_group(A, claim, lane);
              claim = ~0ull;
            }
          }
        }
        if (lane == 0) diag_time(A, 2);
        if (lane == 0) {  // the next launch of the search needs the lock
          fence_release();
          atomicExch(lock, 0ull);
        }
      } else {
        advancer = true;  // someone else holds the advance for this launch
      }
    }
    if (!claims_done && claim == ~0ull) {
      unsigned long long c = 0;
      if (lane == 0) c = atomicAdd(A.copy_cursor, 1ull);
      c = __shfl_sync(kFull, c, 0) + gbeg;
      if (c >= gend)
        claims_done = true;
      else
        claim = c;
    }
    if (claim != ~0ull && claim < W) {
      fence_gpu();
      copy_group(A, claim, lane);
      claim = ~0ull;
      progress = true;
    }
    if (claims_done && claim == ~0ull && W >= gend) break;
    if (progress) {
      idle = 0;
    } else {
      __nanosleep(idle < 16 ? 64 : 200);
      ++idle;
    }
  }
}

}  // namespace
}  // namespace magb
