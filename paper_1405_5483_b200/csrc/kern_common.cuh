// Device helpers shared by the scan kernels (scan_staged.cuh, scan_direct.cu,
// scan_roll.cu): PTX wrappers (mbarrier, 1-D TMA bulk copies, L2 policy),
// warp scans, exact compares against the text, the window-key bucket walk,
// and the slice publication the finish grid reads (scan_dispatch.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "scan_launch.h"

namespace magb {
namespace {

constexpr unsigned kFull = 0xffffffffu;

// Diagnostics builds only (-DMAG_B200_DIAGNOSTICS, MAG_B200_DIAG): stage-skip
// bits of the plan; product builds compile the checks away.
#ifdef MAG_B200_DIAGNOSTICS
#define MAG_DIAG(A, bits) ((A).plan.diag & (bits))
#else
#define MAG_DIAG(A, bits) 0
#endif

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

// Exact compare of pattern pid against text[a, a + len) in global memory:
// 16 pattern bytes at a time against two aligned 16-byte text loads
// (independent, one round trip per piece) realigned with funnel shifts.
__device__ __forceinline__ uint32_t fsr(uint32_t lo, uint32_t hi, uint32_t b) { return __funnelshift_r(lo, hi, b); }
__device__ bool equal_text_p(const ScanArgs& A, unsigned long long a, const uint8_t* p, uint32_t len) {
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

__device__ __forceinline__ bool equal_text(const ScanArgs& A, unsigned long long a, uint32_t pid, uint32_t len) {
  return equal_text_p(A, a, A.pat_bytes + __ldg(A.pat_off + pid), len);
}

// Window-key bucket walk: a candidate window's key (read at its gram
// boundary a0) against the (pattern, shift) index; entry shift s names the
// start a0 - s.  Entries come in (shift descending, pattern ascending) order
// = text order.  Counted (the first match kept in *first), or written
// (dst != nullptr) from dst[idx].  A pattern's length and offset are loaded
// together, so a hit costs four dependent round trips: bucket bounds, entry,
// {length, offset}, {text, pattern bytes}.
__device__ uint32_t window_probe(const ScanArgs& A, unsigned long long a0, uint32_t key, uint64_t* dst,
                                 uint32_t idx, uint64_t* first = nullptr) {
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
    const uint64_t off = __ldg(A.pat_off + pid);
    if (a + len > A.n || !equal_text_p(A, a, A.pat_bytes + off, len)) continue;
    if (dst) {
      if (idx + c < A.slice_cap) dst[idx + c] = pack_match(a, pid);
    } else if (first && c == 0) {
      *first = pack_match(a, pid);
    }
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
    uint64_t first = 0;
    if (i < nlive) {
      e = pq[i];
      c = window_probe(A, pbase + e.y, e.x, nullptr, 0, &first);
    }
    if (!__any_sync(kFull, c != 0)) continue;
    if (!__any_sync(kFull, c > 1)) {  // at most one match per key (the common case): one pass
      const unsigned one = __ballot_sync(kFull, c == 1);
      const uint32_t at = fill + __popc(one & ((1u << lane) - 1u));
      if (c && at < A.slice_cap) out[at] = first;
      fill += __popc(one);
      continue;
    }
    const uint32_t excl = warp_excl_scan(c, lane);
    const uint32_t total = __shfl_sync(kFull, excl + c, 31);
    if (c) window_probe(A, pbase + e.y, e.x, out, fill + excl);
    fill += total;
  }
  __syncwarp();
  return fill;
}

// ------------------------------------------------------------ ordered output
// Diagnostics builds (MAG_B200_DIAG bit 2048): a timeline of the search in
// spare control words, ns after the first scan CTA started (the host prints
// it): [kCtrTime] ~first scan start, +1 last scan warp end, +2 first finish
// CTA past its wait, +3 last finish CTA done.
constexpr unsigned kCtrTime = 56;
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void diag_time(const ScanArgs& A, unsigned slot, bool first = false) {
  if (!(A.plan.diag & 2048)) return;
  const uint64_t t = global_ns();
  atomicMax(A.counters + kCtrTime + slot, static_cast<unsigned long long>(first ? ~t : t));
}

// Slice end (whole warp): the count, and for a nonzero count one atomic into
// its group's sum and one into the largest-slice counter (staging overflow
// check, learned density).  No fence: the finish grid reads them after the
// scan grid has completed.
__device__ __forceinline__ void publish_slice(const ScanArgs& A, uint64_t slice, uint32_t count, int lane) {
  if (lane == 0) {
    A.slice_count[slice] = count;
    if (count) {
      atomicAdd(A.group_sum + slice / kGroup, static_cast<unsigned long long>(count));
      atomicMax(A.counters + kCtrMax, static_cast<unsigned long long>(count));
    }
  }
}

// A scanning warp leaves the kernel: its candidate count joins the counters.
__device__ __forceinline__ void scan_exit(const ScanArgs& A, unsigned long long cands, int lane) {
#pragma unroll
  for (int o = 16; o; o >>= 1) cands += __shfl_xor_sync(kFull, cands, o);
  if (lane == 0 && cands) atomicAdd(A.counters + kCtrCands, cands);
  if (lane == 0) diag_time(A, 1);
}

// Let the finish grid launch now (programmatic dependent launch): its CTAs
// take SMs as the scan's CTAs leave and wait there for the scan to complete.
__device__ __forceinline__ void allow_gather(const ScanArgs& A) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) diag_time(A, 0, true);
}

}  // namespace
}  // namespace magb
