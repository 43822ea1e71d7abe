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
__device__ __forceinline__ void st_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Exact compare of pattern pid against text[a, a + len) in global memory:
// 16 pattern bytes at a time against two aligned 16-byte text loads
// (independent, one round trip per piece) realigned with funnel shifts.
__device__ __forceinline__ uint32_t fsr(uint32_t lo, uint32_t hi, uint32_t b) { return __funnelshift_r(lo, hi, b); }
__device__ __noinline__ bool equal_text(const ScanArgs& A, unsigned long long a, uint32_t pid, uint32_t len) {
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
// Slice end (whole warp): the slice's staged matches become visible before
// its state says "done with `count` matches".
// The largest slice count (staging overflow check, learned density) is a
// fire-and-forget reduction.
__device__ __forceinline__ void publish_slice(const ScanArgs& A, uint64_t slice, uint32_t count, int lane) {
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    st_gpu(A.slice_state + slice, (static_cast<uint64_t>(A.epoch) << 32) | count);
    if (count) atomicMax(A.counters + 3, static_cast<unsigned long long>(count));
  }
  __syncwarp();
}

// A warp leaves the kernel: its candidate count joins the counters; the last warp of the final launch publishes them to the host and
// clears the next search's control words.
__device__ __forceinline__ void warp_exit(const ScanArgs& A, unsigned long long cands, int lane) {
#pragma unroll
  for (int o = 16; o; o >>= 1) cands += __shfl_xor_sync(kFull, cands, o);
  unsigned long long old = 0;
  if (lane == 0) {
    if (cands) atomicAdd(A.counters + 1, cands);
    __threadfence();
    old = atomicAdd(A.exits, 1ull);
  }
  old = __shfl_sync(kFull, old, 0);
  if (old + 1 != A.launch_warps || !A.final_launch) return;
  __threadfence();
  if (lane < 3) {
    const unsigned long long v = ld_gpu(reinterpret_cast<const uint64_t*>(A.counters) + 1 + lane);
    reinterpret_cast<volatile unsigned long long*>(A.host_ctr)[1 + lane] = v;
  }
  for (uint32_t i = lane; i < A.reset_words; i += 32) A.reset[i] = 0;
  __threadfence_system();
}

// The gather warp: advance the watermark over published slices (inclusive
// prefix counts + one CAS), copy the claimed slices' staged matches to their
// final place, until every slice of this launch is below the watermark.
// Progress only depends on slices already claimed by running warps, so it
// cannot deadlock on CTAs that are not resident.
__device__ __noinline__ void gather_warp_run(const ScanArgs& A, int lane) {
  const uint64_t epoch = A.epoch;
  uint64_t W = ld_gpu(reinterpret_cast<const uint64_t*>(A.counters));
  __threadfence();
  uint32_t idle = 0;
  while (W < A.slice_end) {
    const uint64_t x = W + lane;
    uint64_t st = 0;
    if (x < A.slice_end) st = ld_gpu(A.slice_state + x);
    const bool done = x < A.slice_end && (st >> 32) == epoch;
    const unsigned nd = __ballot_sync(kFull, !done);
    const uint32_t j = nd ? static_cast<uint32_t>(__ffs(nd) - 1) : 32u;  // leading published slices
    if (j == 0) {
      __nanosleep(idle < 4 ? 200 : 800);
      ++idle;
      W = ld_gpu(reinterpret_cast<const uint64_t*>(A.counters));
      __threadfence();
      continue;
    }
    idle = 0;
    __threadfence();  // the states above were observed: their staging is visible
    const uint64_t base = W == 0 ? 0ull : ld_gpu(A.incl + W - 1);
    const uint32_t cnt = static_cast<uint32_t>(lane < static_cast<int>(j) ? st : 0ull);
    // inclusive prefix of the j counts (64-bit)
    unsigned long long v = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(kFull, v, o);
      if (lane >= o) v += y;
    }
    if (lane < static_cast<int>(j)) st_gpu(A.incl + x, base + v);
    const unsigned long long last = __shfl_sync(kFull, base + v, j - 1);
    if (W + j == A.num_slices && lane == 0) st_gpu(reinterpret_cast<uint64_t*>(A.counters) + 2, last);
    __threadfence();
    unsigned long long old = 0;
    if (lane == 0) old = atomicCAS(A.counters, static_cast<unsigned long long>(W), W + j);
    old = __shfl_sync(kFull, old, 0);
    if (old != W) {  // another gather warp advanced first
      W = old;
      __threadfence();
      continue;
    }
    // claimed slices [W, W + j): copy their staged matches in order
    const unsigned nz = __ballot_sync(kFull, cnt != 0);
    for (unsigned m = nz; m; m &= m - 1) {
      const int s = __ffs(m) - 1;
      const uint32_t c = __shfl_sync(kFull, cnt, s);
      const unsigned long long dst = __shfl_sync(kFull, base + v, s) - c;
      const uint32_t cc = c < A.slice_cap ? c : A.slice_cap;
      const uint64_t* src = A.staging + (W + s) * A.slice_cap;
      for (uint32_t i = lane; i < cc; i += 32)
        if (dst + i < A.out_cap) A.out[dst + i] = __ldcg(src + i);
    }
    W += j;
  }
}

}  // namespace
}  // namespace magb
