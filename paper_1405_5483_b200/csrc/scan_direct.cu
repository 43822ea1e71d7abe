// Direct kernel: q = W (16 or 8), k = m' = 1 hashed plans (cfg1-cfg4 shapes,
// m >= 2W - 1).  Sample t is the aligned W-byte word text[W t, W t + W),
// which every occurrence covers at one of W shifts.  Each scanning warp
// streams its slices through a small ring of TMA-filled steps (4 KiB / 2 KiB),
// so shared memory goes to the filter table (2^19-2^20 bits, or a blocked
// multi-probe table).  A hit's window key is the sample's own gram hash; its
// L2 screen word is loaded at once and resolved a step later, survivors
// queue per warp, walk their (pattern, shift) bucket and are compared against
// the text in global memory.  Output: per-slice ordered staging, placed by
// the finish grid (scan_dispatch.cu).
//
// Replaces FilterMachine::scan_range (filter.hpp:51-74) + verify_window
// (verify.hpp:28-31) for these plans; the match set is the reference's.
#include "kern_common.cuh"

namespace magb {
namespace {

// Multi-probe membership on a 64-entry block given as two words.
template <int H>
__device__ __forceinline__ bool bloom_admits_w(uint32_t lo, uint32_t hi, uint32_t h) {
  const uint64_t g = bloom_mix(h);
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const uint32_t b = bloom_bit(g, i);
    m |= ((b & 32u) ? hi : lo) >> (b & 31u);
  }
  return !(m & 1u);
}

// Step descriptor, written by lane 0 when the step's TMA is issued and read
// by the whole warp when the step is consumed: t first sample, slice,
// valid samples | flags << 16 (1 first step of its slice, 2 last, 4 valid).
struct __align__(16) DirectDesc {
  uint32_t t_lo, slice, lim_flags, pad;  // t_lo: low 32 bits (slices < 2^32 samples)
};

template <int H, int DEPTH, int W>
struct DirectScanner {
  static_assert(W == 8 || W == 16, "sample width");
  const ScanArgs& A;
  const int lane;
  const void* table;
  uint2* pq;
  uint8_t* slots;     // [DEPTH][kStepBytes] staged samples
  uint64_t* bars;     // [DEPTH]
  DirectDesc* desc;   // [DEPTH]
  uint32_t pqn, fill, cands32;
  uint32_t cur_slice; // the current slice
  uint64_t* out;
  // a step: 256 16-byte samples (4 KiB) or 256 8-byte samples (2 KiB)
  static constexpr uint32_t kStepBytes = W == 16 ? 4096u : 2048u;
  static constexpr uint32_t kStep = kStepBytes / W;
  static constexpr int kPer = kStep / 32;  // samples per lane per step
  // screen loads in flight: word and key (the key's low bits rotate its
  // screen bit to bit 31: l2_bits >= 16), and the step's filter-hit mask
  // (sample i at bit kPer - 1 - i)
  uint32_t pend_w[kPer], pend_k[kPer], pend_m, pend_pos;
  const uint32_t tshift, wmask;  // 32 - table_bits; screen words - 1
  // producer cursor (warp-uniform)
  unsigned long long p_t;
  uint32_t p_left;
  bool p_done;
  uint64_t pol;  // L2 evict-first policy of the text stream (created once)

  __device__ DirectScanner(const ScanArgs& a, const void* tab, uint2* q, uint8_t* sl, uint64_t* b, DirectDesc* dsc,
                           int l)
      : A(a), lane(l), table(tab), pq(q), slots(sl), bars(b), desc(dsc), pqn(0), fill(0), cands32(0),
        cur_slice(0), out(nullptr), tshift(32u - a.plan.table_bits), wmask((1u << (a.plan.l2_bits - 5)) - 1u),
        p_t(0), p_left(0), p_done(false), pol(policy_evict_first()) {
    for (int i = 0; i < kPer; ++i) pend_w[i] = pend_k[i] = 0;
    pend_m = 0;
    pend_pos = 0;
  }

  // Claim the next step and stage it into ring slot j (TMA bulk copy,
  // completion on bars[j]); an invalid descriptor marks the end.  `dep` is
  // computed from every value this warp last loaded from slot j and feeds
  // the TMA byte count, so those shared-memory loads have returned before
  // the async proxy overwrites the slot (an empty asm operand would not
  // make ptxas wait on the loads' scoreboard: that race lost the last
  // quarter of a step's samples under load in round 1).
  __device__ __forceinline__ void produce(int j, uint32_t dep = 0) {
    uint32_t slice = 0;
    bool first = false;
    while (!p_done && p_left == 0) {
      unsigned long long x = 0;
      if (lane == 0) x = atomicAdd(A.ticket, 1ull);
      x = __shfl_sync(kFull, x, 0) + A.slice_begin;
      if (x >= A.slice_end) {
        p_done = true;
        break;
      }
      // every slice below num_slices holds samples (num_slices = ceil(samples / S))
      const unsigned long long t0 = slice_t0(A, x), t1 = slice_t1(A, x);
      slice = static_cast<uint32_t>(x);
      p_t = t0;
      p_left = static_cast<uint32_t>(t1 - t0);
      first = true;
    }
    if (lane == 0) {
      DirectDesc d;
      if (p_done) {
        d.t_lo = d.slice = d.lim_flags = d.pad = 0;
      } else {
        const uint32_t lim = p_left < kStep ? p_left : kStep;
        d.t_lo = static_cast<uint32_t>(p_t);
        d.pad = 0;
        d.slice = first ? slice : desc[j == 0 ? DEPTH - 1 : j - 1].slice;
        d.lim_flags = lim | ((4u | (first ? 1u : 0u) | (p_left <= kStep ? 2u : 0u)) << 16);
        // (dep & A.zero) == 0, but only at run time: the byte count, hence the
        // TMA issue, data-depends on every word loaded from the slot.  Bulk
        // copies move whole 16-byte units: an odd 8-byte sample count (the
        // text's last step) leaves one sample for a plain load.
        const uint32_t total = W * lim, bulk = total & ~15u;
        uint8_t* dst = slots + static_cast<size_t>(j) * kStepBytes;
        const uint8_t* src = A.text + static_cast<unsigned long long>(W) * p_t;
        if (total != bulk)
          *reinterpret_cast<uint2*>(dst + bulk) = __ldg(reinterpret_cast<const uint2*>(src + bulk));
        const uint32_t bytes = bulk + (dep & A.zero);
        mbar_arrive_expect_tx(bars + j, bytes);
        if (bulk) tma_load_1d_stream(dst, src, bytes, bars + j, pol);
      }
      desc[j] = d;
    }
    if (!p_done) {
      const uint32_t lim = p_left < kStep ? p_left : kStep;
      p_t += lim;
      p_left -= lim;
    }
  }

  // Table lookup of a gram hash: bit 31 of the result is SET when the gram
  // is not admitted.  Single-probe tables keep entry idx at bit (idx - 1) & 31
  // of word idx >> 5 (host_model.cpp clear_bit), so one wrap-mode funnel
  // shift by idx lands it at bit 31, where a second funnel shift collects it.
  __device__ __forceinline__ uint32_t rejects(uint32_t h) const {
    if constexpr (H > 1) {
      const uint2 blk = static_cast<const uint2*>(table)[bloom_block(h, A.plan.blocks)];
      return bloom_admits_w<H>(blk.x, blk.y, h) ? 0u : 0x80000000u;
    } else {
      const uint32_t idx = h >> tshift;
      const uint32_t wd = static_cast<const uint32_t*>(table)[idx >> 5];
      return __funnelshift_r(wd, wd, idx);
    }
  }

  __device__ __forceinline__ void flush() {
    if (!MAG_DIAG(A, 16))
      fill = flush_queue(A, pq, pqn, W * slice_t0(A, cur_slice), out, fill, lane, true);
    pqn = 0;
  }

  // survivors queue {window key, W * sample - pbase}
  __device__ __forceinline__ void push(bool hit, uint32_t key, uint32_t pos) {
    const unsigned bal = __ballot_sync(kFull, hit);
    if (!bal) return;
    if (pqn + __popc(bal) > kDirectProbeCap) flush();
    if (hit) pq[pqn + __popc(bal & ((1u << lane) - 1u))] = make_uint2(key, pos);
    __syncwarp();
    pqn += __popc(bal);
  }

  // Filter the lane's kPer samples of a step; a filter hit issues its L2
  // screen load now and is resolved one step later (resolve()), so the L2
  // round trip overlaps the next step's filtering instead of stalling.
  // Straight-line code: the hit bits are collected into one mask by funnel
  // shifts, and every sample issues its screen load — a miss loads word 0
  // (one L1-resident address for the whole warp) and is masked off in
  // resolve().  Per sample: hash 7, lookup 6, screen 5 instructions.
  __device__ __forceinline__ void filter(const uint32_t (&h)[kPer], uint32_t lim) {
    uint32_t rej = 0;
    // all lookups first (independent shared-memory loads in flight together)
#pragma unroll
    for (int i = 0; i < kPer; ++i) rej = __funnelshift_l(rejects(h[i]), rej, 1);
    uint32_t m = ~rej & ((1u << kPer) - 1u);
    if (lim < kStep) {  // the text's last step: samples past the end never hit
#pragma unroll
      for (int i = 0; i < kPer; ++i)
        if (static_cast<uint32_t>(lane + 32 * i) >= lim) m &= ~(1u << (kPer - 1 - i));
    }
    cands32 += __popc(m);
    if (MAG_DIAG(A, 8)) m = 0;  // diagnostics: no screen / verification
    pend_m = m;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      // the window key is the sample's gram hash (direct plans: key_gram)
      const uint32_t key = h[i];
      pend_k[i] = key;
      const uint32_t wi = (m >> (kPer - 1 - i)) & 1u ? (key >> 5) & wmask : 0u;
      pend_w[i] = __ldg(A.l2map + wi);
    }
  }

  // The previous step's screen words: bit screen_bit(key) of the map sits at
  // bit (key - 1) & 31 of its word (host_model.cpp, direct plans), so a
  // rotate by key brings it to bit 31.
  __device__ __forceinline__ void resolve() {
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) s = __funnelshift_l(__funnelshift_r(pend_w[i], pend_w[i], pend_k[i]), s, 1);
    s &= pend_m;
    pend_m = 0;
    if (__any_sync(kFull, s != 0)) {
#pragma unroll
      for (int i = 0; i < kPer; ++i) push((s >> (kPer - 1 - i)) & 1u, pend_k[i], pend_pos + 32u * W * i);
    }
  }

  // Step prologue (independent of the step's data: runs while its
  // shared-memory loads are in flight): a new slice resets the output
  // cursor, otherwise the previous step's screen loads are resolved.
  __device__ __forceinline__ void begin(const DirectDesc& d) {
    if ((d.lim_flags >> 16) & 1u) {
      fill = 0;
      pqn = 0;
      cur_slice = d.slice;
      out = A.staging + static_cast<size_t>(d.slice) * A.slice_cap;
    } else {
      resolve();  // the previous step of this slice
    }
  }

  __device__ __forceinline__ void process(const DirectDesc& d, const uint32_t (&h)[kPer]) {
    const uint32_t lim = d.lim_flags & 0xffffu, flags = d.lim_flags >> 16;
    // sample offset within the slice (slices < 2^32 samples; low words suffice)
    pend_pos = W * (d.t_lo - static_cast<uint32_t>(slice_t0(A, cur_slice))) + W * lane;
    filter(h, lim);
    if (MAG_DIAG(A, 64)) resolve();  // diagnostics: no cross-step deferral
    if (flags & 2u) {
      resolve();
      if (pqn) flush();
      publish_slice(A, d.slice, fill, lane);
    }
  }

  // Stage the first DEPTH steps (before the CTA loads its table, so the
  // first text bytes are in flight during the table copy).
  __device__ void start() {
#pragma unroll 1
    for (int j = 0; j < DEPTH; ++j) produce(j);
    __syncwarp();
  }

  __device__ void run() {
    uint32_t phase = 0;  // bit j: parity of slot j's next completion
    int j = 0;
#pragma unroll 1
    while (true) {
      const DirectDesc d = desc[j];
      if (!(d.lim_flags & (4u << 16))) break;  // steps are issued in order: first invalid = end
      mbar_wait(bars + j, (phase >> j) & 1u);
      phase ^= 1u << j;
      uint4 v[kPer];
      uint32_t h[kPer];
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        if constexpr (W == 16) {
          v[i] = reinterpret_cast<const uint4*>(slots + static_cast<size_t>(j) * kStepBytes)[32 * i + lane];
        } else {
          const uint2 x = reinterpret_cast<const uint2*>(slots + static_cast<size_t>(j) * kStepBytes)[32 * i + lane];
          v[i] = make_uint4(x.x, x.y, 0u, 0u);
        }
      }
      begin(d);
      // one word of every 16-byte load gates the TMA refill of this slot (a
      // vector load returns all its words together; see produce)
      uint32_t dep = 0;
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        h[i] = hash_gram_words(v[i].x, v[i].y, v[i].z, v[i].w);
        dep ^= v[i].x;
      }
      __syncwarp();
      produce(j, dep);  // refill the slot just read
      __syncwarp();
      process(d, h);
      j = j + 1 == DEPTH ? 0 : j + 1;
    }
    scan_exit(A, cands32, lane);
  }
};

// NT: launch bound (512 threads; W = 16 plans launch 15 warps, W = 8 plans 16).
template <int H, int DEPTH, int NT, int W>
__global__ void __launch_bounds__(NT, 1) mag_direct_kernel(const __grid_constant__ ScanArgs A) {
  extern __shared__ __align__(128) uint8_t smem[];
  const size_t tbytes = align16(A.plan.table_bytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = static_cast<int>(A.nwarps);
  uint8_t* p = smem + tbytes;
  uint2* pq = reinterpret_cast<uint2*>(p) + static_cast<size_t>(warp) * kDirectProbeCap;
  p += align16(size_t(nw) * kDirectProbeCap * 8);
  uint8_t* slots = p + static_cast<size_t>(warp) * DEPTH * direct_step_bytes(W);
  p += size_t(nw) * DEPTH * direct_step_bytes(W);
  DirectDesc* desc = reinterpret_cast<DirectDesc*>(p) + static_cast<size_t>(warp) * DEPTH;
  p += size_t(nw) * DEPTH * sizeof(DirectDesc);
  uint64_t* bars = reinterpret_cast<uint64_t*>(p) + static_cast<size_t>(warp) * DEPTH;
  allow_gather(A);
  if (lane == 0) {
    for (int j = 0; j < DEPTH; ++j) mbar_init(bars + j, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  DirectScanner<H, DEPTH, W> ds(A, smem, pq, slots, bars, desc, lane);
  ds.start();
  {
    const uint4* src = static_cast<const uint4*>(A.table);
    uint4* dst = reinterpret_cast<uint4*>(smem);
    for (size_t i = threadIdx.x; i < tbytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    __syncthreads();
  }
  ds.run();
}

template <int H, int DEPTH, int NT, int W>
cudaError_t launch_direct_hd(const ScanArgs& a, cudaStream_t stream, int grid, size_t smem) {
  if (a.nwarps * 32 > NT) return cudaErrorInvalidConfiguration;
  auto k = mag_direct_kernel<H, DEPTH, NT, W>;
  cudaError_t e = allow_max_smem(reinterpret_cast<const void*>(k), smem);
  if (e != cudaSuccess) return e;
  (void)cudaGetLastError();
  k<<<grid, a.nwarps * 32, smem, stream>>>(a);
  count_launch();
  return cudaGetLastError();
}

template <int H>
cudaError_t launch_direct_h(const ScanArgs& a, cudaStream_t stream, int grid, size_t smem) {
  // at most 16 warps per CTA (a 17th would cut every warp to 96 registers)
  if (a.plan.q == 8) {  // 8-byte samples (m >= 15)
    if constexpr (H <= 4) return launch_direct_hd<H, kDirectDepth, 512, 8>(a, stream, grid, smem);
    return cudaErrorInvalidValue;
  }
  if constexpr (H == 1) {  // shallower rings leave room for a 2^20-bit single-probe table
    if (a.plan.ddepth == 2) return launch_direct_hd<H, 2, 512, 16>(a, stream, grid, smem);
    if (a.plan.ddepth == 3) return launch_direct_hd<H, 3, 512, 16>(a, stream, grid, smem);
  }
  return launch_direct_hd<H, kDirectDepth, 512, 16>(a, stream, grid, smem);
}

}  // namespace

cudaError_t launch_direct(const ScanArgs& a, cudaStream_t stream, int grid) {
  // every direct plan screens its window keys (host_model.cpp: l2_bits >= 16)
  if (a.plan.l2_bits < 16 || a.plan.l2_bits > 32) return cudaErrorInvalidValue;
  const size_t smem = direct_smem(a.plan, a.nwarps);
  switch (a.plan.probes) {
    case 1: return launch_direct_h<1>(a, stream, grid, smem);
    case 2: return launch_direct_h<2>(a, stream, grid, smem);
    case 3: return launch_direct_h<3>(a, stream, grid, smem);
    case 4: return launch_direct_h<4>(a, stream, grid, smem);
    case 5: return launch_direct_h<5>(a, stream, grid, smem);
    case 6: return launch_direct_h<6>(a, stream, grid, smem);
    case 7: return launch_direct_h<7>(a, stream, grid, smem);
    default: return launch_direct_h<8>(a, stream, grid, smem);
  }
}

}  // namespace magb
