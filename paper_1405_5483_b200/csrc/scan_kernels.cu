// B200 (sm_100a) search kernels for the MAG multiple pattern matcher.
//
// One persistent kernel fuses the reference's three search stages:
//   stage 1  q-gram formation       (encode_gram_at qgram.hpp:30-36, or the
//                                     hashed q-gram alphabet of paper §3.3)
//   stage 2  superimposed Shift-Or   (FilterMachine::scan_range
//            over k alignments        filter.hpp:51-74, closed form)
//   stage 3  window verification     (candidate_window / verify_window
//            + ordered output          verify.hpp:21-31, sort_dedup :37-38)
//
// Every warp is an independent scanner.  It takes slices of the sample
// stream with an atomic ticket and streams each slice through its own ring
// of shared-memory slots with 1-D TMA bulk copies (cp.async.bulk, completion
// on a per-slot mbarrier) — no block-level synchronisation after setup.
// The mask table, the verification prefilter and the byte map live in
// shared memory for the whole launch.  One sample per lane: the closed form
// of the packed Shift-Or, D_t = OR_i mask(t-i) << i, takes the previous
// samples' masks from neighbouring lanes (shuffles).  Hits become candidate
// windows in a per-warp queue (warp-scan order = text order); windows are
// verified as (window, start) pairs spread over the lanes, against a
// shared-memory prefilter and then the hashed pattern table in global
// memory.  Matches leave the warp already in (offset, pattern) order into
// the slice's staging area; mag_compact_kernel concatenates the slices.
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "scan_launch.h"

namespace magb {
namespace {

std::atomic<unsigned long long> g_launches{0};

constexpr unsigned kFull = 0xffffffffu;

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
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
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}
// Text is read once: stream it through L2 with an evict-first policy so it
// does not push the pattern tables and the screen bitmap out of L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_1d_stream(void* dst, const void* src, uint32_t bytes,
                                                   uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, int lane) {
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  return x - v;
}

template <typename E>
__device__ __forceinline__ E shfl_up_e(E v, int d) {
  return __shfl_up_sync(kFull, v, d);
}

template <typename E>
__device__ __forceinline__ int top_bit(E v) {
  if constexpr (sizeof(E) == 8)
    return 63 - __clzll(static_cast<long long>(v));
  else
    return 31 - __clz(static_cast<int>(v));
}

template <typename E>
__device__ __forceinline__ uint32_t popc_e(E v) {
  if constexpr (sizeof(E) == 8)
    return __popcll(static_cast<unsigned long long>(v));
  else
    return __popc(static_cast<uint32_t>(v));
}

__device__ __forceinline__ bool bloom_admits(const unsigned long long* tab, const ScanPlan& P,
                                             uint32_t h) {
  const unsigned long long blk = tab[bloom_block(h, P.blocks)];
  const uint64_t g = bloom_mix(h);
  unsigned long long m = 0;
#pragma unroll
  for (unsigned i = 0; i < kMaxProbes; ++i)
    if (i < P.probes) m |= blk >> bloom_bit(g, i);
  return !(m & 1ull);
}

__device__ bool equal_text(const ScanArgs& A, unsigned long long a, uint32_t pid, uint32_t len);
__device__ uint32_t flush_queue(const ScanArgs& A, uint2* pq, uint32_t pqn, unsigned long long pbase,
                                uint64_t* out, uint32_t fill, int lane, bool screened = false);

// Gram formation modes for the kernel template.
enum KGram : int { kKExact = 0, kKHashed = 1, kKCodes = 2 };

struct Smem {
  const void* table;  // smem table (or null)
  const uint32_t* pf;
  const uint8_t* map;
  uint8_t* slots;     // [warp][ring][slot_bytes]
  SlotInfo* info;     // [warp][ring]
  uint32_t* queue;    // [warp][kQueueCap]
  uint2* probe;       // [warp][kProbeCap]
  uint32_t* hits;     // [warp][kHitWords]
  uint64_t* bars;     // [warp][ring]
};

// CMP / CK: compile-time m' and k (0 = read from the plan at run time).
// A4: hashed grams start on 4-byte boundaries (q*k and q multiples of 4).
template <int GM, typename E, bool TSMEM, int QW, int CMP, int CK, bool A4>
struct Scanner {
  static constexpr int kEL = (CMP && CK) ? (CMP * CK <= 1 ? 0 : CMP * CK <= 2 ? 1 : CMP * CK <= 4 ? 2
                                                             : CMP * CK <= 8 ? 3 : CMP * CK <= 16 ? 4 : -1)
                                         : -1;  // entry log2 when known
  const ScanArgs& A;
  const Smem& S;
  const int lane, warp;
  uint8_t* myslots;
  SlotInfo* myinfo;
  uint64_t* mybars;
  uint32_t* queue;
  // chunk being processed
  const uint8_t* sb;            // slot bytes (== text[src])
  const uint32_t* sw;
  unsigned long long src;       // absolute offset of sb[0]
  uint32_t valid;               // staged bytes
  // slice output
  uint64_t* out;                // staging of the current slice
  uint32_t fill;                // matches written for the current slice
  // window keys awaiting the L2 screen: {key, start position - pbase}
  uint2* pq;
  uint32_t* pqw;                // screen words, fetched asynchronously (cp.async)
  uint32_t pqn;
  uint32_t* hbm;                // hit bitmap of the chunk (k = 1 strided)
  uint32_t cands32;             // candidates since the last fold into `cands`
  unsigned long long pbase;
  unsigned long long cands;
  // loader state (warp-uniform)
  unsigned long long ld_slice, ld_t, ld_tend;
  bool ld_done;
  uint32_t loads, cons;
  long long last_start;         // n - m: starts must be <= this
  uint32_t cslot, lslot;        // ring slots of the next consume / load
  // plan constants
  uint32_t qk;                  // text bytes per sample (strided q*k, else 1)
  uint32_t W, invW;             // starts per candidate window, 2^16/W rounded up
  int mp, ov, lead, adv, k;
  uint32_t inv_mp;              // bit / m' == (bit * inv_mp) >> 16

  __device__ Scanner(const ScanArgs& a, const Smem& s, int l, int w)
      : A(a), S(s), lane(l), warp(w), fill(0), pqn(0), pbase(0), cands(0) {
    const ScanPlan& P = A.plan;
    qk = P.overlapping || P.verify_all ? 1u : P.q * P.k;
    W = P.overlapping ? 1u : P.q;
    invW = (65536u + W - 1) / W;
    mp = static_cast<int>(P.m_prime);
    ov = mp - 1;
    lead = mp <= 16 ? ov : 0;
    adv = 32 - lead;
    k = static_cast<int>(P.k);
    inv_mp = (65536u + P.m_prime - 1) / P.m_prime;
    cslot = lslot = 0;
    myslots = S.slots + static_cast<size_t>(w) * A.ring * A.slot_bytes;
    myinfo = S.info + static_cast<size_t>(w) * A.ring;
    mybars = S.bars + static_cast<size_t>(w) * A.ring;
    queue = S.queue + static_cast<size_t>(w) * kQueueCap;
    pq = S.probe + static_cast<size_t>(w) * kProbeCap;
    pqw = reinterpret_cast<uint32_t*>(S.probe + static_cast<size_t>(A.nwarps) * kProbeCap) +
          static_cast<size_t>(w) * kProbeCap;
    hbm = S.hits + static_cast<size_t>(w) * kHitWords;
    cands32 = 0;
    ld_slice = 0;
    ld_t = ld_tend = 0;
    ld_done = false;
    loads = cons = 0;
    last_start = static_cast<long long>(A.n) - static_cast<long long>(A.plan.m);
  }

  // ------------------------------------------------------------- loader
  // A chunk of samples [t0, t1) stages text [lo, hi): the grams of its
  // samples (and of the m'-1 samples before), every candidate window they
  // can raise (starting up to q*k*ov + q - 1 bytes before the first gram)
  // and the pattern reach after the last gram.  lo is 16-byte aligned;
  // interior chunks stage exactly full_bytes.
  __device__ __forceinline__ long long raw_lo(unsigned long long t0) const {
    const ScanPlan& P = A.plan;
    const long long qm1 = (P.overlapping || P.verify_all) ? 0 : static_cast<long long>(P.q) - 1;
    return (static_cast<long long>(t0) - ov) * static_cast<long long>(qk) - qm1;
  }

  // Issue the next chunk of this warp's stream into slot lslot.  Returns
  // false when the warp has no more work.  Warp-uniform.
  __device__ bool issue() {
    while (!ld_done && ld_t >= ld_tend) {
      unsigned long long x = 0;
      if (lane == 0) x = atomicAdd(A.ticket, 1ull);
      x = __shfl_sync(kFull, x, 0) + A.slice_begin;
      if (x >= A.slice_end) {
        ld_done = true;
        break;
      }
      ld_slice = x;
      ld_t = x * A.slice_samples;
      ld_tend = ld_t + A.slice_samples;
      if (ld_tend > A.samples) ld_tend = A.samples;
      if (ld_t >= ld_tend && lane == 0) A.slice_count[x] = 0;  // slice past the last sample
    }
    if (ld_done) return false;
    const unsigned long long t0 = ld_t;
    const unsigned long long left = ld_tend - t0;
    const uint32_t nsamp = left < A.chunk_samples ? static_cast<uint32_t>(left) : A.chunk_samples;
    const long long rl = raw_lo(t0);
    unsigned long long lo = rl > 0 ? static_cast<unsigned long long>(rl) & ~15ull : 0ull;
    uint32_t bulk, len;
    if (nsamp == A.chunk_samples && rl >= 0 && lo + A.full_bytes <= A.n) {
      bulk = len = A.full_bytes;  // interior chunk
    } else {
      const ScanPlan& P = A.plan;
      const unsigned long long extra = P.overlapping ? P.q : 0;
      unsigned long long hi = (t0 + nsamp) * qk + extra + A.back;
      if (hi > A.n) hi = A.n;
      if (hi < lo) hi = lo;
      // whole 16-byte blocks except at the very end of the text
      const unsigned long long hi16 = (hi + 15) & ~15ull;
      const unsigned long long bulk_end = hi16 <= A.n ? hi16 : (A.n & ~15ull);
      bulk = bulk_end > lo ? static_cast<uint32_t>(bulk_end - lo) : 0u;
      len = static_cast<uint32_t>(hi - lo) > bulk ? static_cast<uint32_t>(hi - lo) : bulk;
    }
    const uint32_t slot = lslot;
    lslot = lslot + 1 == A.ring ? 0 : lslot + 1;
    uint8_t* dst = myslots + static_cast<size_t>(slot) * A.slot_bytes;
    if (static_cast<uint32_t>(lane) < len - bulk) dst[bulk + lane] = __ldg(A.text + lo + bulk + lane);
    __syncwarp();
    if (lane == 0) {
      SlotInfo& in = myinfo[slot];
      in.slice = ld_slice;
      in.t0 = t0;
      in.src = lo;
      in.nsamp = nsamp;
      in.valid = len;
      in.flags = (t0 == ld_slice * A.slice_samples ? 1u : 0u) | (t0 + nsamp == ld_tend ? 2u : 0u);
      fence_proxy_async();
      mbar_arrive_expect_tx(mybars + slot, bulk);
      if (bulk) tma_load_1d_stream(dst, A.text + lo, bulk, mybars + slot, policy_evict_first());
    }
    __syncwarp();
    ld_t = t0 + nsamp;
    ++loads;
    return true;
  }

  // ----------------------------------------------------------- stage 1+2
  __device__ __forceinline__ E table_entry(uint32_t idx) const {
    const uint32_t el = kEL >= 0 ? static_cast<uint32_t>(kEL) : A.plan.entry_log2;
    if constexpr (sizeof(E) == 8) {
      const uint64_t* t = TSMEM ? static_cast<const uint64_t*>(S.table)
                                : static_cast<const uint64_t*>(A.table);
      return TSMEM ? t[idx] : __ldg(t + idx);
    } else {
      const uint32_t* t = TSMEM ? static_cast<const uint32_t*>(S.table)
                                : static_cast<const uint32_t*>(A.table);
      const uint32_t word = TSMEM ? t[idx >> (5 - el)] : __ldg(t + (idx >> (5 - el)));
      return word >> ((idx & ((32u >> el) - 1u)) << el);
    }
  }

  // Multi-probe membership (probes >= 2): all probed entries of the gram's
  // 64-entry block admit (bit 0).
  __device__ __forceinline__ bool bloom_test(uint32_t h) const {
    return bloom_admits(static_cast<const unsigned long long*>(S.table), A.plan, h);
  }

  // Mask of the gram at slot offset rel, read by sample t (absolute; used
  // for SMAG's code array).
  __device__ __forceinline__ E gram_mask(uint32_t rel, unsigned long long t) const {
    const ScanPlan& P = A.plan;
    if constexpr (GM == kKCodes) {
      const unsigned long long u = P.overlapping ? t : (t + 1) * P.k - 1;
      return table_entry(__ldg(A.codes + u));
    } else if constexpr (GM == kKHashed) {
      const uint32_t wi = rel >> 2;
      uint32_t x[4] = {0, 0, 0, 0};
      if constexpr (A4) {
        if constexpr (QW == 4) {
          const uint4 v = *reinterpret_cast<const uint4*>(sw + wi);  // 16-byte aligned grams
          x[0] = v.x;
          x[1] = v.y;
          x[2] = v.z;
          x[3] = v.w;
        } else {
#pragma unroll
          for (int i = 0; i < QW; ++i) x[i] = sw[wi + i];
        }
      } else {
        const uint32_t sh = (rel & 3u) << 3;
        uint32_t w[QW + 1];
#pragma unroll
        for (int i = 0; i <= QW; ++i) w[i] = sw[wi + i];
#pragma unroll
        for (int i = 0; i < QW; ++i) x[i] = __funnelshift_r(w[i], w[i + 1], sh);
      }
      if constexpr (!A4) {  // q % 4 == 0 fills the last word
        const uint32_t rem = P.q - 4u * (QW - 1);  // 1..4 bytes in the last word
        x[QW - 1] &= rem >= 4 ? 0xffffffffu : ((1u << (8 * rem)) - 1u);
      }
      const uint32_t h = hash_gram_words(x[0], x[1], x[2], x[3]);
      if constexpr (CMP == 1 && CK == 1 && sizeof(E) == 4 && TSMEM) {
        if (P.probes > 1) return static_cast<E>(bloom_test(h) ? 0u : 1u);
      }
      return table_entry(h >> (32 - P.table_bits));
    } else {
      const uint32_t q = P.q, sp = P.sigma_prime;
      uint32_t code = S.map[sb[rel + q - 1]];
      for (int i = static_cast<int>(q) - 2; i >= 0; --i) code = code * sp + S.map[sb[rel + i]];
      return table_entry(code);
    }
  }

  // ----------------------------------------------------------- stage 3
  __device__ __forceinline__ uint32_t key_at(uint32_t r, uint32_t v) const {
    const uint32_t wi = r >> 2, sh = (r & 3u) << 3;
    const uint32_t w0 = sw[wi], w1 = sw[wi + 1];
    const uint32_t x0 = __funnelshift_r(w0, w1, sh) & key_word_mask(v, 0);
    uint32_t x1 = 0, x2 = 0, x3 = 0;
    if (v > 4) {
      const uint32_t w2 = sw[wi + 2];
      x1 = __funnelshift_r(w1, w2, sh) & key_word_mask(v, 1);
      if (v > 8) {
        const uint32_t w3 = sw[wi + 3];
        x2 = __funnelshift_r(w2, w3, sh) & key_word_mask(v, 2);
        if (v > 12) x3 = __funnelshift_r(w3, sw[wi + 4], sh) & key_word_mask(v, 3);
      }
    }
    return key_words(x0, x1, x2, x3);
  }

  __device__ __forceinline__ bool prefilter_pass(uint32_t key) const {
    const uint32_t pb = A.plan.pf_bits;
    if (pb == 0) return true;
    const uint32_t i1 = key >> (32 - pb);
    const uint32_t i2 = ((key ^ (key >> 15)) * 0x2C1B3C6Du) >> (32 - pb);
    return ((S.pf[i1 >> 5] >> (i1 & 31)) & (S.pf[i2 >> 5] >> (i2 & 31)) & 1u) != 0;
  }

  // Exact comparison of pattern pid (len bytes) with the text at slot
  // offset r (a + len <= n is checked by the caller).
  __device__ bool equal_at(uint32_t r, uint32_t pid, uint32_t len) const {
    const uint8_t* p = A.pat_bytes + __ldg(A.pat_off + pid);
    if (r + len <= valid) {
      const uint32_t wi = r >> 2, sh = (r & 3u) << 3;
      const uint4* pv4 = reinterpret_cast<const uint4*>(p);
      for (uint32_t i = 0; i < len; i += 16) {
        const uint4 pv = __ldg(pv4 + (i >> 4));
        const uint32_t pw[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t o = i + 4 * j;
          if (o >= len) break;
          const uint32_t tw = __funnelshift_r(sw[wi + (o >> 2)], sw[wi + (o >> 2) + 1], sh);
          const uint32_t rem = len - o;
          const uint32_t msk = rem >= 4 ? 0xffffffffu : ((1u << (8 * rem)) - 1u);
          if ((tw ^ pw[j]) & msk) return false;
        }
      }
      return true;
    }
    const uint8_t* t = A.text + src + r;
    for (uint32_t i = 0; i < len; ++i)
      if (__ldg(t + i) != __ldg(p + i)) return false;
    return true;
  }

  // Patterns matching at slot offset r with key `key`: counted, or written
  // (dst != nullptr) as packed keys in pattern order from dst[idx].
  __device__ uint32_t probe(uint32_t r, uint32_t key, uint64_t* dst, uint32_t idx) const {
    const uint32_t b = key & ((1u << A.plan.bucket_bits) - 1u);
    const uint32_t lo = __ldg(A.bucket_start + b), hi = __ldg(A.bucket_start + b + 1);
    const unsigned long long a = src + r;
    uint32_t c = 0;
    for (uint32_t e = lo; e < hi; ++e) {
      const uint2 ent = __ldg(A.bucket_entries + e);
      if (ent.x != key) continue;
      const uint32_t len = __ldg(A.pat_len + ent.y);
      if (a + len > A.n || !equal_at(r, ent.y, len)) continue;
      if (dst && idx + c < A.slice_cap) dst[idx + c] = pack_match(a, ent.y);
      ++c;
    }
    return c;
  }

  // One start per lane (lane order = text order): count, then ordered write.
  __device__ __forceinline__ void verify_batch(bool act, long long a) {
    uint32_t key = 0, c = 0;
    const uint32_t r = static_cast<uint32_t>(a - static_cast<long long>(src));
    if (act) {
      key = key_at(r, A.plan.key_len);
      if (prefilter_pass(key)) c = probe(r, key, nullptr, 0);
    }
    if (!__any_sync(kFull, c != 0)) return;
    const uint32_t excl = warp_excl_scan(c, lane);
    const uint32_t total = __shfl_sync(kFull, excl + c, 31);
    if (c) probe(r, key, out, fill + excl);
    fill += total;
  }

  // Window keys: a candidate window's key (read at its gram boundary
  // a0 = q*ss while the chunk is staged) against the (pattern, shift)
  // index; entry shift s names start a0 - s.  Entries come in (shift
  // descending, pattern ascending) order = text order.  Key hits are rare
  // (true matches and 32-bit key collisions) and compare against the text in
  // global memory, so queued keys outlive the staged chunk.
  __device__ bool equal_global(unsigned long long a, uint32_t pid, uint32_t len) const {
    return equal_text(A, a, pid, len);
  }

  __device__ uint32_t probe_window(unsigned long long a0, uint32_t key, uint64_t* dst,
                                   uint32_t idx) const {
    const uint32_t b = key & ((1u << A.plan.bucket_bits) - 1u);
    const uint32_t lo = __ldg(A.bucket_start + b), hi = __ldg(A.bucket_start + b + 1);
    uint32_t c = 0;
    for (uint32_t e = lo; e < hi; ++e) {
      const uint2 ent = __ldg(A.bucket_entries + e);
      if (ent.x != key) continue;
      const uint32_t s = ent.y >> kPidBits, pid = ent.y & ((1u << kPidBits) - 1u);
      if (s > a0) continue;  // start before the text
      const unsigned long long a = a0 - s;
      const uint32_t len = __ldg(A.pat_len + pid);
      if (a + len > A.n || !equal_global(a, pid, len)) continue;
      if (dst && idx + c < A.slice_cap) dst[idx + c] = pack_match(a, pid);
      ++c;
    }
    return c;
  }

  // Screen + verify the probe queue: 4 consecutive keys per lane (lane-major
  // = text order); the four L2 bitmap loads are independent, so one round
  // trip covers 128 windows.  Survivors walk their bucket.
  __device__ void flush_pq() {
    cp_async_wait_all();
    if (!(A.plan.diag & 2)) fill = flush_queue(A, pq, pqn, pbase, out, fill, lane);
    pqn = 0;
  }

  // One candidate window per lane (super position ss, lane order = text
  // order): its key, read now from the staged chunk, joins the probe queue.
  // Windows whose key would run past the text cannot match.
  __device__ __forceinline__ void push_window(bool live, long long ss) {
    const uint32_t v = A.plan.wkey_len;
    const unsigned long long a0 = static_cast<unsigned long long>(ss) * A.plan.q;
    bool ok = live && a0 + v <= A.n;
    uint32_t key = 0;
    if (ok) {
      key = key_at(static_cast<uint32_t>(a0 - src), v);
      ok = prefilter_pass(key);
    }
    const unsigned bal = __ballot_sync(kFull, ok);
    if (!bal) return;
    if (pqn + __popc(bal) > kProbeCap) flush_pq();
    if (ok) {
      const uint32_t at = pqn + __popc(bal & ((1u << lane) - 1u));
      pq[at] = make_uint2(key, static_cast<uint32_t>(a0 - pbase));
      const uint32_t lb = A.plan.l2_bits;
    }
    __syncwarp();
    pqn += __popc(bal);
  }

  // Queued candidate windows -> keys (read from the staged chunk now) in the
  // probe queue.  Windows whose key would run past the text cannot match.
  __device__ void drain_windows(uint32_t qlen, long long ss_ref) {
    __syncwarp();
    const uint32_t q = A.plan.q, v = A.plan.wkey_len;
    for (uint32_t i0 = 0; i0 < qlen; i0 += 32) {
      const uint32_t i = i0 + lane;
      bool ok = false;
      uint32_t key = 0;
      unsigned long long a0 = 0;
      if (i < qlen) {
        a0 = static_cast<unsigned long long>(ss_ref + static_cast<long long>(queue[i])) * q;
        ok = a0 + v <= A.n;
        if (ok) {
          key = key_at(static_cast<uint32_t>(a0 - src), v);
          ok = prefilter_pass(key);
        }
      }
      const unsigned bal = __ballot_sync(kFull, ok);
      if (!bal) continue;
      if (pqn + __popc(bal) > kProbeCap) flush_pq();
      if (ok) {
        const uint32_t at = pqn + __popc(bal & ((1u << lane) - 1u));
        pq[at] = make_uint2(key, static_cast<uint32_t>(a0 - pbase));

      }
      __syncwarp();
      pqn += __popc(bal);
    }
    __syncwarp();
  }

  // Verify the queued windows: (window, start) pairs spread over the lanes
  // in order, so each lane checks one start.  Entries are super positions
  // relative to ss_ref.
  __device__ void drain(uint32_t qlen, long long ss_ref) {
    if (A.plan.window_key) {
      drain_windows(qlen, ss_ref);
      return;
    }
    drain_starts(qlen, ss_ref);
  }

  __device__ void drain_starts(uint32_t qlen, long long ss_ref) {
    __syncwarp();
    const uint32_t pairs = qlen * W;
    for (uint32_t p0 = 0; p0 < pairs; p0 += 32) {
      const uint32_t p = p0 + lane;
      bool act = p < pairs;
      long long a = 0;
      if (act) {
        const uint32_t ci = (p * invW) >> 16;
        const uint32_t d = p - ci * W;
        const long long ss = static_cast<long long>(queue[ci]) + ss_ref;
        a = ss * static_cast<long long>(W) - static_cast<long long>(W - 1) + d;
        act = a >= 0 && a <= last_start;
      }
      verify_batch(act, a);
    }
    __syncwarp();
  }

  // ------------------------------------------------------------ a chunk
  // Queue the candidates of a sub-iteration (lane order = sample order).
  __device__ __forceinline__ void enqueue(E hits, int tr, int k, uint32_t inv_mp, uint32_t& qlen,
                                          long long ss_ref) {
    const unsigned hb = __ballot_sync(kFull, hits != 0);
    if (!hb) return;
    if (k == 1) {
      // one alignment: at most one candidate per lane
      const uint32_t total = __popc(hb);
      cands += hits ? 1u : 0u;
      if (qlen + total > kQueueCap) {
        drain(qlen, ss_ref);
        qlen = 0;
      }
      if (hits) queue[qlen + __popc(hb & ((1u << lane) - 1u))] = static_cast<uint32_t>(tr);
      __syncwarp();
      qlen += total;
      return;
    }
    // k alignments: a lane's candidates in ascending super position
    // (alignment j descending): rel = tr * k + (k - 1 - j)
    const uint32_t cnt = popc_e(hits);
    cands += cnt;
    const uint32_t excl = warp_excl_scan(cnt, lane);
    const uint32_t total = __shfl_sync(kFull, excl + cnt, 31);
    const int rel_base = tr * k + (k - 1);
    uint32_t done = 0;
    while (done < total) {
      if (qlen == kQueueCap) {
        drain(qlen, ss_ref);
        qlen = 0;
      }
      const uint32_t take = min(static_cast<uint32_t>(kQueueCap) - qlen, total - done);
      if (cnt) {
        uint32_t rank = excl;
        E h = hits;
        while (h) {
          const int bit = top_bit(h);
          h &= static_cast<E>(~(E(1) << bit));
          if (rank >= done && rank < done + take) {
            const int j = static_cast<int>((static_cast<uint32_t>(bit) * inv_mp) >> 16);
            queue[qlen + rank - done] = static_cast<uint32_t>(rel_base - j);
          }
          ++rank;
        }
      }
      __syncwarp();
      qlen += take;
      done += take;
    }
  }

  // q = 16, m' = k = 1, 16-byte window keys (the cfg2/cfg4 plan shape): a
  // candidate's window key is the very gram the filter just hashed, so hit
  // lanes hash their key from the registers and append it to the probe queue
  // in place — no bitmap, no expansion, no second read of the slot.
  __device__ __forceinline__ void push_inline(bool hit, uint32_t key, unsigned long long a0) {
    const unsigned bal = __ballot_sync(kFull, hit);
    if (!bal) return;
    cands32 += hit ? 1u : 0u;
    if (pqn + __popc(bal) > kProbeCap) flush_pq();
    if (hit) {
      const uint32_t at = pqn + __popc(bal & ((1u << lane) - 1u));
      pq[at] = make_uint2(key, static_cast<uint32_t>(a0 - pbase));

    }
    __syncwarp();
    pqn += __popc(bal);
  }

  __device__ void fused_window_loop(const SlotInfo& in, int g0, int nsamp) {
    const ScanPlan& P = A.plan;
    const uint32_t tb = P.table_bits;
    const uint32_t* tab = static_cast<const uint32_t*>(S.table);
    const unsigned long long gbase = src + static_cast<unsigned long long>(g0);  // absolute byte of sample 0
    for (int base = 0; base < nsamp; base += 64) {
      uint32_t key[2];
      bool hit[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int t = base + 32 * h + lane;
        const uint4 v = *reinterpret_cast<const uint4*>(sw + ((g0 + 16 * t) >> 2));
        const uint32_t gh = hash_gram_words(v.x, v.y, v.z, v.w);
        if (P.probes > 1) {
          hit[h] = bloom_test(gh);
        } else {
          const uint32_t idx = gh >> (32 - tb);
          hit[h] = !((tab[idx >> 5] >> (idx & 31u)) & 1u);
        }
        key[h] = key_words(v.x, v.y, v.z, v.w);
      }
      push_inline(hit[0], key[0], gbase + 16ull * (base + lane));
      push_inline(hit[1], key[1], gbase + 16ull * (base + 32 + lane));
    }
  }

  // k = 1 strided chunk: the filter only records hit ballots (one bit per
  // sample, in a per-chunk bitmap); the bitmap is expanded into candidate
  // windows once at the end of the chunk.
  __device__ void bitmap_chunk(const SlotInfo& in, int mp) {
    const ScanPlan& P = A.plan;
    const int nsamp = static_cast<int>(in.nsamp);
    const int ov = mp - 1;
    const int g0 = static_cast<int>(((in.t0 + 1) * P.k - 1) * P.q - src);
    const int gstep = static_cast<int>(P.q);
    const long long ss_ref = static_cast<long long>(in.t0) - ov;  // ss = ss_ref + t_rel
    const int tmin = in.t0 < static_cast<unsigned long long>(ov) ? -static_cast<int>(in.t0) : -ov;
    const int thit = in.t0 < static_cast<unsigned long long>(ov) ? ov - static_cast<int>(in.t0) : 0;
    const E mm = static_cast<E>(P.match_mask);
    const E ones = static_cast<E>(~E(0));
    const int nwords = (nsamp + 31) >> 5;
    if (lane < nwords) hbm[lane] = 0u;
    __syncwarp();
    if constexpr (GM == kKHashed && A4 && QW == 4 && CMP == 1 && CK == 1) {
      if ((nsamp & 63) == 0 && thit == 0 && P.window_key && P.wkey_len == 16 && !(P.diag & 1)) {
        fused_window_loop(in, g0, nsamp);
        return;
      }
    }
    if (CMP == 1 && (nsamp & 63) == 0 && thit == 0) {
      // interior m' = 1 chunk: every lane valid, hits are ~mask & 1
      for (int base = 0; base < nsamp; base += 64) {
        const int ta = base + lane, tb = ta + 32;
        const E ma = gram_mask(static_cast<uint32_t>(g0 + ta * gstep), in.t0 + ta);
        const E mb = gram_mask(static_cast<uint32_t>(g0 + tb * gstep), in.t0 + tb);
        const unsigned ba = __ballot_sync(kFull, !(ma & mm));
        const unsigned bb = __ballot_sync(kFull, !(mb & mm));
        if (lane == 0) {
          hbm[base >> 5] = ba;
          hbm[(base >> 5) + 1] = bb;
        }
      }
    } else {
      const int lead = ov;
      for (int base = -lead; base + lead < nsamp; base += 64 - lead) {
        const int ta = base + lane, tb = ta + 32;
        const bool va = ta >= tmin && ta < nsamp, vb = tb < nsamp;
        const E ma = gram_mask(static_cast<uint32_t>(va ? g0 + ta * gstep : 0), in.t0 + (va ? ta : 0));
        const E mb = gram_mask(static_cast<uint32_t>(vb ? g0 + tb * gstep : 0), in.t0 + (vb ? tb : 0));
        const E Ma = va ? ma : ones, Mb = vb ? mb : ones;
        E Da = Ma, Db = Mb;
#pragma unroll
        for (int i = 1; i <= (CMP ? CMP - 1 : 15); ++i) {
          if (!CMP && i > ov) break;
          const E ua = shfl_up_e(Ma, i);
          const E ub = shfl_up_e(Mb, i);
          const E wa = __shfl_sync(kFull, Ma, (lane - i) & 31);
          Da |= static_cast<E>(ua << i);
          Db |= static_cast<E>((lane >= i ? ub : wa) << i);
        }
        const unsigned ba = __ballot_sync(kFull, lane >= lead && ta >= thit && ta < nsamp && !(Da & mm));
        const unsigned bb = __ballot_sync(kFull, tb >= thit && tb < nsamp && !(Db & mm));
        if (lane == 0) {
          // samples [base, base + 64) -> bits; base may be unaligned (m' > 1)
          const int s0 = base + 32 * 0, s1 = base + 32;
          if (ba) {
            const int w = s0 >> 5, off = s0 & 31;  // s0 >= -lead: lanes < lead carry no bits
            if (s0 >= 0) {
              hbm[w] |= ba << off;
              if (off && w + 1 < kHitWords) hbm[w + 1] |= ba >> (32 - off);
            } else {
              hbm[0] |= ba >> (-s0);
            }
          }
          if (bb) {
            const int w = s1 >> 5, off = s1 & 31;
            hbm[w] |= bb << off;
            if (off && w + 1 < kHitWords) hbm[w + 1] |= bb >> (32 - off);
          }
        }
      }
    }
    __syncwarp();
    // expand: lane l owns bitmap word l; candidate ranks in text order
    const uint32_t word = lane < nwords ? hbm[lane] : 0u;
    const uint32_t cnt = __popc(word);
    cands32 += cnt;
    const uint32_t excl = warp_excl_scan(cnt, lane);
    const uint32_t total = __shfl_sync(kFull, excl + cnt, 31);
    if (P.diag & 1) return;
    // lane r takes the candidate of rank r: its word is found by binary
    // search over the word prefix counts, its bit with __fns
    for (uint32_t r0 = 0; r0 < total; r0 += 32) {
      const uint32_t rank = r0 + lane;
      int w = 0;
#pragma unroll
      for (int step = 16; step; step >>= 1) {
        const int c = w + step;
        const uint32_t e = __shfl_sync(kFull, excl, c & 31);
        if (c < nwords && e <= rank) w = c;
      }
      const uint32_t ww = __shfl_sync(kFull, word, w);
      const uint32_t ew = __shfl_sync(kFull, excl, w);
      const bool live = rank < total;
      const int t_rel = 32 * w + static_cast<int>(__fns(ww, 0, static_cast<int>(rank - ew) + 1));
      if (P.diag & 4) {  // diagnostics: expansion only
        if (live && t_rel < 0) cands32 += 1;
        continue;
      }
      if (P.window_key) {
        push_window(live, ss_ref + t_rel);
      } else {
        const uint32_t bal = __ballot_sync(kFull, live);
        if (live) queue[lane] = static_cast<uint32_t>(t_rel);
        __syncwarp();
        drain_starts(__popc(bal), ss_ref);
      }
    }
  }

  __device__ void process_chunk(const SlotInfo& in) {
    const ScanPlan& P = A.plan;
    const int nsamp = static_cast<int>(in.nsamp);
    if (P.verify_all) {
      // every start is a candidate: one start per lane, in order
      const long long t0 = static_cast<long long>(in.t0);
      for (int b = 0; b < nsamp; b += 32) {
        const long long a = t0 + b + lane;
        verify_batch(b + lane < nsamp && a <= last_start, a);
      }
      return;
    }
    const int mp = CMP ? CMP : this->mp;
    const int ov = mp - 1;
    const int k = CK ? CK : this->k;
    const uint32_t inv_mp = CMP ? (65536u + CMP - 1) / CMP : this->inv_mp;
    if (k == 1 && !P.overlapping && mp <= 16) {
      bitmap_chunk(in, mp);
      return;
    }
    // slot offset of the gram of relative sample 0, and per-sample stride
    const int g0 = static_cast<int>(
        (P.overlapping ? in.t0 : ((in.t0 + 1) * P.k - 1) * P.q) - src);
    const int gstep = CK ? (P.overlapping ? 1 : static_cast<int>(P.q) * CK) : static_cast<int>(qk);
    // super positions: ss = ss_ref + rel, rel = tr * k + (k - 1 - j) >= 0
    const long long ss_ref = (static_cast<long long>(in.t0) - ov) * k;
    // samples before the text start have no gram; samples < m'-1 never hit
    const int tmin = in.t0 < static_cast<unsigned long long>(ov) ? -static_cast<int>(in.t0) : -ov;
    const int thit = in.t0 < static_cast<unsigned long long>(ov) ? ov - static_cast<int>(in.t0) : 0;
    const E mm = static_cast<E>(P.match_mask);
    const E ones = static_cast<E>(~E(0));
    uint32_t qlen = 0;
    if (mp <= 16) {
      // two samples per lane per step (tr and tr + 32): independent gram
      // chains for the scheduler; D needs the m'-1 previous samples' masks
      const int lead = ov;
      for (int base = -lead; base + lead < nsamp; base += 64 - lead) {
        const int ta = base + lane, tb = ta + 32;
        const bool va = ta >= tmin && ta < nsamp, vb = tb < nsamp;
        // divergence-free: invalid lanes read a safe slot offset
        const E ma = gram_mask(static_cast<uint32_t>(va ? g0 + ta * gstep : 0), in.t0 + (va ? ta : 0));
        const E mb = gram_mask(static_cast<uint32_t>(vb ? g0 + tb * gstep : 0), in.t0 + (vb ? tb : 0));
        const E Ma = va ? ma : ones, Mb = vb ? mb : ones;
        E Da = Ma, Db = Mb;
#pragma unroll
        for (int i = 1; i <= (CMP ? CMP - 1 : 15); ++i) {
          if (!CMP && i > ov) break;
          const E ua = shfl_up_e(Ma, i);
          const E ub = shfl_up_e(Mb, i);
          const E wa = __shfl_sync(kFull, Ma, (lane - i) & 31);  // b's predecessors in a
          Da |= static_cast<E>(ua << i);
          Db |= static_cast<E>((lane >= i ? ub : wa) << i);
        }
        const E ha = (lane >= lead && ta >= thit && ta < nsamp) ? static_cast<E>(~Da & mm) : static_cast<E>(0);
        const E hb = (tb >= thit && tb < nsamp) ? static_cast<E>(~Db & mm) : static_cast<E>(0);
        enqueue(ha, ta, k, inv_mp, qlen, ss_ref);
        enqueue(hb, tb, k, inv_mp, qlen, ss_ref);
      }
    } else {
      for (int base = 0; base < nsamp; base += 32) {
        const int tr = base + lane;
        E D = static_cast<E>(0);
        for (int i = 0; i < mp; ++i) {
          const int ti = tr - i;
          const bool v = ti >= tmin && ti < nsamp;
          const E M = gram_mask(static_cast<uint32_t>(v ? g0 + ti * gstep : 0), in.t0 + (v ? ti : 0));
          D |= static_cast<E>((v ? M : ones) << i);
        }
        const E hits = (tr >= thit && tr < nsamp) ? static_cast<E>(~D & mm) : static_cast<E>(0);
        enqueue(hits, tr, k, inv_mp, qlen, ss_ref);
      }
    }
    if (qlen) drain(qlen, ss_ref);
  }

  // ------------------------------------------------------------- driver
  __device__ void run() {
    for (uint32_t r = 0; r < A.ring; ++r)
      if (!issue()) break;
    uint32_t phase = 0;
    while (cons < loads) {
      const uint32_t slot = cslot;
      mbar_wait(mybars + slot, phase);
      cslot = cslot + 1 == A.ring ? 0 : cslot + 1;
      phase ^= cslot == 0;
      const SlotInfo in = myinfo[slot];
      sb = myslots + static_cast<size_t>(slot) * A.slot_bytes;
      sw = reinterpret_cast<const uint32_t*>(sb);
      src = in.src;
      valid = in.valid;
      if (in.flags & 1u) {
        fill = 0;
        pqn = 0;
        pbase = in.src;
      }
      out = A.staging + static_cast<size_t>(in.slice) * A.slice_cap;
      process_chunk(in);
      if (in.flags & 2u) {
        if (pqn) flush_pq();
        if (lane == 0) A.slice_count[in.slice] = fill;
      }
      __syncwarp();
      ++cons;
      issue();
    }
    unsigned long long c = cands + cands32;
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
    if (lane == 0 && c) atomicAdd(A.counters + 1, c);
  }
};

template <int GM, typename E, bool TSMEM, int QW, int CMP, int CK, bool A4>
__global__ void __launch_bounds__(kMaxWarps * 32, 1) mag_scan_kernel(const __grid_constant__ ScanArgs A) {
  // let the dependent gather grid launch early (it waits for our completion)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(128) uint8_t smem[];
  const SmemLayout L = smem_layout(A.plan, A.slot_bytes, A.ring, A.nwarps);
  Smem S;
  S.table = smem + L.table;
  S.pf = reinterpret_cast<const uint32_t*>(smem + L.pf);
  S.map = smem + L.map;
  S.slots = smem + L.slots;
  S.info = reinterpret_cast<SlotInfo*>(smem + L.info);
  S.queue = reinterpret_cast<uint32_t*>(smem + L.queue);
  S.probe = reinterpret_cast<uint2*>(smem + L.probe);
  S.hits = reinterpret_cast<uint32_t*>(smem + L.hits);
  S.bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  {
    const int tid = threadIdx.x, nt = blockDim.x;
    if (TSMEM && A.plan.table_in_smem) {
      const uint4* src = static_cast<const uint4*>(A.table);
      uint4* dst = reinterpret_cast<uint4*>(smem + L.table);
      const size_t nv = A.plan.table_bytes / 16;
      for (size_t i = tid; i < nv; i += nt) dst[i] = __ldg(src + i);
    }
    {
      const uint4* src = reinterpret_cast<const uint4*>(A.prefilter);
      uint4* dst = reinterpret_cast<uint4*>(smem + L.pf);
      const size_t nv = ((size_t(1) << A.plan.pf_bits) / 8 + 15) / 16;
      for (size_t i = tid; i < nv; i += nt) dst[i] = __ldg(src + i);
    }
    for (int i = tid; i < 256; i += nt) smem[L.map + i] = A.map ? __ldg(A.map + i) : 0;
    for (uint32_t b = tid; b < A.nwarps * A.ring; b += nt) mbar_init(S.bars + b, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
  }
  Scanner<GM, E, TSMEM, QW, CMP, CK, A4> sc(A, S, threadIdx.x & 31, threadIdx.x >> 5);
  sc.run();
}

// ============================================================ direct kernel
// q = W (16 or 8), k = m' = 1 hashed plans (cfg1-cfg4 shapes, m >= 2W - 1):
// sample t is the aligned W-byte word text[W t, W t + W), which every
// occurrence covers at one of W shifts.  Each warp streams its slices
// through a small ring of TMA-filled steps (2.5 KiB / 2 KiB), so shared
// memory goes to the filter table (2^19-2^20 bits, or a blocked multi-probe
// table).  A hit's window key is the sample's own gram hash; its L2 screen
// word is loaded at once and resolved a step later, survivors queue per warp,
// walk their (pattern, shift) bucket and are compared against the text in
// global memory.  Output: per-slice ordered staging, as every scan kernel.

// Read-only load under a predicate (0 when off): one predicated LDG, no branch.
__device__ __forceinline__ uint32_t ld_nc_pred(const uint32_t* p, bool on) {
  uint32_t v;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\tmov.u32 %0, 0;\n\t"
      "@q ld.global.nc.u32 %0, [%1];\n\t}"
      : "=r"(v)
      : "l"(p), "r"(static_cast<uint32_t>(on)));
  return v;
}

// Exact compare of pattern pid against text[a, a + len) in global memory:
// 16 pattern bytes at a time against two aligned 16-byte text loads
// (independent, one round trip per piece) realigned with funnel shifts.
__device__ __forceinline__ uint32_t fsr(uint32_t lo, uint32_t hi, uint32_t b) {
  return __funnelshift_r(lo, hi, b);
}
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

// Window-key bucket walk (see Scanner::probe_window).
__device__ uint32_t window_probe(const ScanArgs& A, unsigned long long a0, uint32_t key,
                                 uint64_t* dst, uint32_t idx) {
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

// Screen + verify a probe queue (shared by both kernels).  Keys are
// screened 4 per lane (independent L2 loads, one round trip per 128); the
// survivors — true matches and ~0.5% strays — are compacted in queue order
// into `live` (reusing the queue's own storage) so each bucket-walk round
// serves up to 32 of them.  Output is ordered: queue order = text order.
__device__ __noinline__ uint32_t flush_queue(const ScanArgs& A, uint2* pq, uint32_t pqn,
                                             unsigned long long pbase, uint64_t* out, uint32_t fill, int lane,
                                             bool screened) {
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
    // compact in place: live entries of this block land at nlive + rank (<= i0)
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
// by the whole warp when the step is consumed: x first sample, y slice,
// z valid samples | flags << 8 (1 first step of its slice, 2 last, 4 valid).
struct __align__(16) DirectDesc {
  uint32_t t, slice, lim_flags, pad;
};

template <int H, int DEPTH, int W, int CL = 1>
struct DirectScanner {
  static_assert(W == 8 || W == 16, "sample width");
  const ScanArgs& A;
  const int lane;
  const void* table;
  uint32_t table_s;   // shared-window address of the (local slice of the) table
  uint2* pq;
  uint8_t* slots;     // [DEPTH][kStepBytes] staged samples
  uint64_t* bars;     // [kDirectDepth]
  DirectDesc* desc;   // [kDirectDepth]
  uint32_t pqn, fill, cands32;
  uint32_t pbase_t;   // first sample of the current slice
  uint64_t* out;
  // a step: 256 16-byte samples (4 KiB) or 256 8-byte samples (2 KiB)
  static constexpr uint32_t kStepBytes = W == 16 ? 4096u : 2048u;
  static constexpr uint32_t kStep = kStepBytes / W;
  static constexpr int kPer = kStep / 32;  // samples per lane per step
  uint32_t pend_w[kPer], pend_b[kPer], pend_k[kPer], pend_pos;  // screen loads in flight
  // producer cursor (warp-uniform)
  uint32_t p_t, p_left;
  bool p_done;
  uint64_t pol;  // L2 evict-first policy of the text stream (created once)

  __device__ DirectScanner(const ScanArgs& a, const void* tab, uint2* q, uint8_t* sl, uint64_t* b, DirectDesc* dsc,
                           int l)
      : A(a), lane(l), table(tab), table_s(smem_addr(tab)), pq(q), slots(sl), bars(b), desc(dsc), pqn(0), fill(0),
        cands32(0),
        pbase_t(0), out(nullptr), p_t(0), p_left(0), p_done(false), pol(policy_evict_first()) {
    for (int i = 0; i < kPer; ++i) pend_w[i] = pend_b[i] = pend_k[i] = 0;
    pend_pos = 0;
  }

  // Claim the next step and stage it into ring slot j (TMA bulk copy,
  // completion on bars[j]); an invalid descriptor marks the end.  `dep` is
  // computed from every value this warp last loaded from slot j and feeds
  // the TMA byte count, so those shared-memory loads have returned before
  // the async proxy overwrites the slot (an empty asm operand would not
  // make ptxas wait on the loads' scoreboard: that race lost the last
  // quarter of a step's samples under load).
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
      const unsigned long long t0 = x * A.slice_samples;
      const unsigned long long t1 = t0 + A.slice_samples < A.samples ? t0 + A.slice_samples : A.samples;
      if (t1 <= t0) {
        if (lane == 0) A.slice_count[x] = 0;
        continue;
      }
      slice = static_cast<uint32_t>(x);
      p_t = static_cast<uint32_t>(t0);
      p_left = static_cast<uint32_t>(t1 - t0);
      first = true;
    }
    if (lane == 0) {
      DirectDesc d;
      if (p_done) {
        d.t = d.slice = d.lim_flags = d.pad = 0;
      } else {
        const uint32_t lim = p_left < kStep ? p_left : kStep;
        d.t = p_t;
        d.slice = first ? slice : desc[j == 0 ? DEPTH - 1 : j - 1].slice;
        d.lim_flags = lim | ((4u | (first ? 1u : 0u) | (p_left <= kStep ? 2u : 0u)) << 16);
        d.pad = 0;
        // (dep & A.zero) == 0, but only at run time: the byte count, hence the
        // TMA issue, data-depends on every word loaded from the slot
        // bulk copies move whole 16-byte units: an odd 8-byte sample count
        // (the text's last step) leaves one sample for a plain load
        const uint32_t total = W * lim, bulk = total & ~15u;
        uint8_t* dst = slots + static_cast<size_t>(j) * kStepBytes;
        const uint8_t* src = A.text + static_cast<uint64_t>(W) * p_t;
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

  __device__ __forceinline__ bool admits(uint32_t h) const {
    if constexpr (CL > 1) {
      // the table is split over the cluster: slice = top log2(CL) index bits,
      // read through distributed shared memory (mapa + ld.shared::cluster)
      constexpr uint32_t kLog = CL == 8 ? 3 : (CL == 4 ? 2 : 1);
      const uint32_t idx = h >> (32 - A.plan.table_bits);
      const uint32_t lbits = A.plan.table_bits - kLog;
      const uint32_t rank = idx >> lbits, off = idx & ((1u << lbits) - 1u);
      const uint32_t laddr = table_s + (off >> 5) * 4u;
      uint32_t raddr, wd;
      asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(laddr), "r"(rank));
      // not volatile: the table is constant during the scan, so the compiler
      // may issue a step's four remote loads together
      asm("ld.shared::cluster.u32 %0, [%1];" : "=r"(wd) : "r"(raddr));
      return !(__funnelshift_r(wd, wd, off) & 1u);
    } else if constexpr (H > 1) {
      const uint2 blk = static_cast<const uint2*>(table)[bloom_block(h, A.plan.blocks)];
      return bloom_admits_w<H>(blk.x, blk.y, h);
    } else {
      // word h >> (37 - tb), bit (h >> (32 - tb)) & 31 via a wrap-mode funnel shift
      const uint32_t idx = h >> (32 - A.plan.table_bits);
      const uint32_t wd = static_cast<const uint32_t*>(table)[idx >> 5];
      return !(__funnelshift_r(wd, wd, idx) & 1u);
    }
  }

  __device__ __forceinline__ void flush() {
    if (!(A.plan.diag & 16))
      fill = flush_queue(A, pq, pqn, static_cast<unsigned long long>(W) * pbase_t, out, fill, lane, true);
    pqn = 0;
  }

  // survivors queue {window key, 16 * sample - pbase}
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
  __device__ __forceinline__ void filter(const uint32_t (&h)[kPer], uint32_t lim) {
    const uint32_t lb = A.plan.l2_bits;
    const bool count_only = A.plan.diag & 8;  // diagnostics: no screen / verification
    const bool screen = lb && !(A.plan.diag & 128);
    bool hit[kPer];
    // all lookups first (independent shared-memory loads in flight together)
#pragma unroll
    for (int i = 0; i < kPer; ++i) hit[i] = admits(h[i]);
    if (lim < kStep) {  // the text's last step: samples past the end never hit
#pragma unroll
      for (int i = 0; i < kPer; ++i) hit[i] = hit[i] && static_cast<uint32_t>(lane + 32 * i) < lim;
    }
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      cands32 += hit[i] ? 1u : 0u;
      // the window key is the sample's gram hash (direct plans: key_gram)
      const uint32_t key = h[i];
      pend_k[i] = key;
      const uint32_t sb = lb ? screen_bit(key, lb) : 0u;
      pend_b[i] = sb;  // resolve() shifts in wrap mode: bit sb & 31
      // the screen word is only consumed by resolve() one step later.  W = 16
      // plans (a quarter to most samples hit: cfg2/cfg4) issue it as one
      // predicated load, no branch per sample (cfg2 +5%); W = 8 plans (rare
      // hits: cfg1/cfg3) branch around it, which skips whole warps
      const bool want = hit[i] && !count_only;
      uint32_t w;
      if constexpr (W == 16) {
        if (screen)
          w = ld_nc_pred(A.l2map + (sb >> 5), want);
        else
          w = want ? ~0u : 0u;
      } else {
        w = 0;
        if (want) w = screen ? __ldg(A.l2map + (sb >> 5)) : ~0u;
      }
      pend_w[i] = w;
    }
  }

  __device__ __forceinline__ void resolve() {
    uint32_t surv = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) surv |= (__funnelshift_r(pend_w[i], pend_w[i], pend_b[i]) & 1u) << i;
    if (__any_sync(kFull, surv != 0)) {
#pragma unroll
      for (int i = 0; i < kPer; ++i) push((surv >> i) & 1u, pend_k[i], pend_pos + 32u * W * i);
    }
#pragma unroll
    for (int i = 0; i < kPer; ++i) pend_w[i] = 0;
  }

  // Step prologue (independent of the step's data: runs while its
  // shared-memory loads are in flight): a new slice resets the output
  // cursor, otherwise the previous step's screen loads are resolved.
  __device__ __forceinline__ void begin(const DirectDesc& d) {
    if ((d.lim_flags >> 16) & 1u) {
      fill = 0;
      pqn = 0;
      pbase_t = d.t;
      out = A.staging + static_cast<size_t>(d.slice) * A.slice_cap;
    } else {
      resolve();  // the previous step of this slice
    }
  }

  __device__ __forceinline__ void process(const DirectDesc& d, const uint4 (&v)[kPer], const uint32_t (&h)[kPer]) {
    const uint32_t lim = d.lim_flags & 0xffffu, flags = d.lim_flags >> 16;
    pend_pos = W * (d.t - pbase_t) + W * lane;
    filter(h, lim);
    if (A.plan.diag & 64) resolve();  // diagnostics: no cross-step deferral
    if (flags & 2u) {
      resolve();
      if (pqn) flush();
      if (lane == 0) A.slice_count[d.slice] = fill;
    }
  }

  __device__ void run() {
#pragma unroll 1
    for (int j = 0; j < DEPTH; ++j) produce(j);
    __syncwarp();
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
      process(d, v, h);
      j = j + 1 == DEPTH ? 0 : j + 1;
    }
    unsigned long long c = cands32;
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
    if (lane == 0 && c) atomicAdd(A.counters + 1, c);
  }
};

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <int H, int DEPTH, int NT, int W, int CL = 1>
__global__ void __launch_bounds__(NT, 1) mag_direct_kernel(const __grid_constant__ ScanArgs A) {
  // let the dependent gather grid launch early (it waits for our completion)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(128) uint8_t smem[];
  // CL > 1: this CTA holds slice cluster_rank() of the table
  const size_t tbytes = align16(A.plan.table_bytes / CL);
  {
    const uint4* src = static_cast<const uint4*>(A.table) + (CL > 1 ? cluster_rank() * (tbytes / 16) : 0);
    uint4* dst = reinterpret_cast<uint4*>(smem);
    for (size_t i = threadIdx.x; i < tbytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    __syncthreads();
    if constexpr (CL > 1) cluster_sync_all();  // every slice loaded before any remote read
  }
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint8_t* p = smem + tbytes;
  uint2* pq = reinterpret_cast<uint2*>(p) + static_cast<size_t>(warp) * kDirectProbeCap;
  p += align16(size_t(nw) * kDirectProbeCap * 8);
  uint8_t* slots = p + static_cast<size_t>(warp) * DEPTH * direct_step_bytes(W);
  p += size_t(nw) * DEPTH * direct_step_bytes(W);
  DirectDesc* desc = reinterpret_cast<DirectDesc*>(p) + static_cast<size_t>(warp) * DEPTH;
  p += size_t(nw) * DEPTH * sizeof(DirectDesc);
  uint64_t* bars = reinterpret_cast<uint64_t*>(p) + static_cast<size_t>(warp) * DEPTH;
  if ((threadIdx.x & 31) == 0) {
    for (int j = 0; j < DEPTH; ++j) mbar_init(bars + j, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  DirectScanner<H, DEPTH, W, CL> ds(A, smem, pq, slots, bars, desc, threadIdx.x & 31);
  ds.run();
  if constexpr (CL > 1) cluster_sync_all();  // keep this slice alive until the cluster is done
}

template <int H, int DEPTH, int NT, int W>
cudaError_t launch_direct_hd(const ScanArgs& a, cudaStream_t stream, int grid, size_t smem) {
  static int configured = -1;
  if (configured != static_cast<int>(smem)) {
    cudaError_t e = cudaFuncSetAttribute(mag_direct_kernel<H, DEPTH, NT, W>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = static_cast<int>(smem);
  }
  (void)cudaGetLastError();
  mag_direct_kernel<H, DEPTH, NT, W><<<grid, a.nwarps * 32, smem, stream>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

// Cluster launch: CL CTAs share one table through distributed shared
// memory; the grid is a whole number of clusters (idle CTAs just sync).
template <int CL>
cudaError_t launch_direct_cluster(const ScanArgs& a, cudaStream_t stream, int grid, size_t smem) {
  auto k = mag_direct_kernel<1, 2, 512, 16, CL>;
  static int configured = -1;
  if (configured != static_cast<int>(smem)) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = static_cast<int>(smem);
  }
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(a.nwarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // as many clusters as can be co-resident (GPC packing), none beyond
  static int resident = -1, resident_smem = -1;
  if (resident_smem != static_cast<int>(smem)) {
    cfg.gridDim = dim3(CL * 64);
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, k, &cfg) != cudaSuccess || nc <= 0) {
      (void)cudaGetLastError();
      nc = 148 / CL;
    }
    resident = nc;
    resident_smem = static_cast<int>(smem);
  }
  const int want = (grid + CL - 1) / CL;
  cfg.gridDim = dim3(static_cast<unsigned>(CL * (want < resident ? want : resident)));
  (void)cudaGetLastError();
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, a);
  if (e != cudaSuccess) return e;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <int H>
cudaError_t launch_direct_h(const ScanArgs& a, cudaStream_t stream, int grid, size_t smem) {
  if (a.plan.q == 8) {  // 8-byte samples (m >= 15)
    if constexpr (H <= 4) return launch_direct_hd<H, kDirectDepth, 512, 8>(a, stream, grid, smem);
    return cudaErrorInvalidValue;
  }
  if (a.nwarps > 16) return launch_direct_hd<H, 3, kDirectMaxWarps * 32, 16>(a, stream, grid, smem);
  if constexpr (H == 1) {  // shallower rings leave room for a 2^20-bit single-probe table
    if (a.plan.cluster == 8 && a.plan.ddepth == 2 && a.nwarps <= 16)
      return launch_direct_cluster<8>(a, stream, grid, smem);
    if (a.plan.ddepth == 2) return launch_direct_hd<H, 2, 512, 16>(a, stream, grid, smem);
    if (a.plan.ddepth == 3) return launch_direct_hd<H, 3, 512, 16>(a, stream, grid, smem);
  }
  return launch_direct_hd<H, kDirectDepth, 512, 16>(a, stream, grid, smem);
}

cudaError_t launch_direct(const ScanArgs& a, cudaStream_t stream, int grid) {
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

// ============================================================== roll kernel
// Dense scan for pattern sets whose q-grams saturate any strided filter
// (many short patterns, e.g. r = 100k, m = 12 over DNA): every text
// position p is a sample whose key is the rolling hash H(p) of the q-byte
// pattern prefix (mag_common.h roll_*), tested against a blocked Bloom
// filter resident in shared memory — one 32-bit word and `H` bit tests per
// position, two IMADs to roll.  Each warp streams steps of kRollStep bytes
// (+ halo) through a kRollDepth-slot TMA ring; lane l owns the runs
// [1024 r + 32 l, +32) of a step (two independent rolling chains per lane).
// Hits of a run form a 32-bit mask per lane; they are expanded in text order
// (warp prefix over the masks) and verified while the step is still staged:
// start key of the candidate's first min(m,16) bytes -> bucket walk ->
// byte compare against the staged text.  Output: per-slice ordered staging,
// as every other scan kernel (mag_compact_kernel gathers).
struct __align__(16) RollDesc {
  unsigned long long t;  // first position (= byte offset) of the step
  uint32_t slice;
  uint32_t lim_flags;    // valid positions | flags << 16 (1 first, 2 last, 4 live)
  uint32_t valid;        // staged bytes
  uint32_t pad[3];
};

template <int Q, int H>
struct RollScanner {
  static constexpr int kRun = 32;                  // positions per lane run
  static constexpr int kBytes = kRun + Q - 1;      // bytes one run reads
  static constexpr int kV4 = (kBytes + 15) / 16;   // 16-byte loads per run
  static constexpr int kW = kV4 * 4;
  const ScanArgs& A;
  const int lane;
  const uint32_t* bloom;
  uint32_t bloom_s;         // shared-window address of the Bloom words
  uint16_t* list;           // [kRollList] hit positions of the current step
  uint8_t* slots;
  uint64_t* bars;
  RollDesc* desc;
  const uint32_t slot_bytes;
  const uint32_t bq;        // B^Q
  uint32_t fill, cands32;
  uint64_t* out;
  // producer cursor (warp-uniform)
  unsigned long long p_t, p_end;
  uint32_t p_slice;
  bool p_done, p_first;
  uint64_t pol;

  __device__ RollScanner(const ScanArgs& a, const uint32_t* bl, uint8_t* sl, uint64_t* b, RollDesc* d,
                         uint16_t* li, int l)
      : A(a), lane(l), bloom(bl), bloom_s(smem_addr(bl)), list(li), slots(sl), bars(b), desc(d),
        slot_bytes(roll_slot_bytes(a.back)),
        bq(roll_pow(Q)), fill(0), cands32(0), out(nullptr), p_t(0), p_end(0), p_slice(0), p_done(false),
        p_first(false), pol(policy_evict_first()) {}

  // Claim (if needed) and stage the next step into slot j.
  __device__ __forceinline__ void produce(int j) {
    while (!p_done && p_t >= p_end) {
      unsigned long long x = 0;
      if (lane == 0) x = atomicAdd(A.ticket, 1ull);
      x = __shfl_sync(kFull, x, 0) + A.slice_begin;
      if (x >= A.slice_end) {
        p_done = true;
        break;
      }
      const unsigned long long t0 = x * A.slice_samples;
      const unsigned long long t1 = t0 + A.slice_samples < A.samples ? t0 + A.slice_samples : A.samples;
      if (t1 <= t0) {
        if (lane == 0) A.slice_count[x] = 0;
        continue;
      }
      p_slice = static_cast<uint32_t>(x);
      p_t = t0;
      p_end = t1;
      p_first = true;
    }
    uint8_t* dst = slots + static_cast<size_t>(j) * slot_bytes;
    if (p_done) {
      if (lane == 0) desc[j].lim_flags = 0;
      __syncwarp();
      return;
    }
    const uint32_t lim = p_end - p_t < static_cast<unsigned long long>(kRollStep)
                             ? static_cast<uint32_t>(p_end - p_t) : static_cast<uint32_t>(kRollStep);
    const unsigned long long hi = p_t + slot_bytes < A.n ? p_t + slot_bytes : A.n;
    const uint32_t valid = static_cast<uint32_t>(hi - p_t);
    const uint32_t bulk = valid & ~15u;
    if (static_cast<uint32_t>(lane) < valid - bulk) dst[bulk + lane] = __ldg(A.text + p_t + bulk + lane);
    __syncwarp();
    if (lane == 0) {
      RollDesc& d = desc[j];
      d.t = p_t;
      d.slice = p_slice;
      d.valid = valid;
      d.lim_flags = lim | ((4u | (p_first ? 1u : 0u) | (p_t + lim >= p_end ? 2u : 0u)) << 16);
      fence_proxy_async();
      mbar_arrive_expect_tx(bars + j, bulk);
      if (bulk) tma_load_1d_stream(dst, A.text + p_t, bulk, bars + j, pol);
    }
    __syncwarp();
    p_t += lim;
    p_first = false;
  }

  static __device__ __forceinline__ uint32_t byte_at(const uint32_t (&w)[kW], int k) {
    return __byte_perm(w[k >> 2], 0u, 0x4440u | static_cast<uint32_t>(k & 3));
  }

  // Bloom probe bits sit at 31 - (s_i & 31) (mag_common.h roll_probe_shift),
  // so rotl(word, s_i) (funnel shift, wrap mode: the count is taken mod 32)
  // brings each to bit 31; their AND's bit 31 is the verdict.  s_0 = g and
  // s_i = umulhi(h, C_i): the extra probes cost fma-pipe IMAD.HIs, not
  // alu-pipe shifts.
  __device__ __forceinline__ uint32_t test(uint32_t h) const {
    const uint32_t g = h * kRollMix;
    // word address by IMAD (fma pipe; the alu pipe is the busier one)
    uint32_t addr, wd;
    asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(addr) : "r"(roll_word(g, A.plan.roll_words)), "r"(bloom_s));
    asm("ld.shared.u32 %0, [%1];" : "=r"(wd) : "r"(addr));
    uint32_t r = __funnelshift_l(wd, wd, g);
#pragma unroll
    for (int i = 1; i < H; ++i) r &= __funnelshift_l(wd, wd, __umulhi(h, roll_probe_mul(i)));
    return r;  // verdict in bit 31
  }

  // Bloom hits of the lane's run starting at slot offset `base` (32
  // positions; bit p = position base + p).  Prefix form of the rolling hash:
  // P(i+1) = P(i)*B + t[i], H(p) = P(p+Q) - P(p)*B^Q — one byte extraction
  // and two IMADs per position.
  __device__ __forceinline__ uint32_t filter_run(const uint8_t* sb, int base) const {
    uint32_t w[kW];
    const uint4* src = reinterpret_cast<const uint4*>(sb + base);
#pragma unroll
    for (int v = 0; v < kV4; ++v) {
      const uint4 x = src[v];
      w[4 * v] = x.x;
      w[4 * v + 1] = x.y;
      w[4 * v + 2] = x.z;
      w[4 * v + 3] = x.w;
    }
    uint32_t P[kRun + Q];
    P[0] = 0;
#pragma unroll
    for (int i = 0; i + 1 < kRun + Q; ++i) P[i + 1] = P[i] * kRollB + byte_at(w, i);
    uint32_t hits = 0;
#pragma unroll
    for (int p = 0; p < kRun; ++p) hits = __funnelshift_l(test(P[p + Q] - P[p] * bq), hits, 1);
    return __brev(hits);
  }

  // The 16 text bytes at slot offset pr (four little-endian words).
  static __device__ __forceinline__ uint4 text16(const uint32_t* sw, uint32_t pr) {
    const uint32_t wi = pr >> 2, sh = (pr & 3u) << 3;
    uint32_t x[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) x[k] = sw[wi + k];
    return make_uint4(__funnelshift_r(x[0], x[1], sh), __funnelshift_r(x[1], x[2], sh),
                      __funnelshift_r(x[2], x[3], sh), __funnelshift_r(x[3], x[4], sh));
  }

  // Start key: the first key_len bytes (mag_common.h key_words).
  __device__ __forceinline__ uint32_t key_of(const uint4& t) const {
    const uint32_t v = A.plan.key_len;
    return key_words(t.x & key_word_mask(v, 0), t.y & key_word_mask(v, 1), t.z & key_word_mask(v, 2),
                     t.w & key_word_mask(v, 3));
  }

  // Pattern pid (len bytes) against the staged text at slot offset pr.
  __device__ bool equal_slot(const uint32_t* sw, uint32_t valid, unsigned long long a, uint32_t pr,
                             uint32_t pid, uint32_t len) const {
    if (pr + len + 4 > valid) return equal_text(A, a, pid, len);
    const uint4* pv4 = reinterpret_cast<const uint4*>(A.pat_bytes + __ldg(A.pat_off + pid));
    const uint32_t wi = pr >> 2, sh = (pr & 3u) << 3;
    for (uint32_t i = 0; i < len; i += 16) {
      const uint4 pv = __ldg(pv4 + (i >> 4));
      const uint32_t pw[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t o = i + 4 * j;
        if (o >= len) break;
        const uint32_t tw = __funnelshift_r(sw[wi + (o >> 2)], sw[wi + (o >> 2) + 1], sh);
        const uint32_t rem = len - o;
        const uint32_t msk = rem >= 4 ? 0xffffffffu : ((1u << (8 * rem)) - 1u);
        if ((tw ^ pw[j]) & msk) return false;
      }
    }
    return true;
  }

  // Matches at slot offset pr (text bytes t, start key): one L2 round trip
  // per verification slot — {key, pid, len, off} and the pattern's first 16
  // bytes sit in the same 32-byte sector; longer patterns finish against
  // the pattern bytes.  Counted (first pid kept), or written from dst[idx].
  // One verification slot against the candidate: 1 = match.
  __device__ __forceinline__ bool slot_match(const uint32_t* sw, uint32_t valid, unsigned long long a,
                                             uint32_t pr, const uint4& t, uint32_t key, const uint4& h,
                                             const uint4& b) const {
    const uint32_t len = h.z & 0x7fffffffu;
    if (h.x != key || a + len > A.n) return false;
    const uint32_t d = ((t.x ^ b.x) & key_word_mask(len, 0)) | ((t.y ^ b.y) & key_word_mask(len, 1)) |
                       ((t.z ^ b.z) & key_word_mask(len, 2)) | ((t.w ^ b.w) & key_word_mask(len, 3));
    if (d) return false;
    return len <= 16 || equal_slot(sw, valid, a, pr, h.y, len);
  }

  // Linear-probe run from the key's home slot (h, b already loaded): bit 31
  // of a slot's len word says whether the next slot is occupied, so with a
  // load factor <= 1/4 nearly every lookup is one L2 round trip.
  __device__ uint32_t probe(const uint32_t* sw, uint32_t valid, unsigned long long a, uint32_t pr,
                            const uint4& t, uint32_t key, uint64_t* dst, uint32_t idx, uint32_t* first,
                            uint4 h, uint4 b) const {
    uint32_t s = key & A.vmask, c = 0;
    while (h.y != 0xffffffffu) {
      if (slot_match(sw, valid, a, pr, t, key, h, b)) {
        if (dst && idx + c < A.slice_cap) dst[idx + c] = pack_match(a, h.y);
        if (c == 0 && first) *first = h.y;
        ++c;
      }
      if (!(h.z >> 31)) break;
      s = (s + 1) & A.vmask;
      h = __ldg(A.vtab + 2 * s);
      b = __ldg(A.vtab + 2 * s + 1);
    }
    return c;
  }

  // Expand and verify a step's hits in text order: run 0 (positions
  // [32 l, 32 l + 32) of lane l) before run 1 ([1024 + 32 l, ...)).  Two
  // candidates per lane per batch, so both verification-slot loads (one L2
  // round trip each) are in flight together.
  static constexpr int kVK = 3;
  __device__ void verify_step(const uint32_t* sw, uint32_t valid, unsigned long long t, uint32_t h0,
                              uint32_t h1) {
    const uint32_t c0 = __popc(h0), c1 = __popc(h1);
    const uint32_t e0 = warp_excl_scan(c0, lane), e1 = warp_excl_scan(c1, lane);
    const uint32_t t0 = __shfl_sync(kFull, e0 + c0, 31), t1 = __shfl_sync(kFull, e1 + c1, 31);
    const uint32_t total = t0 + t1;
    cands32 += c0 + c1;
    if (A.plan.diag & 8) return;
    const uint32_t packed = e0 | (e1 << 16);
    // Expansion: with at most kRollList hits each lane writes its own hit
    // positions at its prefix offsets (text order) into the warp's list;
    // denser steps rank-search the lane masks instead.
    const bool listed = total <= static_cast<uint32_t>(kRollList);
    if (listed) {
      uint32_t idx = e0;
      for (uint32_t m = h0; m; m &= m - 1) list[idx++] = static_cast<uint16_t>(32 * lane + __ffs(m) - 1);
      idx = t0 + e1;
      for (uint32_t m = h1; m; m &= m - 1) list[idx++] = static_cast<uint16_t>(1024 + 32 * lane + __ffs(m) - 1);
      __syncwarp();
    }
    for (uint32_t base = 0; base < total; base += 32 * kVK) {
      uint32_t pr[kVK], key[kVK], c[kVK], pid0[kVK];
      uint4 tx[kVK], hq[kVK], bq[kVK];
      bool live[kVK];
#pragma unroll
      for (int k = 0; k < kVK; ++k) {
        const uint32_t rank = base + 32 * k + lane;
        live[k] = rank < total;
        if (listed) {
          pr[k] = live[k] ? list[rank] : 0u;
        } else {
          const bool r1 = rank >= t0;
          const uint32_t rr = r1 ? rank - t0 : rank;
          const uint32_t sh = r1 ? 16u : 0u;
          int o = 0;
#pragma unroll
          for (int step = 16; step; step >>= 1) {
            const uint32_t e = (__shfl_sync(kFull, packed, o + step) >> sh) & 0xffffu;
            if (e <= rr) o += step;
          }
          const uint32_t m0 = __shfl_sync(kFull, h0, o), m1 = __shfl_sync(kFull, h1, o);
          const uint32_t eo = (__shfl_sync(kFull, packed, o) >> sh) & 0xffffu;
          pr[k] = (r1 ? 1024u : 0u) + 32u * static_cast<uint32_t>(o) +
                  static_cast<uint32_t>(__fns(r1 ? m1 : m0, 0, static_cast<int>(rr - eo) + 1));
        }
        if (!live[k]) pr[k] = 0;
        tx[k] = text16(sw, pr[k]);
        key[k] = key_of(tx[k]);
      }
      // all slot loads after all expansions: a shuffle of candidate k+1
      // would otherwise share a scoreboard with candidate k's loads and wait
      // for them, serialising the round trips
#pragma unroll
      for (int k = 0; k < kVK; ++k) {
        const uint32_t slot = key[k] & A.vmask;
        const uint4 empty = make_uint4(0, 0xffffffffu, 0, 0);
        hq[k] = live[k] ? __ldg(A.vtab + 2 * slot) : empty;
        bq[k] = live[k] ? __ldg(A.vtab + 2 * slot + 1) : empty;
      }
#pragma unroll
      for (int k = 0; k < kVK; ++k) {
        pid0[k] = 0;
        c[k] = probe(sw, valid, t + pr[k], pr[k], tx[k], key[k], nullptr, 0, &pid0[k], hq[k], bq[k]);
      }
#pragma unroll
      for (int k = 0; k < kVK; ++k) {
        if (!__any_sync(kFull, c[k] != 0)) continue;
        const uint32_t ex = warp_excl_scan(c[k], lane);
        const uint32_t tot = __shfl_sync(kFull, ex + c[k], 31);
        if (c[k] == 1) {
          if (fill + ex < A.slice_cap) out[fill + ex] = pack_match(t + pr[k], pid0[k]);
        } else if (c[k] > 1) {
          const uint32_t slot = key[k] & A.vmask;
          probe(sw, valid, t + pr[k], pr[k], tx[k], key[k], out, fill + ex, nullptr, __ldg(A.vtab + 2 * slot),
                __ldg(A.vtab + 2 * slot + 1));
        }
        fill += tot;
      }
    }
  }

  __device__ void run() {
#pragma unroll 1
    for (int j = 0; j < kRollDepth; ++j) produce(j);
    uint32_t phase = 0;
    int j = 0;
#pragma unroll 1
    while (true) {
      const RollDesc d = desc[j];
      if (!(d.lim_flags & (4u << 16))) break;  // steps are issued in order: first dead slot = end
      mbar_wait(bars + j, (phase >> j) & 1u);
      phase ^= 1u << j;
      const uint32_t lim = d.lim_flags & 0xffffu, flags = d.lim_flags >> 16;
      if (flags & 1u) {
        fill = 0;
        out = A.staging + static_cast<size_t>(d.slice) * A.slice_cap;
      }
      const uint8_t* sb = slots + static_cast<size_t>(j) * slot_bytes;
      const uint32_t* sw = reinterpret_cast<const uint32_t*>(sb);
      const int b0 = 32 * lane, b1 = 1024 + 32 * lane;
      // one copy of the (large, fully unrolled) run body: instruction-cache
      // footprint matters with 16 warps at different points of the step
      uint32_t h0 = 0, h1 = 0;
#pragma unroll 1
      for (int r = 0; r < 2; ++r) {
        const uint32_t x = filter_run(sb, r ? b1 : b0);
        if (r) h1 = x; else h0 = x;
      }
      // positions past the step's valid range never hit
      auto keep = [&](int base) -> uint32_t {
        const int m = static_cast<int>(lim) - base;
        return m >= 32 ? 0xffffffffu : (m <= 0 ? 0u : ((1u << m) - 1u));
      };
      h0 &= keep(b0);
      h1 &= keep(b1);
      verify_step(sw, d.valid, d.t, h0, h1);
      if ((flags & 2u) && lane == 0) A.slice_count[d.slice] = fill;
      __syncwarp();
      produce(j);  // the slot is free again
      j = j + 1 == kRollDepth ? 0 : j + 1;
    }
    unsigned long long c = cands32;
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
    if (lane == 0 && c) atomicAdd(A.counters + 1, c);
  }
};

template <int Q, int H>
__global__ void __launch_bounds__(kMaxWarps * 32, 1) mag_roll_kernel(const __grid_constant__ ScanArgs A) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(128) uint8_t smem[];
  const size_t tbytes = align16(A.plan.table_bytes);
  {
    const uint4* src = static_cast<const uint4*>(A.table);
    uint4* dst = reinterpret_cast<uint4*>(smem);
    for (size_t i = threadIdx.x; i < tbytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t sbytes = roll_slot_bytes(A.back);
  uint8_t* p = smem + tbytes;
  uint8_t* slots = p + static_cast<size_t>(warp) * kRollDepth * sbytes;
  p += static_cast<size_t>(nw) * kRollDepth * sbytes;
  RollDesc* desc = reinterpret_cast<RollDesc*>(p) + static_cast<size_t>(warp) * kRollDepth;
  p += static_cast<size_t>(nw) * kRollDepth * sizeof(RollDesc);
  uint64_t* bars = reinterpret_cast<uint64_t*>(p) + static_cast<size_t>(warp) * kRollDepth;
  p += static_cast<size_t>(nw) * kRollDepth * 8;
  uint16_t* list = reinterpret_cast<uint16_t*>(p) + static_cast<size_t>(warp) * kRollList;
  if ((threadIdx.x & 31) == 0) {
    for (int j = 0; j < kRollDepth; ++j) mbar_init(bars + j, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  RollScanner<Q, H> rs(A, reinterpret_cast<const uint32_t*>(smem), slots, bars, desc, list, threadIdx.x & 31);
  rs.run();
}

template <int Q, int H>
cudaError_t launch_roll_qh(const ScanArgs& a, cudaStream_t stream, int grid, size_t smem) {
  static int configured = -1;
  if (configured != static_cast<int>(smem)) {
    cudaError_t e = cudaFuncSetAttribute(mag_roll_kernel<Q, H>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = static_cast<int>(smem);
  }
  (void)cudaGetLastError();
  mag_roll_kernel<Q, H><<<grid, a.nwarps * 32, smem, stream>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <int Q>
cudaError_t launch_roll_q(const ScanArgs& a, cudaStream_t stream, int grid, size_t smem) {
  if (a.plan.probes >= 3) return launch_roll_qh<Q, 3>(a, stream, grid, smem);
  if (a.plan.probes == 2) return launch_roll_qh<Q, 2>(a, stream, grid, smem);
  return launch_roll_qh<Q, 1>(a, stream, grid, smem);
}

cudaError_t launch_roll(const ScanArgs& a, cudaStream_t stream, int grid) {
  const size_t smem = roll_smem(a.plan.roll_words, a.back, a.nwarps);
  switch (a.plan.q) {
    case 8: return launch_roll_q<8>(a, stream, grid, smem);
    case 12: return launch_roll_q<12>(a, stream, grid, smem);
    case 16: return launch_roll_q<16>(a, stream, grid, smem);
    case 20: return launch_roll_q<20>(a, stream, grid, smem);
    case 24: return launch_roll_q<24>(a, stream, grid, smem);
    case 32: return launch_roll_q<32>(a, stream, grid, smem);
    default: return cudaErrorInvalidValue;
  }
}

// Gather: block b owns slices [b*per, (b+1)*per); its output offset is the
// sum of all earlier slice counts (each block reduces that prefix itself —
// at most a few tens of thousands of words from L2), then it copies its
// slices in order.  The last block publishes the total.
__global__ void __launch_bounds__(1024) mag_compact_kernel(const __grid_constant__ ScanArgs A,
                                                            uint64_t* __restrict__ out,
                                                            uint64_t out_cap) {
  // Block b owns slices [s0, s1): its base is the sum of every earlier
  // slice's count (parallel reduction), then the owned slices are scanned
  // 1024 at a time in shared memory and each warp copies whole slices.
  __shared__ unsigned long long red[32];
  __shared__ unsigned long long s_pre[1024];
  __shared__ uint32_t s_cnt[1024];
  // launched with programmatic stream serialization: wait for the scan grid
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (blockIdx.x == 0 && A.reset)
    for (uint32_t i = threadIdx.x; i < A.reset_words; i += blockDim.x) A.reset[i] = 0;
  const uint64_t ns = A.num_slices;
  const uint64_t per = (ns + gridDim.x - 1) / gridDim.x;
  uint64_t s0 = blockIdx.x * per;
  if (s0 > ns) s0 = ns;
  uint64_t s1 = s0 + per;
  if (s1 > ns) s1 = ns;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  unsigned long long acc = 0;
  {
    // sum of every earlier slice: 16-byte loads, 4 independent per round trip
    const uint64_t s0v = s0 & ~3ull;
    const uint4* cv = reinterpret_cast<const uint4*>(A.slice_count);
    uint64_t i = tid;
    for (; i + 3 * blockDim.x < s0v / 4; i += 4 * blockDim.x) {
      uint4 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = cv[i + u * blockDim.x];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += (unsigned long long)x[u].x + x[u].y + x[u].z + x[u].w;
    }
    for (; i < s0v / 4; i += blockDim.x) {
      const uint4 x = cv[i];
      acc += (unsigned long long)x.x + x.y + x.z + x.w;
    }
    if (tid < s0 - s0v) acc += A.slice_count[s0v + tid];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
  if (lane == 0) red[wid] = acc;
  __syncthreads();
  unsigned long long base = 0;
  for (int w = 0; w < nw; ++w) base += red[w];
  __syncthreads();
  uint32_t mx = 0;
  for (uint64_t c0 = s0; c0 < s1; c0 += blockDim.x) {
    const uint64_t s = c0 + tid;
    const uint32_t c = s < s1 ? A.slice_count[s] : 0u;
    mx = c > mx ? c : mx;
    // block-wide exclusive scan of c
    unsigned long long v = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(kFull, v, o);
      if (lane >= o) v += y;
    }
    if (lane == 31) red[wid] = v;
    __syncthreads();
    if (wid == 0) {
      unsigned long long t = lane < nw ? red[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(kFull, t, o);
        if (lane >= o) t += y;
      }
      red[lane] = t;  // inclusive warp totals
    }
    __syncthreads();
    const unsigned long long wbase = wid ? red[wid - 1] : 0;
    s_pre[tid] = base + wbase + v - c;
    s_cnt[tid] = c;
    const unsigned long long total = red[nw - 1];
    __syncthreads();
    const int len = static_cast<int>(s1 - c0 < blockDim.x ? s1 - c0 : blockDim.x);
    for (int j = wid; j < len; j += nw) {
      const uint32_t cj = s_cnt[j];
      if (!cj) continue;
      const uint32_t cc = cj < A.slice_cap ? cj : A.slice_cap;
      const uint64_t* srcp = A.staging + (c0 + j) * A.slice_cap;
      const unsigned long long b = s_pre[j];
      for (uint32_t i = lane; i < cc; i += 32)
        if (b + i < out_cap) out[b + i] = srcp[i];
    }
    base += total;
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint32_t y = __shfl_xor_sync(kFull, mx, o);
    mx = y > mx ? y : mx;
  }
  if (lane == 0 && mx) atomicMax(A.counters + 3, static_cast<unsigned long long>(mx));
  if (blockIdx.x == gridDim.x - 1 && tid == 0) A.counters[2] = base;
}

// SMAG prepare (encode_text qgram.cpp:29-37) on the device.
__global__ void mag_encode_kernel(const ScanPlan P, const uint8_t* __restrict__ text, uint64_t nq,
                                  const uint8_t* __restrict__ map, uint32_t* __restrict__ codes) {
  __shared__ uint8_t smap[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) smap[i] = map ? map[i] : 0;
  __syncthreads();
  const uint32_t q = P.q;
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < nq;
       u += (uint64_t)gridDim.x * blockDim.x) {
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

template <int GM, typename E, bool TSMEM, int QW, int CMP = 0, int CK = 0, bool A4 = false>
cudaError_t launch_t(const ScanArgs& a, cudaStream_t st, int grid, size_t smem) {
  auto k = mag_scan_kernel<GM, E, TSMEM, QW, CMP, CK, A4>;
  static int configured_smem = -1;  // per instantiation
  if (configured_smem != static_cast<int>(smem)) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured_smem = static_cast<int>(smem);
  }
  (void)cudaGetLastError();  // a stale error of another runtime user (e.g. torch) is not ours
  k<<<grid, a.nwarps * 32, smem, st>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

// Hashed plans with (m', k) in {(1,1), (2,1), (1,2)} get fully specialised
// inner loops; everything else runs the generic (run-time m', k) loop.
template <int GM, typename E, bool TSMEM, int QW, bool A4>
cudaError_t launch_mk(const ScanArgs& a, cudaStream_t st, int grid, size_t smem) {
  if constexpr (sizeof(E) == 4) {
    const uint32_t mp = a.plan.m_prime, k = a.plan.k;
    if (mp == 1 && k == 1) return launch_t<GM, E, TSMEM, QW, 1, 1, A4>(a, st, grid, smem);
    if (mp == 2 && k == 1) return launch_t<GM, E, TSMEM, QW, 2, 1, A4>(a, st, grid, smem);
    if (mp == 1 && k == 2) return launch_t<GM, E, TSMEM, QW, 1, 2, A4>(a, st, grid, smem);
  }
  return launch_t<GM, E, TSMEM, QW, 0, 0, A4>(a, st, grid, smem);
}

template <int GM, typename E, bool TSMEM, int QW>
cudaError_t launch_a4(const ScanArgs& a, cudaStream_t st, int grid, size_t smem) {
  // grams start on 4-byte boundaries when q and the sample stride are
  // multiples of 4 (strided only; slot bases are 16-byte aligned)
  const bool a4 = !a.plan.overlapping && a.plan.q % 4 == 0;
  if (a4) return launch_mk<GM, E, TSMEM, QW, true>(a, st, grid, smem);
  return launch_mk<GM, E, TSMEM, QW, false>(a, st, grid, smem);
}

template <int GM, typename E, bool TSMEM>
cudaError_t launch_qw(const ScanArgs& a, cudaStream_t st, int grid, size_t smem) {
  if constexpr (GM == kKHashed) {
    switch ((a.plan.q + 3) / 4) {
      case 1: return launch_a4<GM, E, TSMEM, 1>(a, st, grid, smem);
      case 2: return launch_a4<GM, E, TSMEM, 2>(a, st, grid, smem);
      case 3: return launch_a4<GM, E, TSMEM, 3>(a, st, grid, smem);
      default: return launch_a4<GM, E, TSMEM, 4>(a, st, grid, smem);
    }
  } else {
    return launch_t<GM, E, TSMEM, 1>(a, st, grid, smem);
  }
}

template <int GM>
cudaError_t launch_e(const ScanArgs& a, cudaStream_t st, int grid, size_t smem) {
  const bool wide = a.plan.entry_log2 == 6;
  if constexpr (GM == kKHashed) {
    // hashed tables are sized to shared memory
    return wide ? launch_qw<GM, uint64_t, true>(a, st, grid, smem)
                : launch_qw<GM, uint32_t, true>(a, st, grid, smem);
  } else {
    if (a.plan.table_in_smem)
      return wide ? launch_qw<GM, uint64_t, true>(a, st, grid, smem)
                  : launch_qw<GM, uint32_t, true>(a, st, grid, smem);
    return wide ? launch_qw<GM, uint64_t, false>(a, st, grid, smem)
                : launch_qw<GM, uint32_t, false>(a, st, grid, smem);
  }
}

}  // namespace

LaunchShape scan_shape(const ScanArgs& a) {
  LaunchShape s;
  s.smem_bytes = smem_layout(a.plan, a.slot_bytes, a.ring, a.nwarps).total;
  s.threads = a.nwarps * 32;
  return s;
}

cudaError_t launch_scan(const ScanArgs& a, cudaStream_t stream, int grid) {
  if (a.plan.direct) return launch_direct(a, stream, grid);
  if (a.plan.roll) return launch_roll(a, stream, grid);
  const size_t smem = smem_layout(a.plan, a.slot_bytes, a.ring, a.nwarps).total;
  if (a.plan.smag) return launch_e<kKCodes>(a, stream, grid, smem);
  if (a.plan.gram_mode == kGramHashed) return launch_e<kKHashed>(a, stream, grid, smem);
  return launch_e<kKExact>(a, stream, grid, smem);
}

cudaError_t launch_compact(const ScanArgs& a, uint64_t* out, uint64_t out_cap, cudaStream_t stream,
                           int grid) {
  // programmatic dependent launch: the gather's CTAs are scheduled while the
  // scan drains and wait in griddepcontrol.wait for its completion
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  (void)cudaGetLastError();
  cudaError_t e = cudaLaunchKernelEx(&cfg, mag_compact_kernel, a, out, out_cap);
  if (e != cudaSuccess) return e;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_encode(const ScanPlan& plan, const uint8_t* text, uint64_t n,
                          const uint8_t* map, uint32_t* codes, cudaStream_t stream) {
  const uint64_t nq = n / plan.q;
  if (nq == 0) return cudaSuccess;
  const int threads = 256;
  uint64_t blocks = (nq + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  (void)cudaGetLastError();
  mag_encode_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(plan, text, nq, map,
                                                                           codes);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

unsigned long long kernel_launch_count() { return g_launches.load(); }

}  // namespace magb
