// The general staged machine (mag_scan_kernel): exact-code plans with the
// reference's explicit (q, k, sigma', mapping), SMAG code arrays and the
// overlapping shiftor_og scan, m' >= 1.  One persistent kernel fuses the
// reference's three search stages:
//   stage 1  q-gram formation       (encode_gram_at qgram.hpp:30-36, or the
//                                     hashed q-gram alphabet of paper §3.3)
//   stage 2  superimposed Shift-Or   (FilterMachine::scan_range
//            over k alignments        filter.hpp:51-74, closed form)
//   stage 3  window verification     (candidate_window / verify_window
//            + ordered output          verify.hpp:21-31, sort_dedup :37-38)
//
// Every scanning warp is independent: it takes slices of the sample stream
// with an atomic ticket and streams each slice through its own ring of
// shared-memory slots with 1-D TMA bulk copies (cp.async.bulk, completion on
// a per-slot mbarrier).  The mask table, the verification prefilter and the
// byte map live in shared memory for the whole launch.  One sample per
// lane: the closed form of the packed Shift-Or, D_t = OR_i mask(t-i) << i,
// takes the previous samples' masks from neighbouring lanes (shuffles).
// Hits become candidate windows in a per-warp queue (warp-scan order = text
// order); windows are verified against a shared-memory prefilter and then the
// hashed pattern table in global memory.  Matches leave the warp already in
// (offset, pattern) order into the slice's staging area; the CTA's gather
// warp (kern_common.cuh) places the slices in the output.
//
// This header is included by scan_staged_{exact,hashed,codes}.cu, one gram
// mode each (MAG_STAGED_GM), so the ~60 instantiations compile in parallel.
#pragma once

#include "kern_common.cuh"

namespace magb {
namespace {

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
      ld_t = slice_t0(A, x);
      ld_tend = slice_t1(A, x);
      if (ld_t >= ld_tend) publish_slice(A, x, 0, lane);  // slice past the last sample
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
      in.flags = (t0 == slice_t0(A, ld_slice) ? 1u : 0u) | (t0 + nsamp == ld_tend ? 2u : 0u);
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
    if (!(A.plan.diag & 2)) fill = flush_queue(A, pq, pqn, pbase, out, fill, lane, false);
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
        publish_slice(A, in.slice, fill, lane);
      }
      __syncwarp();
      ++cons;
      issue();
    }
    scan_exit(A, cands + cands32, lane);
  }
};

template <int GM, typename E, bool TSMEM, int QW, int CMP, int CK, bool A4>
__global__ void __launch_bounds__(kMaxWarps * 32, 1) mag_scan_kernel(const __grid_constant__ ScanArgs A) {
  allow_gather(A);
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
template <int GM, typename E, bool TSMEM, int QW, int CMP = 0, int CK = 0, bool A4 = false>
cudaError_t launch_t(const ScanArgs& a, cudaStream_t st, int grid, size_t smem) {
  auto k = mag_scan_kernel<GM, E, TSMEM, QW, CMP, CK, A4>;
  cudaError_t e = allow_max_smem(reinterpret_cast<const void*>(k), smem);
  if (e != cudaSuccess) return e;
  (void)cudaGetLastError();  // a stale error of another runtime user (e.g. torch) is not ours
  k<<<grid, a.nwarps * 32, smem, st>>>(a);
  count_launch();
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
cudaError_t launch_e(const ScanArgs& a, cudaStream_t st, int grid) {
  const size_t smem = smem_layout(a.plan, a.slot_bytes, a.ring, a.nwarps).total;
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
}  // namespace magb
