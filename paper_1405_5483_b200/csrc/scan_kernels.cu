// B200 (sm_100a) search kernels for the MAG multiple pattern matcher.
//
// One persistent, warp-specialised kernel fuses the reference's three search
// stages over each text tile:
//   stage 1  q-gram formation       (encode_gram_at qgram.hpp:30-36, or the
//                                     hashed q-gram alphabet of §3.3)
//   stage 2  superimposed Shift-Or   (FilterMachine::scan_range
//            over k alignments        filter.hpp:51-74, closed form)
//   stage 3  window verification     (candidate_window / verify_window
//            + ordered output          verify.hpp:21-31, sort_dedup :37-38)
//
// Data movement: a producer warp streams text tiles (+ halo) into a ring of
// shared-memory stages with 1-D TMA bulk copies (cp.async.bulk + mbarrier
// complete_tx); consumer warps each own a contiguous slice of a tile.  The
// mask table, the verification prefilter and the byte map live in shared
// memory for the whole launch.  Candidates never leave the SM: they are
// compacted with warp ballots/scans into a per-warp queue and verified from
// the staged bytes against a hashed pattern table.  Matches come out already
// in (offset, pattern) order: each tile's total is published through a
// decoupled look-back, and the tile's matches are written at their final
// position, so no sort/merge pass is needed.
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "scan_launch.h"

namespace magb {
namespace {

std::atomic<unsigned long long> g_launches{0};

constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned long long kFlagA = 1ull << 62;  // aggregate published
constexpr unsigned long long kFlagP = 2ull << 62;  // inclusive prefix published
constexpr unsigned long long kValMask = (1ull << 62) - 1;

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
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
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long warp_sum64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ uint32_t warp_sum32(uint32_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
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

// ----------------------------------------------------------- look-back
// Exclusive prefix of `tile` over the published statuses of its
// predecessors (decoupled look-back).  Warp-collective; all lanes return it.
__device__ unsigned long long lookback_excl(const unsigned long long* status, long long tile,
                                            int lane) {
  unsigned long long excl = 0;
  long long j = tile - 1;
  while (j >= 0) {
    long long idx = j - lane;
    unsigned long long v = idx >= 0 ? ld_acquire(status + idx) : kFlagP;
    unsigned flag = static_cast<unsigned>(v >> 62);
    unsigned zero = __ballot_sync(kFull, flag == 0);
    unsigned pm = __ballot_sync(kFull, flag == 2);
    unsigned lim = kFull;
    if (pm) {
      int first = __ffs(pm) - 1;
      lim = first == 31 ? kFull : ((1u << (first + 1)) - 1);
    }
    if (zero & lim) {
      __nanosleep(64);
      continue;
    }
    unsigned long long val = ((lim >> lane) & 1u) ? (v & kValMask) : 0ull;
    excl += warp_sum64(val);
    if (pm) break;
    j -= 32;
  }
  return excl;
}

// ------------------------------------------------------------- kernel
struct Smem {
  const void* table;          // smem table (or null)
  const uint32_t* pf;         // prefilter bitmap
  const uint8_t* map;         // byte map
  uint8_t* stage;             // stage buffers
  uint64_t* mbuf;             // match buffers [stage][warp][mbuf]
  uint32_t* queue;            // per-warp window queue
  StageMeta* meta;
  uint64_t* full;
  uint64_t* empty;
  uint32_t stage_bytes;
};

__host__ __device__ inline SmemLayout make_layout(const ScanArgs& a) {
  return smem_layout(a.plan, a.tile_bytes, a.halo, a.stages, a.nwarps, a.mbuf);
}

// Gram formation modes for the kernel template.
enum KGram : int { kKExact = 0, kKHashed = 1, kKCodes = 2 };

template <int GM, typename E, bool TSMEM, int QW>
struct Scanner {
  const ScanArgs& A;
  const Smem& S;
  int lane, warp;
  // per-warp tile state
  const uint8_t* sb;            // stage base (== text[A0])
  const uint32_t* sw;           // stage as words
  long long A0;                 // first byte of the tile
  uint64_t stage_valid;         // staged bytes [A0, A0+stage_valid)
  uint64_t* buf;                // this warp's match buffer for the stage
  StageMeta* meta;
  long long tile;
  uint32_t bn;                  // matches in buf
  bool direct;
  unsigned long long dbase, written;
  unsigned long long cands;     // candidate counter (this warp, whole launch)
  long long own_lo, own_hi;     // owned start offsets, clipped to [0, n-m]
  long long S0;                 // first super position of the tile

  __device__ Scanner(const ScanArgs& a, const Smem& s, int l, int w)
      : A(a), S(s), lane(l), warp(w), cands(0) {}

  // ----------------------------------------------------------- stage 1+2
  __device__ __forceinline__ E table_entry(uint32_t idx) const {
    const uint32_t el = A.plan.entry_log2;
    if constexpr (sizeof(E) == 8) {
      const uint64_t* t = TSMEM ? static_cast<const uint64_t*>(S.table)
                                : static_cast<const uint64_t*>(A.table);
      return TSMEM ? t[idx] : __ldg(t + idx);
    } else {
      const uint32_t* t = TSMEM ? static_cast<const uint32_t*>(S.table)
                                : static_cast<const uint32_t*>(A.table);
      uint32_t word = TSMEM ? t[idx >> (5 - el)] : __ldg(t + (idx >> (5 - el)));
      uint32_t sh = (idx & ((32u >> el) - 1u)) << el;
      return word >> sh;
    }
  }

  // Mask index of the gram read by sample t.
  __device__ __forceinline__ uint32_t gram_index(long long t) const {
    const ScanPlan& P = A.plan;
    const long long u = P.overlapping ? t : (t + 1) * (long long)P.k - 1;
    if constexpr (GM == kKCodes) {
      return __ldg(A.codes + u);
    } else {
      const uint32_t rel = static_cast<uint32_t>((P.overlapping ? u : u * (long long)P.q) - A0);
      if constexpr (GM == kKHashed) {
        const uint32_t wi = rel >> 2, sh = (rel & 3u) << 3;
        uint32_t w[QW + 1];
#pragma unroll
        for (int i = 0; i <= QW; ++i) w[i] = sw[wi + i];
        uint32_t x[4] = {0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < QW; ++i) x[i] = __funnelshift_r(w[i], w[i + 1], sh);
        const uint32_t q = P.q;
        // zero bytes past q in the last word
        const uint32_t rem = q - 4u * (QW - 1);  // 1..4 bytes in the last word
        x[QW - 1] &= rem >= 4 ? 0xffffffffu : ((1u << (8 * rem)) - 1u);
        return hash_gram_words(x[0], x[1], x[2], x[3]) >> (32 - P.table_bits);
      } else {
        const uint32_t q = P.q, sp = P.sigma_prime;
        uint32_t code = S.map[sb[rel + q - 1]];
        for (int i = static_cast<int>(q) - 2; i >= 0; --i) code = code * sp + S.map[sb[rel + i]];
        return code;
      }
    }
  }

  __device__ __forceinline__ E mask_at(long long t, long long t_last) const {
    if (t < 0 || t > t_last) return static_cast<E>(~E(0));
    return table_entry(gram_index(t));
  }

  // ----------------------------------------------------------- stage 3
  __device__ __forceinline__ uint32_t byte_at(long long x) const {
    return sb[static_cast<uint32_t>(x - A0)];
  }

  __device__ __forceinline__ uint32_t key_direct(long long a) const {
    const uint32_t v = A.plan.key_len;
    uint32_t h = 0;
    for (uint32_t i = 0; i < v; ++i) h = h * kKeyBase + byte_at(a + i);
    return h;
  }

  __device__ __forceinline__ bool prefilter_pass(uint32_t key) const {
    const uint32_t pb = A.plan.pf_bits;
    const uint32_t i1 = key >> (32 - pb);
    const uint32_t i2 = ((key ^ (key >> 15)) * 0x2C1B3C6Du) >> (32 - pb);
    return ((S.pf[i1 >> 5] >> (i1 & 31)) & (S.pf[i2 >> 5] >> (i2 & 31)) & 1u) != 0;
  }

  // Exact byte comparison of pattern pid at text offset a (a+len <= n given).
  __device__ bool equal_at(long long a, uint32_t pid, uint32_t len) const {
    const uint8_t* p = A.pat_bytes + __ldg(A.pat_off + pid);
    const uint64_t rel = static_cast<uint64_t>(a - A0);
    if (rel + len <= stage_valid) {
      const uint32_t wi = static_cast<uint32_t>(rel >> 2), sh = static_cast<uint32_t>(rel & 3) << 3;
      const uint32_t* pw = reinterpret_cast<const uint32_t*>(p);
      for (uint32_t i = 0; i < len; i += 4) {
        uint32_t tw = __funnelshift_r(sw[wi + (i >> 2)], sw[wi + (i >> 2) + 1], sh);
        uint32_t pv = __ldg(pw + (i >> 2));
        uint32_t rem = len - i;
        uint32_t msk = rem >= 4 ? 0xffffffffu : ((1u << (8 * rem)) - 1u);
        if ((tw ^ pv) & msk) return false;
      }
      return true;
    }
    const uint8_t* t = A.text + a;
    for (uint32_t i = 0; i < len; ++i)
      if (__ldg(t + i) != __ldg(p + i)) return false;
    return true;
  }

  // Number of patterns matching at a whose key hash is `key`.
  __device__ uint32_t probe_count(long long a, uint32_t key) const {
    const uint32_t b = key & ((1u << A.plan.bucket_bits) - 1u);
    const uint32_t lo = __ldg(A.bucket_start + b), hi = __ldg(A.bucket_start + b + 1);
    uint32_t c = 0;
    for (uint32_t e = lo; e < hi; ++e) {
      uint2 ent = __ldg(A.bucket_entries + e);
      if (ent.x != key) continue;
      uint32_t len = __ldg(A.pat_len + ent.y);
      if (static_cast<uint64_t>(a) + len > A.n) continue;
      if (equal_at(a, ent.y, len)) ++c;
    }
    return c;
  }

  // Ordered emission of this warp's matches for one batch.
  __device__ void emit_matches(uint32_t cnt, long long a0, uint32_t flagged) {
    const uint32_t excl = warp_excl_scan(cnt, lane);
    const uint32_t total = __shfl_sync(kFull, excl + cnt, 31);
    if (total == 0) return;
    if (!direct && bn + total > A.mbuf) enter_direct();
    uint32_t pos = excl;
    while (flagged) {
      const int d = __ffs(flagged) - 1;
      flagged &= flagged - 1;
      const long long a = a0 + d;
      const uint32_t key = key_mix(key_direct(a));
      const uint32_t b = key & ((1u << A.plan.bucket_bits) - 1u);
      const uint32_t lo = __ldg(A.bucket_start + b), hi = __ldg(A.bucket_start + b + 1);
      for (uint32_t e = lo; e < hi; ++e) {
        uint2 ent = __ldg(A.bucket_entries + e);
        if (ent.x != key) continue;
        uint32_t len = __ldg(A.pat_len + ent.y);
        if (static_cast<uint64_t>(a) + len > A.n) continue;
        if (!equal_at(a, ent.y, len)) continue;
        const uint64_t k = pack_match(static_cast<uint64_t>(a), ent.y);
        if (direct) {
          const unsigned long long idx = dbase + written + pos;
          if (idx < A.out_cap) A.out[idx] = k;
        } else {
          buf[bn + pos] = k;
        }
        ++pos;
      }
    }
    if (direct)
      written += total;
    else
      bn += total;
    __syncwarp();
  }

  // Verifies windows [a0, a0+W) (one per lane), clipped to the owned starts.
  __device__ void verify_windows(bool active, long long a0, uint32_t W) {
    uint32_t cnt = 0, flagged = 0;
    if (active) {
      long long lo = a0 < own_lo ? own_lo : a0;
      long long hi = a0 + W - 1 > own_hi - 1 ? own_hi - 1 : a0 + W - 1;
      if (lo <= hi) {
        const uint32_t v = A.plan.key_len;
        uint32_t h = key_direct(lo);
        const uint32_t pw = A.plan.key_pow;
        for (long long a = lo;; ++a) {
          const uint32_t key = key_mix(h);
          if (prefilter_pass(key)) {
            uint32_t c = probe_count(a, key);
            if (c) {
              cnt += c;
              flagged |= 1u << static_cast<uint32_t>(a - a0);
            }
          }
          if (a == hi) break;
          h = (h - byte_at(a) * pw) * kKeyBase + byte_at(a + v);
        }
      }
    }
    if (__any_sync(kFull, cnt != 0)) emit_matches(cnt, a0, flagged);
  }

  // ------------------------------------------------------ output protocol
  __device__ void enter_direct() {
    // Exclusive prefix of the tile, then of this warp inside the tile.
    unsigned long long excl;
    if (*(volatile unsigned int*)&meta->excl_ready) {
      excl = *(volatile unsigned long long*)&meta->excl;
    } else {
      excl = lookback_excl(A.status, tile, lane);
      if (lane == 0) {
        *(volatile unsigned long long*)&meta->excl = excl;
        __threadfence_block();
        *(volatile unsigned int*)&meta->excl_ready = 1;
      }
    }
    uint32_t mine = 0;
    if (lane < warp) {
      volatile unsigned int* wc = &meta->wc[lane];
      unsigned int v;
      while ((v = *wc) == 0xffffffffu) __nanosleep(32);
      mine = v;
    }
    __syncwarp();
    __threadfence_block();
    dbase = excl + warp_sum32(mine);
    if (lane == 0) atomicOr(&meta->direct_mask, 1u << warp);
    for (uint32_t i = lane; i < bn; i += 32) {
      const unsigned long long idx = dbase + i;
      if (idx < A.out_cap) A.out[idx] = buf[i];
    }
    written = bn;
    bn = 0;
    direct = true;
    __syncwarp();
  }

  __device__ void finish_tile(int s) {
    const uint32_t count = direct ? static_cast<uint32_t>(written) : bn;
    unsigned int old = 0;
    if (lane == 0) {
      *(volatile unsigned int*)&meta->wc[warp] = count;
      __threadfence_block();
      old = atomicAdd(&meta->done, 1u);
      __threadfence_block();
    }
    old = __shfl_sync(kFull, old, 0);
    if (old != A.nwarps - 1) return;
    // Last warp of the tile: publish, look back, flush the buffered warps.
    uint32_t wv = lane < static_cast<int>(A.nwarps) ? *(volatile unsigned int*)&meta->wc[lane] : 0;
    const unsigned long long agg = warp_sum32(wv);
    unsigned long long excl;
    if (tile == 0) {
      excl = 0;
    } else if (*(volatile unsigned int*)&meta->excl_ready) {
      excl = *(volatile unsigned long long*)&meta->excl;
    } else {
      if (lane == 0) st_release(A.status + tile, kFlagA | agg);
      excl = lookback_excl(A.status, tile, lane);
    }
    if (lane == 0) {
      st_release(A.status + tile, kFlagP | (excl + agg));
      if (static_cast<unsigned long long>(tile) == A.num_tiles - 1) A.counters[2] = excl + agg;
    }
    const unsigned int dmask = *(volatile unsigned int*)&meta->direct_mask;
    unsigned long long run = excl;
    const uint64_t* sbuf = S.mbuf + static_cast<size_t>(s) * A.nwarps * A.mbuf;
    for (uint32_t v = 0; v < A.nwarps; ++v) {
      const uint32_t c = *(volatile unsigned int*)&meta->wc[v];
      if (!((dmask >> v) & 1u)) {
        const uint64_t* src = sbuf + static_cast<size_t>(v) * A.mbuf;
        for (uint32_t i = lane; i < c; i += 32) {
          const unsigned long long idx = run + i;
          if (idx < A.out_cap) A.out[idx] = src[i];
        }
      }
      run += c;
    }
    __syncwarp();
  }

  // ------------------------------------------------------ one tile slice
  __device__ void process(int s, long long tile_id) {
    const ScanPlan& P = A.plan;
    tile = tile_id;
    meta = S.meta + s;
    sb = S.stage + static_cast<size_t>(s) * S.stage_bytes;
    sw = reinterpret_cast<const uint32_t*>(sb);
    A0 = tile * static_cast<long long>(A.tile_bytes);
    const long long n = static_cast<long long>(A.n);
    long long A1 = A0 + static_cast<long long>(A.tile_bytes);
    if (A1 > n) A1 = n;
    stage_valid = static_cast<uint64_t>(
        (A0 + A.tile_bytes + A.halo > A.n ? A.n : A0 + A.tile_bytes + A.halo) - A0);
    buf = S.mbuf + (static_cast<size_t>(s) * A.nwarps + warp) * A.mbuf;
    bn = 0;
    direct = false;
    written = 0;

    const long long gs = P.overlapping ? 1 : P.q;
    const long long Wn = P.overlapping ? 1 : P.q;  // starts per window
    S0 = A0 / gs;
    const long long S1 = (A1 == n) ? (n + gs - 1) / gs : A1 / gs;
    const long long span = S1 - S0;
    const long long s_lo = S0 + span * warp / A.nwarps;
    const long long s_hi = S0 + span * (warp + 1) / A.nwarps;
    own_lo = s_lo * gs;
    own_hi = (warp == static_cast<int>(A.nwarps) - 1) ? A1 : s_hi * gs;
    const long long last_start = n - static_cast<long long>(P.m);  // inclusive
    if (own_hi > last_start + 1) own_hi = last_start + 1;

    if (P.verify_all) {
      // Every start is a candidate (q = k = m' = 1 with an all-admitting
      // table): windows of 16 consecutive starts, one per lane.
      for (long long base = own_lo; base < own_hi; base += 32 * 16) {
        const long long a0 = base + 16LL * lane;
        verify_windows(a0 < own_hi, a0, 16);
      }
    } else if (s_lo < s_hi) {
      scan_slice(s_lo, s_hi, gs, Wn);
    }
    finish_tile(s);
  }

  // Filter the slice's samples, queue candidate windows in order, verify.
  __device__ void scan_slice(long long s_lo, long long s_hi, long long gs, long long Wn) {
    const ScanPlan& P = A.plan;
    const int mp = static_cast<int>(P.m_prime);
    const int ov = mp - 1;
    const long long k = P.k;
    const long long T = static_cast<long long>(A.samples);
    // verified super positions: [s_lo, s_ver]; counted: [s_lo, s_hi)
    const long long s_ver = P.overlapping ? s_hi - 1 : s_hi;
    long long t_first, t_last;
    if (P.overlapping) {
      t_first = s_lo + ov;
      t_last = s_ver + ov;
    } else {
      t_first = s_lo / k + ov;
      t_last = s_ver / k + ov;
    }
    if (t_last > T - 1) t_last = T - 1;
    if (t_first > t_last) return;
    uint32_t* queue = S.queue + warp * kQueueCap;
    uint32_t qlen = 0;
    const E mm = static_cast<E>(P.match_mask);
    const bool shuffle_path = mp <= 16;
    const long long adv = shuffle_path ? 32 - ov : 32;
    const long long start = shuffle_path ? t_first - ov : t_first;
    for (long long base = start; base + (shuffle_path ? ov : 0) <= t_last; base += adv) {
      const long long t = base + lane;
      E D;
      if (shuffle_path) {
        const E M = mask_at(t, t_last);
        D = M;
        for (int i = 1; i <= ov; ++i) D |= static_cast<E>(shfl_up_e(M, i) << i);
      } else {
        D = static_cast<E>(0);
        for (int i = 0; i < mp; ++i) D |= static_cast<E>(mask_at(t - i, t_last) << i);
      }
      E hits = static_cast<E>(0);
      const bool out_lane = (shuffle_path ? lane >= ov : true) && t >= t_first && t <= t_last;
      if (out_lane) hits = static_cast<E>(~D) & mm;
      // candidates of this lane, ascending super position (alignment j descending)
      uint32_t cnt = 0;
      long long ss_base = P.overlapping ? t - ov : (t - ov) * k;
      {
        E h = hits;
        while (h) {
          const int bit = top_bit(h);
          h &= static_cast<E>(~(E(1) << bit));
          const long long j = bit / mp;
          const long long ss = P.overlapping ? ss_base : ss_base + (k - 1 - j);
          if (ss < s_lo || ss > s_ver) continue;
          if (ss < s_hi) ++cands;
          ++cnt;
        }
      }
      const uint32_t excl = warp_excl_scan(cnt, lane);
      const uint32_t total = __shfl_sync(kFull, excl + cnt, 31);
      uint32_t done = 0;
      while (done < total) {
        if (qlen == kQueueCap) {
          drain(queue, qlen, gs, Wn);
          qlen = 0;
        }
        const uint32_t take = min(kQueueCap - qlen, total - done);
        if (cnt) {
          uint32_t rank = excl;
          E h = hits;
          while (h) {
            const int bit = top_bit(h);
            h &= static_cast<E>(~(E(1) << bit));
            const long long j = bit / mp;
            const long long ss = P.overlapping ? ss_base : ss_base + (k - 1 - j);
            if (ss < s_lo || ss > s_ver) continue;
            if (rank >= done && rank < done + take)
              queue[qlen + rank - done] = static_cast<uint32_t>(ss - S0);
            ++rank;
          }
        }
        __syncwarp();
        qlen += take;
        done += take;
      }
    }
    if (qlen) drain(queue, qlen, gs, Wn);
  }

  __device__ void drain(const uint32_t* queue, uint32_t qlen, long long gs, long long Wn) {
    __syncwarp();
    for (uint32_t i0 = 0; i0 < qlen; i0 += 32) {
      const uint32_t i = i0 + lane;
      const bool act = i < qlen;
      long long a0 = 0;
      if (act) {
        const long long ss = S0 + queue[i];
        a0 = A.plan.overlapping ? ss : gs * ss - (Wn - 1);
      }
      verify_windows(act, a0, static_cast<uint32_t>(Wn));
    }
    __syncwarp();
  }
};

template <int GM, typename E, bool TSMEM, int QW>
__global__ void __launch_bounds__((kMaxWarps + 1) * 32, 1)
    mag_scan_kernel(const __grid_constant__ ScanArgs A) {
  extern __shared__ __align__(128) uint8_t smem[];
  const SmemLayout L = make_layout(A);
  Smem S;
  S.table = smem + L.table;
  S.pf = reinterpret_cast<const uint32_t*>(smem + L.pf);
  S.map = smem + L.map;
  S.stage = smem + L.stage;
  S.mbuf = reinterpret_cast<uint64_t*>(smem + L.mbuf);
  S.queue = reinterpret_cast<uint32_t*>(smem + L.queue);
  S.meta = reinterpret_cast<StageMeta*>(smem + L.meta);
  S.full = reinterpret_cast<uint64_t*>(smem + L.bars);
  S.empty = S.full + A.stages;
  S.stage_bytes = L.stage_bytes;

  // Resident tables: mask table, prefilter, byte map.
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
    if (tid == 0) {
      for (uint32_t s = 0; s < A.stages; ++s) {
        mbar_init(S.full + s, 1);
        mbar_init(S.empty + s, A.nwarps);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t NS = A.stages;
  unsigned long long* ticket = A.ticket;

  if (warp == static_cast<int>(A.nwarps)) {
    // ---------------- producer warp: tile tickets + TMA bulk loads
    if (lane == 0) {
      for (uint32_t it = 0;; ++it) {
        const uint32_t s = it % NS, ph = (it / NS) & 1u;
        mbar_wait(S.empty + s, ph ^ 1u);
        long long tile = static_cast<long long>(A.tile_begin + atomicAdd(ticket, 1ull));
        if (tile >= static_cast<long long>(A.tile_end)) tile = -1;
        StageMeta* m = S.meta + s;
        m->tile = tile;
        m->done = 0;
        m->excl_ready = 0;
        m->direct_mask = 0;
        for (int w = 0; w < kMaxWarps; ++w) m->wc[w] = 0xffffffffu;
        if (tile < 0) {
          mbar_arrive(S.full + s);
          break;
        }
        const uint64_t a0 = static_cast<uint64_t>(tile) * A.tile_bytes;
        uint64_t end = a0 + A.tile_bytes + A.halo;
        if (end > A.n) end = A.n;
        const uint32_t len = static_cast<uint32_t>(end - a0);
        const uint32_t bulk = len & ~15u;
        uint8_t* dst = S.stage + static_cast<size_t>(s) * S.stage_bytes;
        for (uint32_t i = bulk; i < len; ++i) dst[i] = __ldg(A.text + a0 + i);
        mbar_arrive_expect_tx(S.full + s, bulk);
        if (bulk) tma_load_1d(dst, A.text + a0, bulk, S.full + s);
      }
    }
    return;
  }

  // ---------------- consumer warps
  Scanner<GM, E, TSMEM, QW> sc(A, S, lane, warp);
  for (uint32_t it = 0;; ++it) {
    const uint32_t s = it % NS, ph = (it / NS) & 1u;
    mbar_wait(S.full + s, ph);
    const long long tile = *(volatile long long*)&S.meta[s].tile;
    if (tile < 0) break;
    sc.process(static_cast<int>(s), tile);
    __syncwarp();
    if (lane == 0) mbar_arrive(S.empty + s);
  }
  const unsigned long long c = warp_sum64(sc.cands);
  if (lane == 0 && c) atomicAdd(A.counters + 1, c);
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

template <int GM, typename E, bool TSMEM, int QW>
cudaError_t launch_t(const ScanArgs& a, cudaStream_t st, int grid, size_t smem) {
  auto k = mag_scan_kernel<GM, E, TSMEM, QW>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  k<<<grid, (a.nwarps + 1) * 32, smem, st>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <int GM, typename E, bool TSMEM>
cudaError_t launch_qw(const ScanArgs& a, cudaStream_t st, int grid, size_t smem) {
  if constexpr (GM == kKHashed) {
    switch ((a.plan.q + 3) / 4) {
      case 1: return launch_t<GM, E, TSMEM, 1>(a, st, grid, smem);
      case 2: return launch_t<GM, E, TSMEM, 2>(a, st, grid, smem);
      case 3: return launch_t<GM, E, TSMEM, 3>(a, st, grid, smem);
      default: return launch_t<GM, E, TSMEM, 4>(a, st, grid, smem);
    }
  } else {
    return launch_t<GM, E, TSMEM, 1>(a, st, grid, smem);
  }
}

template <int GM>
cudaError_t launch_e(const ScanArgs& a, cudaStream_t st, int grid, size_t smem) {
  const bool wide = a.plan.entry_log2 == 6;
  if constexpr (GM == kKHashed) {
    // hashed tables are always sized to shared memory
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
  s.smem_bytes = make_layout(a).total;
  s.threads = (a.nwarps + 1) * 32;
  return s;
}

cudaError_t launch_scan(const ScanArgs& a, cudaStream_t stream, int grid) {
  const size_t smem = make_layout(a).total;
  if (a.plan.smag) return launch_e<kKCodes>(a, stream, grid, smem);
  if (a.plan.gram_mode == kGramHashed) return launch_e<kKHashed>(a, stream, grid, smem);
  return launch_e<kKExact>(a, stream, grid, smem);
}

cudaError_t launch_encode(const ScanPlan& plan, const uint8_t* text, uint64_t n,
                          const uint8_t* map, uint32_t* codes, cudaStream_t stream) {
  const uint64_t nq = n / plan.q;
  if (nq == 0) return cudaSuccess;
  const int threads = 256;
  uint64_t blocks = (nq + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  mag_encode_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(plan, text, nq, map,
                                                                           codes);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

unsigned long long kernel_launch_count() { return g_launches.load(); }

}  // namespace magb
