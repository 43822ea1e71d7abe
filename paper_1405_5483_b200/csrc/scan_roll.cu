// Roll kernel: the dense scan for pattern sets whose q-grams saturate any
// strided filter (many short patterns, e.g. r = 100k, m = 12 over DNA).
// Replaces FilterMachine::scan_range + verify_window (filter.hpp:51-74,
// verify.hpp:28-31) for those plans with an every-position filter.
#include "kern_common.cuh"

namespace magb {
namespace {

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
// as every other scan kernel (mag_finish_kernel places the slices in order).
struct __align__(16) RollDesc {
  unsigned long long t;  // first position (= byte offset) of the step
  uint32_t slice;
  uint32_t lim_flags;    // valid positions | flags << 16 (1 first, 2 last, 4 live)
  uint32_t valid;        // staged bytes
  uint32_t pad[3];
};

// EQ: every pattern has the same length m = key_len <= 12: 1 KiB steps, a
// verification table of two-entry sectors and verification pipelined across
// steps (request / consume); other sets take verify_step.
template <int Q, int H, bool EQ>
struct RollScanner {
  static constexpr int kStep = EQ ? kRollStepEq : kRollStep;  // positions per step
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
  const uint32_t km0, km1, km2, km3;  // byte masks of the key_len-byte start key per word
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
        slot_bytes(roll_slot_bytes(kStep, a.back)),
        bq(roll_pow(Q)), km0(key_word_mask(a.plan.key_len, 0)), km1(key_word_mask(a.plan.key_len, 1)),
        km2(key_word_mask(a.plan.key_len, 2)), km3(key_word_mask(a.plan.key_len, 3)), fill(0), cands32(0), out(nullptr), p_t(0), p_end(0), p_slice(0), p_done(false),
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
      const unsigned long long t0 = slice_t0(A, x), t1 = slice_t1(A, x);
      if (t1 <= t0) {
        publish_slice(A, x, 0, lane);
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
    const uint32_t lim = p_end - p_t < static_cast<unsigned long long>(kStep)
                             ? static_cast<uint32_t>(p_end - p_t) : static_cast<uint32_t>(kStep);
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
  // brings each to bit 31; their AND's bit 31 is the verdict.  s_0 = h and
  // s_i = umulhi(h, C_i): the extra probes cost fma-pipe IMAD.HIs, not
  // alu-pipe shifts.
  __device__ __forceinline__ uint32_t test(uint32_t h) const {
    uint32_t addr, wd;
    asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(addr) : "r"(roll_word(h, A.plan.roll_words)), "r"(bloom_s));
    asm("ld.shared.u32 %0, [%1];" : "=r"(wd) : "r"(addr));
    uint32_t r = __funnelshift_l(wd, wd, h);
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
  // per verification slot — {len | F, pid, key, off} and the pattern's first 16
  // bytes sit in the same 32-byte sector; longer patterns finish against
  // the pattern bytes.  Counted (first pid kept), or written from dst[idx].
  // One verification slot against the candidate: 1 = match.
  __device__ __forceinline__ bool slot_match(const uint32_t* sw, uint32_t valid, unsigned long long a,
                                             uint32_t pr, const uint4& t, uint32_t key, const uint4& h,
                                             const uint4& b) const {
    const uint32_t len = h.x & 0x7fffffffu;
    if (h.z != key || a + len > A.n) return false;
    const uint32_t d = ((t.x ^ b.x) & key_word_mask(len, 0)) | ((t.y ^ b.y) & key_word_mask(len, 1)) |
                       ((t.z ^ b.z) & key_word_mask(len, 2)) | ((t.w ^ b.w) & key_word_mask(len, 3));
    if (d) return false;
    return len <= 16 || equal_slot(sw, valid, a, pr, h.y, len);
  }

  // Rest of a linear-probe run after its home slot, up to the first empty
  // slot.  Taken only when the home slot's len word has bit 31 set: some
  // pattern whose home this is lives further along (host_model.cpp gives
  // every home slot to one of its own patterns first, so ~1% of lookups come
  // here).  Adds to c (first pid kept in *first when c was 0), or writes
  // from dst[idx + c].
  __device__ __noinline__ uint32_t probe_rest(const uint32_t* sw, uint32_t valid, unsigned long long a, uint32_t pr,
                                              const uint4& t, uint32_t key, uint64_t* dst, uint32_t idx, uint32_t c,
                                              uint32_t* first) const {
    uint32_t s = key & A.vmask;
    while (true) {
      s = (s + 1) & A.vmask;
      const uint4 h = __ldg(A.vtab + 2 * s);
      if (h.y == 0xffffffffu) break;
      const uint4 b = __ldg(A.vtab + 2 * s + 1);
      if (slot_match(sw, valid, a, pr, t, key, h, b)) {
        if (dst && idx + c < A.slice_cap) dst[idx + c] = pack_match(a, h.y);
        if (c == 0 && first) *first = h.y;
        ++c;
      }
    }
    return c;
  }

  // ---- EQ sets (every pattern has the same length m <= 12): verification
  // pipelined across steps.  The verification table is 32-byte sectors of
  // two 16-byte entries {pattern, pid | F << 31} (host_model.cpp).  A step's
  // candidates (<= 64: two per lane) have their start masked, keyed and
  // their home sector requested (request()); the loads stay in flight while
  // the NEXT step is filtered and are decided by consume() after it, so the
  // L2 round trip is not waited for.  Denser steps and a slice's last step
  // are consumed at once.
  uint32_t pend_n = 0;            // warp-uniform: candidates in flight
  unsigned long long pend_t = 0;  // first position of their step
  uint32_t pend_pr[2];            // position within the step; 0xffffffff = no candidate
  uint32_t pend_tx[2][3];         // the start's 12 bytes, masked to the pattern length
  uint4 pend_e0[2], pend_e1[2];   // the home sector's entries

  static __device__ __forceinline__ bool entry_is(const uint4& e, uint32_t x, uint32_t y, uint32_t z) {
    return e.w != 0xffffffffu && ((e.x ^ x) | (e.y ^ y) | (e.z ^ z)) == 0u;
  }

  // Sectors after `home` up to the first one with a free entry (where pass 2
  // of the host build stopped): matches counted, or written from dst[idx].
  // The first two sectors are requested together.
  __device__ __noinline__ uint32_t walk(uint32_t x, uint32_t y, uint32_t z, uint32_t home, unsigned long long a,
                                        uint64_t* dst, uint32_t idx) const {
    uint32_t c = 0, s = home;
    uint4 n0 = __ldg(A.vtab + 2 * ((s + 1) & A.vmask)), n1 = __ldg(A.vtab + 2 * ((s + 1) & A.vmask) + 1);
    uint4 m0 = __ldg(A.vtab + 2 * ((s + 2) & A.vmask)), m1 = __ldg(A.vtab + 2 * ((s + 2) & A.vmask) + 1);
    while (true) {
      if (entry_is(n0, x, y, z)) {
        if (dst && idx + c < A.slice_cap) dst[idx + c] = pack_match(a, n0.w & 0xffffffu);
        ++c;
      }
      if (entry_is(n1, x, y, z)) {
        if (dst && idx + c < A.slice_cap) dst[idx + c] = pack_match(a, n1.w & 0xffffffu);
        ++c;
      }
      if (n0.w == 0xffffffffu || n1.w == 0xffffffffu) break;
      ++s;
      n0 = m0;
      n1 = m1;
      m0 = __ldg(A.vtab + 2 * ((s + 2) & A.vmask));
      m1 = __ldg(A.vtab + 2 * ((s + 2) & A.vmask) + 1);
    }
    return c;
  }

  __device__ __forceinline__ void consume() {
    if (pend_n == 0) return;
    const bool two = pend_n > 32;  // warp-uniform: the lanes' second candidates exist (20% of cfg5's steps)
    pend_n = 0;
    bool hit0[2], hit1[2];
    bool slow = false;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (k == 1 && !two) {
        hit0[1] = hit1[1] = false;
        continue;
      }
      const bool live = pend_pr[k] != 0xffffffffu;
      hit0[k] = live && entry_is(pend_e0[k], pend_tx[k][0], pend_tx[k][1], pend_tx[k][2]);
      hit1[k] = live && entry_is(pend_e1[k], pend_tx[k][0], pend_tx[k][1], pend_tx[k][2]);
      // walk on: the home sector overflowed; two outputs: duplicate patterns
      slow = slow || (live && pend_e0[k].w != 0xffffffffu && (pend_e0[k].w >> 31)) || (hit0[k] && hit1[k]);
    }
    if (!__any_sync(kFull, slow)) {  // the common case: at most one match, decided by the home sector
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (k == 1 && !two) continue;
        const bool hit = hit0[k] || hit1[k];
        const unsigned one = __ballot_sync(kFull, hit);
        if (hit) {
          const uint32_t at = fill + __popc(one & ((1u << lane) - 1u));
          const uint32_t pid = (hit0[k] ? pend_e0[k].w : pend_e1[k].w) & 0xffffffu;
          if (at < A.slice_cap) out[at] = pack_match(pend_t + pend_pr[k], pid);
        }
        fill += __popc(one);
      }
      return;
    }
    // count (home sector + the walk), then place in (start, pid) order
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (k == 1 && !two) continue;
      const bool live = pend_pr[k] != 0xffffffffu;
      const bool go = live && pend_e0[k].w != 0xffffffffu && (pend_e0[k].w >> 31);
      const unsigned long long a = pend_t + pend_pr[k];
      const uint32_t home = key_words(pend_tx[k][0], pend_tx[k][1], pend_tx[k][2], 0u) & A.vmask;
      uint32_t cw = 0;
      if (go) cw = walk(pend_tx[k][0], pend_tx[k][1], pend_tx[k][2], home, a, nullptr, 0);
      const uint32_t c = (hit0[k] ? 1u : 0u) + (hit1[k] ? 1u : 0u) + cw;
      const uint32_t ex = warp_excl_scan(c, lane);
      const uint32_t tc = __shfl_sync(kFull, ex + c, 31);
      uint32_t at = fill + ex;
      if (hit0[k]) {
        if (at < A.slice_cap) out[at] = pack_match(a, pend_e0[k].w & 0xffffffu);
        ++at;
      }
      if (hit1[k]) {
        if (at < A.slice_cap) out[at] = pack_match(a, pend_e1[k].w & 0xffffffu);
        ++at;
      }
      if (cw) walk(pend_tx[k][0], pend_tx[k][1], pend_tx[k][2], home, a, out, at);
      fill += tc;
    }
  }

  // Candidates of ranks [base, base + 64) of the step: start, key, sector loads.
  __device__ __forceinline__ void request(const uint32_t* sw, uint32_t base, uint32_t total, bool listed,
                                          uint32_t h, uint32_t excl, int tail) {
    uint32_t key[2];
    const bool two = total - base > 32;  // warp-uniform
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (k == 1 && !two) {
        pend_pr[1] = 0xffffffffu;
        key[1] = 0;
        continue;
      }
      const uint32_t rank = base + 32 * k + lane;
      bool live = rank < total;
      uint32_t pr;
      if (listed) {
        pr = live ? list[rank] : 0u;
      } else {  // dense step: rank search over the lanes' hit counts
        int o = 0;
#pragma unroll
        for (int step = 16; step; step >>= 1) {
          const uint32_t e = __shfl_sync(kFull, excl, o + step);
          if (e <= rank) o += step;
        }
        const uint32_t mo = __shfl_sync(kFull, h, o), eo = __shfl_sync(kFull, excl, o);
        pr = 32u * static_cast<uint32_t>(o) + static_cast<uint32_t>(__fns(mo, 0, static_cast<int>(rank - eo) + 1));
        if (!live) pr = 0;
      }
      live = live && static_cast<int>(pr) <= tail;
      const uint32_t wi = pr >> 2, sh = (pr & 3u) << 3;
      const uint32_t x0 = sw[wi], x1 = sw[wi + 1], x2 = sw[wi + 2], x3 = sw[wi + 3];
      pend_tx[k][0] = __funnelshift_r(x0, x1, sh) & km0;
      pend_tx[k][1] = __funnelshift_r(x1, x2, sh) & km1;
      pend_tx[k][2] = __funnelshift_r(x2, x3, sh) & km2;
      key[k] = key_words(pend_tx[k][0], pend_tx[k][1], pend_tx[k][2], 0u);
      pend_pr[k] = live ? pr : 0xffffffffu;
    }
    // all sector loads after all expansions (a later shuffle would otherwise
    // share a scoreboard with the earlier loads and serialise the trips);
    // lanes without a candidate read sector 0
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (k == 1 && !two) continue;
      const uint32_t sec = pend_pr[k] != 0xffffffffu ? key[k] & A.vmask : 0u;
      pend_e0[k] = __ldg(A.vtab + 2 * sec);
      pend_e1[k] = __ldg(A.vtab + 2 * sec + 1);
    }
  }

  // Expand the step's hit mask (bit p of lane l = position 32 l + p) in text
  // order and request its candidates' sectors.
  __device__ __forceinline__ void issue(const uint32_t* sw, unsigned long long t, uint32_t h) {
    const uint32_t c0 = __popc(h);
    const uint32_t incl = warp_excl_scan(c0, lane) + c0;
    const uint32_t excl = incl - c0, total = __shfl_sync(kFull, incl, 31);
    cands32 += c0;
    if (total == 0 || MAG_DIAG(A, 8)) return;
    // starts past n - m cannot hold a pattern (q < m plans sample them)
    const long long tl = static_cast<long long>(A.n) - static_cast<long long>(A.plan.m) - static_cast<long long>(t);
    const int tail = tl > 0xffff ? 0xffff : static_cast<int>(tl);  // negative: no start fits
    const bool listed = total <= static_cast<uint32_t>(kRollListEq);
    if (listed) {
      uint32_t idx = excl;
      for (uint32_t m = h; m; m &= m - 1) list[idx++] = static_cast<uint16_t>(32 * lane + __ffs(m) - 1);
      __syncwarp();
    }
    pend_t = t;
    if (total <= 64) {
      request(sw, 0, total, listed, h, excl, tail);
      pend_n = total;
      return;
    }
    for (uint32_t base = 0; base < total; base += 64) {  // dense step: in order, at once
      request(sw, base, total, listed, h, excl, tail);
      pend_n = total - base;
      consume();
    }
  }

  // Expand and verify a step's hits in text order: run 0 (positions
  // [32 l, 32 l + 32) of lane l) before run 1 ([1024 + 32 l, ...)).  Each
  // lane takes two candidates per batch (ranks base + lane, base + 32 +
  // lane), both verification-slot loads in flight together; the home slot
  // decides in straight-line code, the rare continued probe runs (and
  // duplicate pattern keys, c > 1) take the slow paths.
  __device__ void verify_step(const uint32_t* sw, uint32_t valid, unsigned long long t, uint32_t h0,
                              uint32_t h1) {
    const uint32_t c0 = __popc(h0), c1 = __popc(h1);
    const uint32_t packed = warp_excl_scan(c0 | (c1 << 16), lane);  // both prefix sums in one scan
    const uint32_t e0 = packed & 0xffffu, e1 = packed >> 16;
    const uint32_t tot = __shfl_sync(kFull, packed + (c0 | (c1 << 16)), 31);
    const uint32_t t0 = tot & 0xffffu, total = t0 + (tot >> 16);
    cands32 += c0 + c1;
    if (MAG_DIAG(A, 8)) return;
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
    const uint4 empty = make_uint4(0, 0xffffffffu, 0, 0);
    for (uint32_t base = 0; base < total; base += 64) {
      uint32_t pr[2], key[2], c[2], pid0[2];
      uint4 tx[2], hq[2], bq[2];
      bool live[2], more[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
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
          if (!live[k]) pr[k] = 0;
        }
        tx[k] = text16(sw, pr[k]);
        key[k] = key_of(tx[k]);
      }
      // all slot loads after all expansions (a later shuffle would otherwise
      // share a scoreboard with the earlier loads and serialise the trips)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const uint32_t slot = key[k] & A.vmask;
        hq[k] = live[k] ? __ldg(A.vtab + 2 * slot) : empty;
        bq[k] = live[k] ? __ldg(A.vtab + 2 * slot + 1) : empty;
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const bool occ = hq[k].y != 0xffffffffu;
        c[k] = occ && slot_match(sw, valid, t + pr[k], pr[k], tx[k], key[k], hq[k], bq[k]) ? 1u : 0u;
        pid0[k] = hq[k].y;
        more[k] = occ && (hq[k].x >> 31);
      }
      if (__any_sync(kFull, more[0] || more[1])) {
#pragma unroll
        for (int k = 0; k < 2; ++k)
          if (more[k]) c[k] = probe_rest(sw, valid, t + pr[k], pr[k], tx[k], key[k], nullptr, 0, c[k], &pid0[k]);
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const unsigned one = __ballot_sync(kFull, c[k] == 1u);
        if (!__any_sync(kFull, c[k] > 1u)) {  // one pattern per start (the common case)
          if (c[k]) {
            const uint32_t at = fill + __popc(one & ((1u << lane) - 1u));
            if (at < A.slice_cap) out[at] = pack_match(t + pr[k], pid0[k]);
          }
          fill += __popc(one);
          continue;
        }
        // duplicate pattern keys: every (start, pid) of the run, in order
        const uint32_t ex = warp_excl_scan(c[k], lane);
        const uint32_t tc = __shfl_sync(kFull, ex + c[k], 31);
        if (c[k] == 1) {
          if (fill + ex < A.slice_cap) out[fill + ex] = pack_match(t + pr[k], pid0[k]);
        } else if (c[k] > 1) {
          const uint32_t slot = key[k] & A.vmask;
          const uint4 h = __ldg(A.vtab + 2 * slot), b = __ldg(A.vtab + 2 * slot + 1);
          uint32_t w = 0;
          if (slot_match(sw, valid, t + pr[k], pr[k], tx[k], key[k], h, b)) {
            if (fill + ex < A.slice_cap) out[fill + ex] = pack_match(t + pr[k], h.y);
            w = 1;
          }
          if (h.x >> 31) probe_rest(sw, valid, t + pr[k], pr[k], tx[k], key[k], out, fill + ex, w, nullptr);
        }
        fill += tc;
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
      if constexpr (EQ) {
        uint32_t h = filter_run(sb, 32 * lane);
        const int mk = static_cast<int>(lim) - 32 * lane;  // positions past the step's valid range never hit
        h &= mk >= 32 ? 0xffffffffu : (mk <= 0 ? 0u : ((1u << mk) - 1u));
        consume();  // the previous step's candidates: their slots arrived during this filter
        issue(sw, d.t, h);
        if (flags & 2u) {
          consume();
          publish_slice(A, d.slice, fill, lane);
        }
        __syncwarp();
        produce(j);  // the slot is free again
        j = j + 1 == kRollDepth ? 0 : j + 1;
        continue;
      }
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
      if (flags & 2u) {
        publish_slice(A, d.slice, fill, lane);
      }
      __syncwarp();
      produce(j);  // the slot is free again
      j = j + 1 == kRollDepth ? 0 : j + 1;
    }
    scan_exit(A, cands32, lane);
  }
};

// NT: launch bound (512; 640 / 768 for the EQ kernel's 20- / 24-warp CTAs)
template <int Q, int H, bool EQ, int NT>
__global__ void __launch_bounds__(NT, 1) mag_roll_kernel(const __grid_constant__ ScanArgs A) {
  allow_gather(A);
  extern __shared__ __align__(128) uint8_t smem[];
  const size_t tbytes = align16(A.plan.table_bytes);
  {
    const uint4* src = static_cast<const uint4*>(A.table);
    uint4* dst = reinterpret_cast<uint4*>(smem);
    for (size_t i = threadIdx.x; i < tbytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5, nw = static_cast<int>(A.nwarps);
  const uint32_t sbytes = roll_slot_bytes(EQ ? kRollStepEq : kRollStep, A.back);
  uint8_t* p = smem + tbytes;
  uint8_t* slots = p + static_cast<size_t>(warp) * kRollDepth * sbytes;
  p += static_cast<size_t>(nw) * kRollDepth * sbytes;
  RollDesc* desc = reinterpret_cast<RollDesc*>(p) + static_cast<size_t>(warp) * kRollDepth;
  p += static_cast<size_t>(nw) * kRollDepth * sizeof(RollDesc);
  uint64_t* bars = reinterpret_cast<uint64_t*>(p) + static_cast<size_t>(warp) * kRollDepth;
  p += static_cast<size_t>(nw) * kRollDepth * 8;
  uint16_t* list = reinterpret_cast<uint16_t*>(p) + static_cast<size_t>(warp) * (EQ ? kRollListEq : kRollList);
  if ((threadIdx.x & 31) == 0) {
    for (int j = 0; j < kRollDepth; ++j) mbar_init(bars + j, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  RollScanner<Q, H, EQ> rs(A, reinterpret_cast<const uint32_t*>(smem), slots, bars, desc, list, threadIdx.x & 31);
  rs.run();
}

template <int Q, int H, bool EQ, int NT>
cudaError_t launch_roll_qhen(const ScanArgs& a, cudaStream_t stream, int grid, size_t smem) {
  if (a.nwarps * 32 > NT) return cudaErrorInvalidConfiguration;
  cudaError_t e = allow_max_smem(reinterpret_cast<const void*>(mag_roll_kernel<Q, H, EQ, NT>), smem);
  if (e != cudaSuccess) return e;
  (void)cudaGetLastError();
  mag_roll_kernel<Q, H, EQ, NT><<<grid, a.nwarps * 32, smem, stream>>>(a);
  count_launch();
  return cudaGetLastError();
}

template <int Q, int H, bool EQ>
cudaError_t launch_roll_qhe(const ScanArgs& a, cudaStream_t stream, int grid, size_t smem) {
  if constexpr (EQ && H == 3) {  // the planner's probes for large sets
    if (a.nwarps > 20) return launch_roll_qhen<Q, H, EQ, 768>(a, stream, grid, smem);
    if (a.nwarps > 16) return launch_roll_qhen<Q, H, EQ, 640>(a, stream, grid, smem);
  }
  return launch_roll_qhen<Q, H, EQ, 512>(a, stream, grid, smem);
}

template <int Q, int H>
cudaError_t launch_roll_qh(const ScanArgs& a, cudaStream_t stream, int grid, size_t smem) {
  // equal-length sets of at most 12 bytes: two-entry sectors, pipelined verification
  if (a.plan.maxlen == a.plan.m && a.plan.m <= 12 && a.plan.key_len == a.plan.m)
    return launch_roll_qhe<Q, H, true>(a, stream, grid, smem);
  return launch_roll_qhe<Q, H, false>(a, stream, grid, smem);
}

template <int Q>
cudaError_t launch_roll_q(const ScanArgs& a, cudaStream_t stream, int grid, size_t smem) {
  if (a.plan.probes >= 3) return launch_roll_qh<Q, 3>(a, stream, grid, smem);
  if (a.plan.probes == 2) return launch_roll_qh<Q, 2>(a, stream, grid, smem);
  return launch_roll_qh<Q, 1>(a, stream, grid, smem);
}

}  // namespace

cudaError_t launch_roll(const ScanArgs& a, cudaStream_t stream, int grid) {
  const bool eq = a.plan.maxlen == a.plan.m && a.plan.m <= 12 && a.plan.key_len == a.plan.m;
  if (a.plan.roll_step != static_cast<uint32_t>(eq ? kRollStepEq : kRollStep)) return cudaErrorInvalidValue;
  const size_t smem = roll_smem(a.plan.roll_words, a.back, a.nwarps, a.plan.roll_step);
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

}  // namespace magb
