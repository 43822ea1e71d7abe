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

  // Rest of a linear-probe run after its home slot: bit 31 of a slot's len
  // word says whether the next slot is occupied.  Adds to c (first pid kept
  // in *first when c was 0), or writes from dst[idx + c].
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
      if (!(h.z >> 31)) break;
    }
    return c;
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
    if (A.plan.diag & 8) return;
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
        more[k] = occ && (hq[k].z >> 31);
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
          if (h.z >> 31) probe_rest(sw, valid, t + pr[k], pr[k], tx[k], key[k], out, fill + ex, w, nullptr);
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

// launch bound: 15 warps are launched (the gather kernel takes the 16th's registers)
constexpr int kRollThreads = 16 * 32;

template <int Q, int H>
__global__ void __launch_bounds__(kRollThreads, 1) mag_roll_kernel(const __grid_constant__ ScanArgs A) {
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
  if (a.nwarps * 32 > kRollThreads) return cudaErrorInvalidConfiguration;
  cudaError_t e = allow_max_smem(reinterpret_cast<const void*>(mag_roll_kernel<Q, H>), smem);
  if (e != cudaSuccess) return e;
  (void)cudaGetLastError();
  mag_roll_kernel<Q, H><<<grid, a.nwarps * 32, smem, stream>>>(a);
  count_launch();
  return cudaGetLastError();
}

template <int Q>
cudaError_t launch_roll_q(const ScanArgs& a, cudaStream_t stream, int grid, size_t smem) {
  if (a.plan.probes >= 3) return launch_roll_qh<Q, 3>(a, stream, grid, smem);
  if (a.plan.probes == 2) return launch_roll_qh<Q, 2>(a, stream, grid, smem);
  return launch_roll_qh<Q, 1>(a, stream, grid, smem);
}

}  // namespace

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

}  // namespace magb
