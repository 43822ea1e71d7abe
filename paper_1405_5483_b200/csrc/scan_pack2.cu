// Pack2 kernel: the dense scan for pattern sets over at most four symbols
// (DNA: cfg5, r = 100k patterns of m = 12).  It is the reference's own
// alphabet reduction to sigma' = 4 with exact q-gram codes: the code of a
// gram is sum map(t[i]) * 4^i (encode_gram_at, qgram.hpp:30-36), with the map
// b -> (b >> s) & 3, injective on the pattern alphabet (bytes outside it
// collide, which only adds candidates).  Every position p is a sample:
//   level 1: the code of its first 10 symbols (20 bits) indexes a 2^20-bit
//            bitmap resident in shared memory (one LDS, no hashing) -- the
//            reference's FilterMachine with exact codes, k = m' = 1;
//   level 2: the code of its first kb = min(m, 16) symbols (<= 32 bits)
//            probes an open-addressing table in L2 keyed by that exact code;
//            a slot holds {code, pattern id, length, first 16 pattern
//            bytes}, so a hit is one round trip and a byte compare.
// Codes come from the staged text packed 16 symbols per word (a shift, a
// mask and one multiply per 4 bytes), then one funnel shift per position.
// Level-1 hits (~9% of positions for cfg5) are listed per warp with their
// codes and verified with every lane busy.  Output as every scan kernel:
// per-slice ordered staging; the finish grid places it.
#include "kern_common.cuh"

namespace magb {
namespace {

struct __align__(16) P2Desc {
  unsigned long long t;  // first position (= byte offset) of the step
  uint32_t slice;
  uint32_t lim_flags;    // valid positions | flags << 16 (1 first, 2 last, 4 live)
  uint32_t valid;        // staged bytes
  uint32_t pad[3];
};

// 4 text bytes -> 4 two-bit codes in the top byte: t has 2-bit fields at
// bits 0, 8, 16, 24; the multiply by 2^24 + 2^18 + 2^12 + 2^6 moves them to
// 24, 26, 28, 30 with no other term reaching bits 24..31.
__device__ __forceinline__ uint32_t pack4_hi(uint32_t w, uint32_t s) {
  return ((w >> s) & 0x03030303u) * 0x01041040u;
}
// 16 bytes -> 16 codes, symbol i at bits 2i.
__device__ __forceinline__ uint32_t pack16(const uint4& v, uint32_t s) {
  const uint32_t a = pack4_hi(v.x, s), b = pack4_hi(v.y, s), c = pack4_hi(v.z, s), d = pack4_hi(v.w, s);
  return __byte_perm(__byte_perm(a, b, 0x0073u), __byte_perm(c, d, 0x0073u), 0x5410u);
}

struct Pack2Scanner {
  static constexpr int kRun = 32;  // positions per lane run (two runs per step)
  const ScanArgs& A;
  const int lane;
  uint32_t tbl_s;        // shared-window address of the level-1 bitmap
  uint2* list;           // [kPack2List] {code, position in step} of level-1 hits
  uint8_t* slots;
  uint64_t* bars;
  P2Desc* desc;
  const uint32_t slot_bytes;
  const uint32_t shift;  // symbol map b -> (b >> shift) & 3
  const uint32_t kmask;  // low 2 kb bits of a code
  uint32_t fill, cands32;
  uint64_t* out;
  unsigned long long p_t, p_end;
  uint32_t p_slice;
  bool p_done, p_first;
  uint64_t pol;

  __device__ Pack2Scanner(const ScanArgs& a, const void* tbl, uint8_t* sl, uint64_t* b, P2Desc* d, uint2* li, int l)
      : A(a), lane(l), tbl_s(smem_addr(tbl)), list(li), slots(sl), bars(b), desc(d),
        slot_bytes(static_cast<uint32_t>(align16(kPack2Step + a.back))), shift(a.plan.pack_shift),
        kmask(a.plan.key_len >= 16 ? 0xffffffffu : ((1u << (2 * a.plan.key_len)) - 1u)), fill(0), cands32(0),
        out(nullptr), p_t(0), p_end(0), p_slice(0), p_done(false), p_first(false), pol(policy_evict_first()) {}

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
      // every slice below num_slices holds samples (num_slices = ceil(samples / S))
      p_slice = static_cast<uint32_t>(x);
      p_t = slice_t0(A, x);
      p_end = slice_t1(A, x);
      p_first = true;
    }
    uint8_t* dst = slots + static_cast<size_t>(j) * slot_bytes;
    if (p_done) {
      if (lane == 0) desc[j].lim_flags = 0;
      __syncwarp();
      return;
    }
    const uint32_t lim = p_end - p_t < static_cast<unsigned long long>(kPack2Step) ? static_cast<uint32_t>(p_end - p_t)
                                                                                     : static_cast<uint32_t>(kPack2Step);
    const unsigned long long hi = p_t + slot_bytes < A.n ? p_t + slot_bytes : A.n;
    const uint32_t valid = static_cast<uint32_t>(hi - p_t);
    const uint32_t bulk = valid & ~15u;
    if (static_cast<uint32_t>(lane) < valid - bulk) dst[bulk + lane] = __ldg(A.text + p_t + bulk + lane);
    __syncwarp();
    if (lane == 0) {
      P2Desc& d = desc[j];
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

  // The lane's run at slot offset `base`: packed codes of its 32 + 15
  // symbols (pk[0..2]) and the level-1 verdicts (bit p = position base + p).
  __device__ __forceinline__ uint32_t filter_run(const uint8_t* sb, int base, uint32_t (&pk)[3]) const {
    const uint4* src = reinterpret_cast<const uint4*>(sb + base);
#pragma unroll
    for (int v = 0; v < 3; ++v) pk[v] = pack16(src[v], shift);
    uint32_t hits = 0;
#pragma unroll
    for (int p = 0; p < kRun; ++p) {
      const uint32_t lo = p < 16 ? pk[0] : pk[1], hi = p < 16 ? pk[1] : pk[2];
      const uint32_t code = __funnelshift_r(lo, hi, 2 * p);  // symbols p .. p + 15; bit test: code & 31
      const uint32_t w5 = code >> 5;                            // word: (code >> 5) & 0x7fff
      uint32_t addr, wd;
      asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(addr) : "r"(w5 & 0x7fffu), "r"(tbl_s));
      asm("ld.shared.u32 %0, [%1];" : "=r"(wd) : "r"(addr));
      hits = __funnelshift_r(hits, __funnelshift_r(wd, wd, code), 1);  // position p lands at bit p
    }
    return hits;
  }

  // The exact kb-symbol code of position p (0..31) of a run.
  static __device__ __forceinline__ uint32_t code_at(const uint32_t (&pk)[3], int p) {
    const uint32_t lo = p < 16 ? pk[0] : pk[1], hi = p < 16 ? pk[1] : pk[2];
    return __funnelshift_r(lo, hi, 2 * p);
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

  // One level-2 slot against a listed position: 1 = match.
  __device__ __forceinline__ bool slot_match(unsigned long long a, const uint4& t, uint32_t code, const uint4& h,
                                             const uint4& b) const {
    const uint32_t len = h.z & 0x7fffffffu;
    if (h.y == 0xffffffffu || h.x != code || a + len > A.n) return false;
    const uint32_t d = ((t.x ^ b.x) & key_word_mask(len, 0)) | ((t.y ^ b.y) & key_word_mask(len, 1)) |
                       ((t.z ^ b.z) & key_word_mask(len, 2)) | ((t.w ^ b.w) & key_word_mask(len, 3));
    return !d && (len <= 16 || equal_text(A, a, h.y, len));
  }

  __device__ __forceinline__ uint32_t home(uint32_t code) const { return pack2_home(code, A.plan.vbits); }

  // Rest of a probe run after the home slot (bit 31 of a slot's len word:
  // the next slot is occupied).  Counts (first pid kept when c was 0) or
  // writes from dst[idx + c].
  __device__ __noinline__ uint32_t probe_rest(unsigned long long a, const uint4& t, uint32_t code, uint64_t* dst,
                                              uint32_t idx, uint32_t c, uint32_t* first) const {
    uint32_t s = home(code);
    while (true) {
      s = (s + 1) & A.vmask;
      const uint4 h = __ldg(A.vtab + 2 * s);
      if (h.y == 0xffffffffu) break;
      const uint4 b = __ldg(A.vtab + 2 * s + 1);
      if (slot_match(a, t, code, h, b)) {
        if (dst && idx + c < A.slice_cap) dst[idx + c] = pack_match(a, h.y);
        if (c == 0 && first) *first = h.y;
        ++c;
      }
      if (!(h.z >> 31)) break;
    }
    return c;
  }

  // Level 2 + output of the listed hits [0, total) in text order,
  // kPack2Batch per lane at a time: the key halves of their home slots load
  // together (one round trip per batch), then the pattern-byte halves of the
  // code hits only, then the compares against the staged text.
  __device__ void verify_list(const uint32_t* sw, unsigned long long t, uint32_t total) {
    constexpr int kB = kPack2Batch;
    const uint4 empty = make_uint4(0, 0xffffffffu, 0, 0), zero = make_uint4(0, 0, 0, 0);
    for (uint32_t base = 0; base < total; base += 32 * kB) {
      uint32_t code[kB], pr[kB];
      uint4 hq[kB], bq[kB];
      bool hit[kB], more[kB];
#pragma unroll
      for (int k = 0; k < kB; ++k) {
        const uint32_t rank = base + 32 * k + lane;
        const bool live = rank < total;
        const uint2 e = live ? list[rank] : make_uint2(0u, 0u);
        code[k] = e.x & kmask;
        pr[k] = e.y;
        hq[k] = live ? __ldg(A.vtab + 2 * home(code[k])) : empty;
      }
#pragma unroll
      for (int k = 0; k < kB; ++k) {
        hit[k] = hq[k].y != 0xffffffffu && hq[k].x == code[k];
        more[k] = hq[k].y != 0xffffffffu && (hq[k].z >> 31);
        bq[k] = hit[k] ? __ldg(A.vtab + 2 * home(code[k]) + 1) : zero;
      }
#pragma unroll
      for (int k = 0; k < kB; ++k) {
        uint32_t c = 0, pid0 = hq[k].y;
        uint4 tx = zero;
        if (__any_sync(kFull, hit[k] || more[k])) {
          tx = text16(sw, pr[k]);
          c = hit[k] && slot_match(t + pr[k], tx, code[k], hq[k], bq[k]) ? 1u : 0u;
          if (__any_sync(kFull, more[k]) && more[k]) c = probe_rest(t + pr[k], tx, code[k], nullptr, 0, c, &pid0);
        }
        const unsigned one = __ballot_sync(kFull, c == 1u);
        if (!__any_sync(kFull, c > 1u)) {  // one pattern per start (the common case)
          if (c) {
            const uint32_t at = fill + __popc(one & ((1u << lane) - 1u));
            if (at < A.slice_cap) out[at] = pack_match(t + pr[k], pid0);
          }
          fill += __popc(one);
          continue;
        }
        // duplicate patterns: every (start, pid) of the probe run, in order
        const uint32_t ex = warp_excl_scan(c, lane);
        const uint32_t tc = __shfl_sync(kFull, ex + c, 31);
        if (c == 1) {
          if (fill + ex < A.slice_cap) out[fill + ex] = pack_match(t + pr[k], pid0);
        } else if (c > 1) {
          uint32_t w = 0;
          if (hit[k] && slot_match(t + pr[k], tx, code[k], hq[k], bq[k])) {
            if (fill + ex < A.slice_cap) out[fill + ex] = pack_match(t + pr[k], hq[k].y);
            w = 1;
          }
          if (more[k]) probe_rest(t + pr[k], tx, code[k], out, fill + ex, w, nullptr);
        }
        fill += tc;
      }
    }
  }

  // (the first kPack2Depth steps were staged before the bitmap load)
  __device__ void run() {
    uint32_t phase = 0;
    int j = 0;
#pragma unroll 1
    while (true) {
      const P2Desc d = desc[j];
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
      // both runs' level 1 (run r: positions [1024 r + 32 lane, + 32))
      uint32_t pk0[3], pk1[3];
      uint32_t h0 = filter_run(sb, 32 * lane, pk0);
      uint32_t h1 = filter_run(sb, 1024 + 32 * lane, pk1);
      auto keep = [&](int b) -> uint32_t {  // positions past the step's valid range never hit
        const int left = static_cast<int>(lim) - b;
        return left >= 32 ? 0xffffffffu : (left <= 0 ? 0u : ((1u << left) - 1u));
      };
      h0 &= keep(32 * lane);
      h1 &= keep(1024 + 32 * lane);
      // one list per step in text order: run 0's hits, then run 1's
      const uint32_t c0 = __popc(h0), c1 = __popc(h1);
      const uint32_t packed = warp_excl_scan(c0 | (c1 << 16), lane);
      const uint32_t tot = __shfl_sync(kFull, packed + (c0 | (c1 << 16)), 31);
      const uint32_t t0 = tot & 0xffffu, total = t0 + (tot >> 16);
      cands32 += c0 + c1;
      if (!(A.plan.diag & 8)) {
        for (uint32_t r0 = 0; r0 < total; r0 += kPack2List) {
          uint32_t idx = packed & 0xffffu;
          for (uint32_t m = h0; m; m &= m - 1, ++idx)
            if (idx >= r0 && idx < r0 + kPack2List) {
              const int p = __ffs(m) - 1;
              list[idx - r0] = make_uint2(code_at(pk0, p), 32u * lane + static_cast<uint32_t>(p));
            }
          idx = t0 + (packed >> 16);
          for (uint32_t m = h1; m; m &= m - 1, ++idx)
            if (idx >= r0 && idx < r0 + kPack2List) {
              const int p = __ffs(m) - 1;
              list[idx - r0] = make_uint2(code_at(pk1, p), 1024u + 32u * lane + static_cast<uint32_t>(p));
            }
          __syncwarp();
          verify_list(sw, d.t, min(total - r0, static_cast<uint32_t>(kPack2List)));
          __syncwarp();
        }
      }
      if (flags & 2u) publish_slice(A, d.slice, fill, lane);
      __syncwarp();
      produce(j);  // the slot is free again
      j = j + 1 == kPack2Depth ? 0 : j + 1;
    }
    scan_exit(A, cands32, lane);
  }
};

// launch bound: 512 threads (15 warps are launched)
constexpr int kPack2Threads = 16 * 32;

__global__ void __launch_bounds__(kPack2Threads, 1) mag_pack2_kernel(const __grid_constant__ ScanArgs A) {
  allow_gather(A);
  extern __shared__ __align__(128) uint8_t smem[];
  const size_t tbytes = align16(A.plan.table_bytes);
  const int warp = threadIdx.x >> 5, nw = static_cast<int>(A.nwarps);
  const uint32_t sbytes = static_cast<uint32_t>(align16(kPack2Step + A.back));
  uint8_t* p = smem + tbytes;
  uint8_t* slots = p + static_cast<size_t>(warp) * kPack2Depth * sbytes;
  p += static_cast<size_t>(nw) * kPack2Depth * sbytes;
  P2Desc* desc = reinterpret_cast<P2Desc*>(p) + static_cast<size_t>(warp) * kPack2Depth;
  p += static_cast<size_t>(nw) * kPack2Depth * sizeof(P2Desc);
  uint64_t* bars = reinterpret_cast<uint64_t*>(p) + static_cast<size_t>(warp) * kPack2Depth;
  p += static_cast<size_t>(nw) * kPack2Depth * 8;
  uint2* list = reinterpret_cast<uint2*>(p) + static_cast<size_t>(warp) * kPack2List;
  if ((threadIdx.x & 31) == 0) {
    for (int j = 0; j < kPack2Depth; ++j) mbar_init(bars + j, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  Pack2Scanner ps(A, smem, slots, bars, desc, list, threadIdx.x & 31);
  {  // the text of the first steps is in flight while the bitmap loads
#pragma unroll 1
    for (int j = 0; j < kPack2Depth; ++j) ps.produce(j);
    const uint4* src = static_cast<const uint4*>(A.table);
    uint4* dst = reinterpret_cast<uint4*>(smem);
    for (size_t i = threadIdx.x; i < tbytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    __syncthreads();
  }
  ps.run();
}

}  // namespace

cudaError_t launch_pack2(const ScanArgs& a, cudaStream_t stream, int grid) {
  if (a.nwarps * 32 > kPack2Threads) return cudaErrorInvalidConfiguration;
  const size_t smem = pack2_smem(a.plan.table_bytes, a.back, a.nwarps);
  cudaError_t e = allow_max_smem(reinterpret_cast<const void*>(mag_pack2_kernel), smem);
  if (e != cudaSuccess) return e;
  (void)cudaGetLastError();
  mag_pack2_kernel<<<grid, a.nwarps * 32, smem, stream>>>(a);
  count_launch();
  return cudaGetLastError();
}

}  // namespace magb
