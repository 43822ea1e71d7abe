// Shared host/device definitions of the B200 search path.
//
// Everything here must be bit-identical between the host (mask-table and
// pattern-table construction) and the device (text scan); the oracle in
// oracle/mag_oracle.c restates hash_gram() for the checker.
#pragma once

#include <stddef.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define MAG_HD __host__ __device__ __forceinline__
#else
#define MAG_HD inline
#endif

namespace magb {

// Gram modes of the filter's stage 1.
//   kGramExact : the reference's code, map(p[0]) + map(p[1])σ' + ...
//                (qgram.hpp:30-36), indexing σ'^q mask entries.
//   kGramHashed: the paper's q-gram-alphabet mapping by hashing (§3.3,
//                SPEC.md:132-135,232): raw q bytes (q <= 16) -> 2^table_bits
//                entries.  A coarsening of the identity-map code, so it only
//                adds candidates; the match set is unchanged.
enum GramMode : int { kGramExact = 0, kGramHashed = 1 };

// Packed output key: offset in the high 40 bits, pattern index in the low 24.
// Sorting keys ascending is exactly the (offset, pattern_index) order of
// core.hpp:38-41.
constexpr unsigned kPidBits = 24;
constexpr uint64_t kMaxPatterns = 1ull << kPidBits;
constexpr uint64_t kMaxText = 1ull << 40;

MAG_HD uint64_t pack_match(uint64_t offset, uint32_t pid) {
  return (offset << kPidBits) | pid;
}

// Filter-side gram hash over q <= 16 raw bytes given as four little-endian
// words with bytes past q already zeroed.  Must match mo_gram_hash().
MAG_HD uint32_t hash_gram_words(uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3) {
  // no final xorshift: table slots take the top bits (already mixed by the
  // multiply) and the L2 screen's low bits measured as selective without it
  uint32_t h = x0 * 0x9E3779B1u + x1 * 0x85EBCA77u + x2 * 0xC2B2AE3Du + x3 * 0x27D4EB2Fu;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  return h;
}

MAG_HD uint32_t hash_gram_bytes(const uint8_t* p, unsigned q) {
  uint32_t x[4] = {0, 0, 0, 0};
  for (unsigned i = 0; i < q; ++i) x[i >> 2] |= (uint32_t)p[i] << (8 * (i & 3));
  return hash_gram_words(x[0], x[1], x[2], x[3]);
}

MAG_HD uint32_t gram_slot(uint32_t h, unsigned table_bits) {
  return table_bits ? (h >> (32 - table_bits)) : 0u;
}

// Multi-probe hashed grams (1-bit entries, probes >= 2): the table is
// `blocks` 64-entry blocks; a gram owns `probes` entries of block
// (h * blocks) >> 32, at bits taken from a 64-bit mix of h, and is admitted
// only where all of them are admitted — an intersection of hashed q-gram
// alphabets (a blocked Bloom filter), which still never rejects a gram a
// pattern contributed.  Entry index = block * 64 + bit.
constexpr unsigned kMaxProbes = 8;
MAG_HD uint32_t bloom_block(uint32_t h, uint32_t blocks) {
  return static_cast<uint32_t>((static_cast<uint64_t>(h) * blocks) >> 32);
}
MAG_HD uint64_t bloom_mix(uint32_t h) { return static_cast<uint64_t>(h) * 0x9E3779B97F4A7C15ull; }
MAG_HD uint32_t bloom_bit(uint64_t g, unsigned i) { return static_cast<uint32_t>(g >> (58 - 6 * i)) & 63u; }

// Rolling q-gram hash of the dense (roll) scan: H(p) = sum_{j<q} t[p+j] *
// B^(q-1-j) mod 2^32, so H(p+1) = H(p)*B + t[p+q] - t[p]*B^q (two IMADs per
// position).  Its filter is a blocked Bloom filter of 32-bit words: word
// umulhi(H, words), bits 31 - (roll_probe_shift(H, i) & 31)
// for i < probes.  H itself picks the word (its top bits) and probe 0 (its
// low bits): a separate mixing multiply (round 1) cost one IMAD per position
// and bought 0.6% fewer candidates on cfg5.
constexpr uint32_t kRollB = 0x9E3779B1u;
constexpr int kRollMaxProbes = 4;
MAG_HD uint32_t roll_hash_bytes(const uint8_t* p, unsigned q) {
  uint32_t h = 0;
  for (unsigned i = 0; i < q; ++i) h = h * kRollB + p[i];
  return h;
}
MAG_HD uint32_t roll_pow(unsigned q) {
  uint32_t x = 1;
  for (unsigned i = 0; i < q; ++i) x *= kRollB;
  return x;
}
MAG_HD uint32_t roll_word(uint32_t g, uint32_t words) {
  return static_cast<uint32_t>((static_cast<uint64_t>(g) * words) >> 32);
}
MAG_HD uint32_t roll_probe_mul(int i) { return i == 1 ? 0x85EBCA77u : 0xC2B2AE3Du; }
// Shift selecting probe i of hash h (the probed bit is 31 - (shift & 31)).
MAG_HD uint32_t roll_probe_shift(uint32_t h, int i) {
  return i == 0 ? h
                : static_cast<uint32_t>((static_cast<uint64_t>(h) * roll_probe_mul(i)) >> 32);
}

// Verification key: the first v = min(m, 16) bytes of a start, read as four
// little-endian words (bytes past v zeroed), mixed.  Top bits index the
// shared-memory prefilter, low bits the bucket table.
MAG_HD uint32_t key_mix(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}

MAG_HD uint32_t key_words(uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3) {
  return key_mix(x0 * 0x9E3779B1u + x1 * 0x7FEB352Du + x2 * 0x846CA68Bu + x3 * 0x68E31DA4u);
}

MAG_HD uint32_t key_bytes(const uint8_t* p, unsigned v) {
  uint32_t x[4] = {0, 0, 0, 0};
  for (unsigned i = 0; i < v; ++i) x[i >> 2] |= (uint32_t)p[i] << (8 * (i & 3));
  return key_words(x[0], x[1], x[2], x[3]);
}

// L2 screen bit of a window key: its low l2_bits bits (one LOP).  For the
// direct kernel's key (the gram hash, whose top bits index the filter
// table) a filter hit fixes only the screen index's top 32 - 19 bits to an
// admitted key's, and ~r*q / 2^19 keys share those, so the screen stays as
// selective as an independent bitmap of the same density.
MAG_HD uint32_t screen_bit(uint32_t key, unsigned l2_bits) {
  return l2_bits >= 32 ? key : (key & ((1u << l2_bits) - 1u));
}

// Byte masks of the v-byte key per word.
MAG_HD uint32_t key_word_mask(unsigned v, unsigned word) {
  if (v >= 4 * (word + 1)) return 0xffffffffu;
  if (v <= 4 * word) return 0u;
  return (1u << (8 * (v - 4 * word))) - 1u;
}

// Scan plan shared by host and kernels (passed by value to the kernel).
struct ScanPlan {
  // geometry of the machine (filter.hpp:27-31)
  int overlapping;        // 1 = shiftor_og (gram step 1, window 1)
  int smag;               // 1 = gram indices come from the prepared code array
  int gram_mode;          // GramMode
  int verify_all;         // 1 = table admits everything (q=k=m'=1): no filter work
  uint32_t q, k, m_prime;
  uint32_t sigma_prime;
  uint32_t table_bits;    // hashed: log2(entries)
  uint32_t probes;        // hashed, m' = k = 1: entries probed per gram (1..kMaxProbes)
  uint32_t blocks;        // probes >= 2: 64-entry blocks in the table
  int direct;             // aligned-sample stream kernel (W = q = 16 or 8)
  uint32_t ddepth;        // direct: TMA ring depth per warp (0 = kDirectDepth)
  int roll;               // dense rolling-hash scan: every position, q-gram Bloom
  uint32_t roll_words;    // roll: 32-bit Bloom words (table_bytes = 4 * roll_words)
  uint32_t roll_step;     // roll: positions per step (kRollStepEq for equal-length short sets, else kRollStep)
  int pack2;              // dense 2-bit-code scan (<= 4 pattern symbols): every position
  uint32_t pack_shift;    // pack2: symbol map b -> (b >> pack_shift) & 3
  uint32_t vbits;         // pack2: log2 level-2 slots
  uint32_t entry_log2;    // log2(bits per mask entry), 0..6
  uint64_t entries;       // number of mask entries
  uint64_t table_bytes;   // packed table size (multiple of 16)
  int table_in_smem;
  uint64_t match_mask;
  // verification
  uint32_t m, maxlen, key_len;
  // Window keys (strided plans, q > 1): the pattern table indexes every
  // (pattern, shift s < q) by the wkey_len bytes p[s, s + wkey_len); a
  // candidate window is checked with ONE key read at its gram boundary q*ss,
  // each hit naming the start q*ss - s directly.
  int window_key;
  uint32_t wkey_len;
  // key_gram: window keys are 16 bytes hashed with hash_gram_words (the
  // filter's own gram hash: q = 16 direct plans reuse one hash per sample)
  int key_gram;
  // Window keys are screened by an L2-resident bitmap of 2^l2_bits bits
  // (bit = screen_bit(key)) before any bucket walk; 0 = no bitmap.
  uint32_t l2_bits;
  // diagnostics only (builds with -DMAG_B200_DIAGNOSTICS read MAG_B200_DIAG;
  // product builds always pass 0): bits skip stages for profiling
  int diag;
  uint32_t pf_bits;       // prefilter bitmap has 2^pf_bits bits (smem)
  uint32_t bucket_bits;   // 2^bucket_bits buckets (global)
  uint32_t r;
};


// ---- shared-memory layout of the scan kernel (host computes the size,
// device carves it; one definition for both).
constexpr int kMaxWarps = 16;   // launch bound: 512 threads (the roll kernel's equal-length path: up to kRollMaxWarps)
constexpr int kQueueCap = 64;   // candidate windows queued per warp (per chunk)
constexpr int kProbeCap = 128;  // window keys awaiting the L2 screen (per slice)
constexpr int kHitWords = 32;   // per-chunk hit bitmap (chunks of <= 1024 samples, k = 1)

// Per ring slot: what the staged bytes are.
struct SlotInfo {
  unsigned long long slice;     // owning slice
  unsigned long long t0;        // first sample of this chunk
  unsigned long long src;       // absolute offset of slot byte 0
  unsigned int nsamp;           // samples [t0, t0 + nsamp)
  unsigned int valid;           // staged bytes
  unsigned int flags;           // 1: first chunk of its slice, 2: last chunk
  unsigned int pad;
};

MAG_HD size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

struct SmemLayout {
  size_t table, pf, map, slots, info, queue, probe, hits, bars, total;
};

// Direct (q = 16) kernel: resident table, per-warp probe queue, and a ring
// of kDirectDepth 1 KiB step buffers (+ mbarriers) per warp.
constexpr int kDirectDepth = 4;
// Ring depth of the direct kernel: the plan's (2..4).
MAG_HD int direct_depth(const ScanPlan& p, uint32_t /*nwarps*/) {
  return p.ddepth >= 2 && p.ddepth <= 4 ? static_cast<int>(p.ddepth) : kDirectDepth;
}
// Text bytes per direct-kernel step: 256 16-byte samples or 256 8-byte
// samples (8 per lane either way).
MAG_HD uint32_t direct_step_bytes(uint32_t q) { return q == 8 ? 2048u : 4096u; }
constexpr int kDirectProbeCap = 64;  // direct kernel: screened window keys queued per warp
MAG_HD size_t direct_smem(const ScanPlan& p, uint32_t nwarps) {
  return align16(p.table_bytes) + align16(size_t(nwarps) * kDirectProbeCap * 8) +
         size_t(nwarps) * direct_depth(p, nwarps) * (direct_step_bytes(p.q) + 16 + 8) + 64;
}

// Roll kernel: Bloom words, per-warp ring of kRollDepth slots of
// kRollStep text bytes + halo (+ mbarriers and step descriptors).
constexpr int kRollDepth = 2;
constexpr int kRollMaxWarps = 24;  // equal-length short sets (80-register kernel); others: kMaxWarps
constexpr int kRollStep = 2048;   // positions per step: 2 runs of 32 per lane
constexpr int kRollStepEq = 1024; // equal-length short sets: 1 run per lane (pipelined verification)
MAG_HD uint32_t roll_slot_bytes(uint32_t step, uint32_t halo) { return static_cast<uint32_t>(align16(step + halo)); }
constexpr int kRollList = 256;     // per-warp list of a step's hit positions (u16)
constexpr int kRollListEq = 128;
MAG_HD size_t roll_smem(uint32_t words, uint32_t halo, uint32_t nwarps, uint32_t step) {
  return align16(size_t(words) * 4) + size_t(nwarps) * kRollDepth * roll_slot_bytes(step, halo) +
         size_t(nwarps) * kRollDepth * (32 + 8) +
         size_t(nwarps) * (step == static_cast<uint32_t>(kRollStepEq) ? kRollListEq : kRollList) * 2 + 64;
}

// Pack2 kernel: 2^20-bit level-1 bitmap, per-warp ring of kPack2Depth slots
// of kPack2Step positions + halo, step descriptors, per-warp hit list.
constexpr int kPack2Step = 2048;
constexpr int kPack2Depth = 2;
constexpr int kPack2List = 256;   // listed level-1 hits per round (uint2 {code, position})
constexpr int kPack2Batch = 6;    // listed hits per lane with level-2 loads in flight
constexpr uint32_t kPack2L1Bits = 20;  // level-1 key: the first 10 symbols
MAG_HD size_t pack2_smem(uint64_t table_bytes, uint32_t halo, uint32_t nwarps) {
  return align16(table_bytes) + size_t(nwarps) * kPack2Depth * align16(kPack2Step + halo) +
         size_t(nwarps) * kPack2Depth * (32 + 8) + size_t(nwarps) * kPack2List * 8 + 64;
}
MAG_HD uint32_t pack2_code(const uint8_t* p, unsigned len, uint32_t shift) {
  uint32_t c = 0;
  for (unsigned i = 0; i < len; ++i) c |= ((static_cast<uint32_t>(p[i]) >> shift) & 3u) << (2 * i);
  return c;
}
MAG_HD uint32_t pack2_home(uint32_t code, uint32_t vbits) { return (code * 0x9E3779B1u) >> (32 - vbits); }

MAG_HD SmemLayout smem_layout(const ScanPlan& p, uint32_t slot_bytes, uint32_t ring,
                              uint32_t nwarps) {
  SmemLayout L;
  size_t o = 0;
  L.table = o;
  o += p.table_in_smem ? align16(p.table_bytes) : 0;
  L.pf = o;
  o += align16((size_t(1) << p.pf_bits) / 8);
  L.map = o;
  o += 256;
  L.slots = o;
  o += size_t(nwarps) * ring * slot_bytes;
  L.info = o;
  o += align16(size_t(nwarps) * ring * sizeof(SlotInfo));
  L.queue = o;
  o += align16(size_t(nwarps) * kQueueCap * 4);
  L.probe = o;
  o += align16(size_t(nwarps) * kProbeCap * 12);  // {key, pos} + prefetched screen word
  L.hits = o;
  o += align16(size_t(nwarps) * kHitWords * 4);
  L.bars = o;
  o += size_t(nwarps) * ring * 8;
  L.total = o;
  return L;
}

}  // namespace magb
