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
  uint32_t h = x0 * 0x9E3779B1u + x1 * 0x85EBCA77u + x2 * 0xC2B2AE3Du + x3 * 0x27D4EB2Fu;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
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

// Verification key: polynomial hash of the first v bytes (v = min(m, 16)),
// H = sum b[i] * B^(v-1-i) mod 2^32, then a murmur3 finaliser.  Polynomial so
// the device can roll it across consecutive starts.
constexpr uint32_t kKeyBase = 0x01000193u;

MAG_HD uint32_t key_mix(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}

MAG_HD uint32_t key_poly(const uint8_t* p, unsigned v) {
  uint32_t h = 0;
  for (unsigned i = 0; i < v; ++i) h = h * kKeyBase + p[i];
  return h;
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
  uint32_t entry_log2;    // log2(bits per mask entry), 0..6
  uint64_t entries;       // number of mask entries
  uint64_t table_bytes;   // packed table size (multiple of 16)
  int table_in_smem;
  uint64_t match_mask;
  // verification
  uint32_t m, maxlen, key_len;
  uint32_t key_pow;       // kKeyBase^(key_len-1) mod 2^32, for rolling
  uint32_t pf_bits;       // prefilter bitmap has 2^pf_bits bits (smem)
  uint32_t bucket_bits;   // 2^bucket_bits buckets (global)
  uint32_t r;
};


// ---- shared-memory layout of the scan kernel (host computes the size,
// device carves it; one definition for both).
constexpr int kMaxWarps = 16;   // consumer warps per CTA
constexpr int kQueueCap = 64;   // candidate windows queued per warp

struct StageMeta {
  long long tile;               // -1: end of work
  unsigned long long excl;      // exclusive prefix of the tile (if excl_ready)
  unsigned int done;            // consumer warps finished with the tile
  unsigned int excl_ready;
  unsigned int direct_mask;     // warps that wrote straight to global
  unsigned int pad;
  unsigned int wc[kMaxWarps];   // per-warp match counts, ~0u = running
};

MAG_HD size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

struct SmemLayout {
  size_t table, pf, map, stage, mbuf, queue, meta, bars, total;
  uint32_t stage_bytes;
};

MAG_HD SmemLayout smem_layout(const ScanPlan& p, uint64_t tile_bytes, uint32_t halo,
                              uint32_t stages, uint32_t nwarps, uint32_t mbuf) {
  SmemLayout L;
  size_t o = 0;
  L.table = o;
  o += p.table_in_smem ? align16(p.table_bytes) : 0;
  L.pf = o;
  o += align16((size_t(1) << p.pf_bits) / 8);
  L.map = o;
  o += 256;
  L.stage_bytes = static_cast<uint32_t>(align16(tile_bytes + halo + 32));
  L.stage = o;
  o += size_t(stages) * L.stage_bytes;
  L.mbuf = o;
  o += size_t(stages) * nwarps * mbuf * 8;
  L.queue = o;
  o += align16(size_t(nwarps) * kQueueCap * 4);
  L.meta = o;
  o += align16(size_t(stages) * sizeof(StageMeta));
  L.bars = o;
  o += size_t(stages) * 2 * 8;
  L.total = o;
  return L;
}

}  // namespace magb
