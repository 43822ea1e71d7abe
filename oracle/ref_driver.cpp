// TEST INFRASTRUCTURE ONLY — never linked into, or called by, the product path.
//
// A thin extern "C" shim over the reference's own compiled sources, built by
// oracle/Makefile from /root/reference/proj/src/*.cpp (unmodified, in place)
// into oracle/_ref/libmagref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's reference/cpu_baseline arm may load it.
//
// What the reference ships with bodies is what we expose:
//   - naive_search / AhoCorasick / ac_search   proj/src/oracles.cpp:9-99
//   - AlphabetMap::{identity,frequency,balanced,lowbits}, Histogram
//                                              proj/src/alphabet_map.cpp:18-114
//   - GramConfig, encode_gram, encode_text, factor_pattern(_overlapping)
//                                              proj/src/qgram.cpp:7-64
//   - SuperPattern, materialize_classes, class_match_count
//                                              proj/src/superimpose.cpp:7-52
//   - PatternSet::validate                     proj/src/core.cpp:7-23
// The engine, filter constructor, verifier and tuner have no bodies in the
// reference and are restated in oracle/mag_oracle.c instead.

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "mag/alphabet_map.hpp"
#include "mag/core.hpp"
#include "mag/oracles.hpp"
#include "mag/qgram.hpp"
#include "mag/superimpose.hpp"

namespace {

thread_local std::string g_err;

std::vector<std::string> unpack(const uint8_t* bytes, const size_t* lens, size_t r) {
  std::vector<std::string> out;
  out.reserve(r);
  size_t off = 0;
  for (size_t i = 0; i < r; ++i) {
    out.emplace_back(reinterpret_cast<const char*>(bytes) + off, lens[i]);
    off += lens[i];
  }
  return out;
}

// Copies an occurrence list into two malloc'd arrays owned by the caller.
int emit(const std::vector<mag::Occurrence>& occ, uint64_t** offs, uint32_t** pids,
         size_t* count) {
  *count = occ.size();
  *offs = static_cast<uint64_t*>(std::malloc(std::max<size_t>(1, occ.size()) * 8));
  *pids = static_cast<uint32_t*>(std::malloc(std::max<size_t>(1, occ.size()) * 4));
  if (!*offs || !*pids) return -1;
  for (size_t i = 0; i < occ.size(); ++i) {
    (*offs)[i] = occ[i].offset;
    (*pids)[i] = occ[i].pattern_index;
  }
  return 0;
}

mag::AlphabetMap make_map(int strategy, const mag::Histogram& h, uint32_t sigma_prime,
                          unsigned lowbits) {
  switch (strategy) {
    case 0: return mag::AlphabetMap::identity();
    case 1: return mag::AlphabetMap::frequency(h, sigma_prime);
    case 2: return mag::AlphabetMap::balanced(h, sigma_prime);
    case 3: return mag::AlphabetMap::lowbits(lowbits);
  }
  throw mag::config_error("unknown mapping strategy");
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_free(void* p) { std::free(p); }

// Reference naive_search (oracles.cpp:9-21). Returns 0, or -1 on a
// validation error (message in ref_last_error()).
int ref_naive_search(const uint8_t* text, size_t n, const uint8_t* pat_bytes,
                     const size_t* lens, size_t r, uint64_t** offs, uint32_t** pids,
                     size_t* count) {
  try {
    auto ps = mag::PatternSet::validate(unpack(pat_bytes, lens, r));
    auto occ = mag::naive_search(ps, std::string_view(reinterpret_cast<const char*>(text), n));
    return emit(occ, offs, pids, count);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Reference Aho–Corasick (oracles.cpp:23-99). With threads > 1 the SAME
// reference automaton is run over `threads` start-ownership ranges, each
// extended by (maxlen-1) bytes of look-ahead; a range keeps only the
// occurrences that start inside it, so concatenation in range order is the
// canonical sorted list (the chunk contract of SPEC.md:354).
int ref_ac_search(const uint8_t* text, size_t n, const uint8_t* pat_bytes, const size_t* lens,
                  size_t r, int threads, uint64_t** offs, uint32_t** pids, size_t* count) {
  try {
    auto ps = mag::PatternSet::validate(unpack(pat_bytes, lens, r));
    mag::AhoCorasick ac(ps);
    const char* t = reinterpret_cast<const char*>(text);
    if (threads <= 1 || n < (1u << 16)) {
      return emit(ac.search(std::string_view(t, n)), offs, pids, count);
    }
    const size_t T = static_cast<size_t>(threads);
    const size_t look = ps.max_length() - 1;
    std::vector<std::vector<mag::Occurrence>> parts(T);
    std::vector<std::thread> pool;
    for (size_t c = 0; c < T; ++c) {
      pool.emplace_back([&, c] {
        const size_t lo = n * c / T, hi = n * (c + 1) / T;
        const size_t end = std::min(n, hi + look);
        auto occ = ac.search(std::string_view(t + lo, end - lo));
        auto& out = parts[c];
        for (auto& o : occ) {
          if (o.offset + lo < hi) out.push_back({o.pattern_index, o.offset + lo});
        }
      });
    }
    for (auto& th : pool) th.join();
    std::vector<mag::Occurrence> all;
    size_t total = 0;
    for (auto& p : parts) total += p.size();
    all.reserve(total);
    for (auto& p : parts) all.insert(all.end(), p.begin(), p.end());
    return emit(all, offs, pids, count);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Builds the reference's byte map. strategy: 0 identity, 1 frequency,
// 2 balanced, 3 lowbits (alphabet_map.cpp:70-114). The histogram is the
// pattern histogram plus the first 1 MiB of `sample` (engine.hpp:31-32).
// Returns 0, or -1 on config_error.
int ref_alphabet_map(int strategy, const uint8_t* pat_bytes, const size_t* lens, size_t r,
                     const uint8_t* sample, size_t sample_len, uint32_t sigma_prime,
                     unsigned lowbits, uint8_t table_out[256], uint32_t* sigma_out) {
  try {
    auto ps = mag::PatternSet::validate(unpack(pat_bytes, lens, r));
    auto h = mag::Histogram::of_patterns(ps);
    if (sample && sample_len)
      h.add(std::string_view(reinterpret_cast<const char*>(sample),
                             std::min<size_t>(sample_len, 1u << 20)));
    auto map = make_map(strategy, h, sigma_prime, lowbits);
    std::memcpy(table_out, map.table().data(), 256);
    *sigma_out = map.sigma_prime();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Map from an explicit histogram (for SPEC's histogram-only examples).
int ref_alphabet_map_hist(int strategy, const uint64_t counts[256], uint32_t sigma_prime,
                          unsigned lowbits, uint8_t table_out[256], uint32_t* sigma_out) {
  try {
    mag::Histogram h;
    for (int i = 0; i < 256; ++i) {
      h.counts[i] = counts[i];
      h.total += counts[i];
    }
    auto map = make_map(strategy, h, sigma_prime, lowbits);
    std::memcpy(table_out, map.table().data(), 256);
    *sigma_out = map.sigma_prime();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// GramConfig validation + encode_text (qgram.cpp:7-37) with the map rebuilt
// from (strategy, patterns). out must hold n/q codes.
int ref_encode_text_strategy(int strategy, const uint8_t* pat_bytes, const size_t* lens,
                             size_t r, uint32_t sigma_prime, unsigned lowbits, unsigned q,
                             const uint8_t* text, size_t n, uint32_t* out) {
  try {
    auto ps = mag::PatternSet::validate(unpack(pat_bytes, lens, r));
    auto h = mag::Histogram::of_patterns(ps);
    mag::GramConfig cfg(q, make_map(strategy, h, sigma_prime, lowbits));
    auto enc = mag::encode_text(cfg, std::string_view(reinterpret_cast<const char*>(text), n));
    std::copy(enc.supers.begin(), enc.supers.end(), out);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// SuperPattern class sets (superimpose.cpp:7-35). mode 0 strided, 1
// overlapping. Writes the class length L to *length; per position the sorted
// distinct codes go to a malloc'd flat array with CSR offsets (L+1 entries).
int ref_classes(int strategy, const uint8_t* pat_bytes, const size_t* lens, size_t r,
                uint32_t sigma_prime, unsigned lowbits, unsigned q, int mode, size_t* length,
                uint64_t** csr, uint32_t** codes) {
  try {
    auto ps = mag::PatternSet::validate(unpack(pat_bytes, lens, r));
    auto h = mag::Histogram::of_patterns(ps);
    mag::GramConfig cfg(q, make_map(strategy, h, sigma_prime, lowbits));
    mag::SuperPattern sp(ps, cfg,
                         mode ? mag::SuperPattern::Mode::overlapping
                              : mag::SuperPattern::Mode::strided);
    auto cls = sp.materialize_classes();
    *length = cls.size();
    *csr = static_cast<uint64_t*>(std::malloc((cls.size() + 1) * 8));
    size_t total = 0;
    for (auto& c : cls) total += c.size();
    *codes = static_cast<uint32_t*>(std::malloc(std::max<size_t>(1, total) * 4));
    size_t o = 0;
    for (size_t i = 0; i < cls.size(); ++i) {
      (*csr)[i] = o;
      for (auto v : cls[i]) (*codes)[o++] = v;
    }
    (*csr)[cls.size()] = o;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// class_match_count (superimpose.cpp:41-52).
int ref_class_match_count(int strategy, const uint8_t* pat_bytes, const size_t* lens, size_t r,
                          uint32_t sigma_prime, unsigned lowbits, unsigned q, uint64_t* value,
                          int* saturated) {
  try {
    auto ps = mag::PatternSet::validate(unpack(pat_bytes, lens, r));
    auto h = mag::Histogram::of_patterns(ps);
    mag::GramConfig cfg(q, make_map(strategy, h, sigma_prime, lowbits));
    auto sp = mag::build_superpattern(ps, cfg);
    auto c = mag::class_match_count(sp);
    *value = c.value;
    *saturated = c.saturated ? 1 : 0;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// PatternSet::validate (core.cpp:7-23): 0 ok, 1 validation_error (index in
// *bad_index), writes m/max length.
int ref_validate(const uint8_t* pat_bytes, const size_t* lens, size_t r, size_t* min_len,
                 size_t* max_len, long* bad_index) {
  try {
    auto ps = mag::PatternSet::validate(unpack(pat_bytes, lens, r));
    *min_len = ps.min_length();
    *max_len = ps.max_length();
    *bad_index = -2;
    return 0;
  } catch (const mag::validation_error& e) {
    g_err = e.what();
    *bad_index = e.index();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
