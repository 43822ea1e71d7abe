// Host model of the search (see host_model.h).  Reference citations are
// /root/reference paths.
#include "host_model.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>

namespace magb {

// ------------------------------------------------------------------ maps
// alphabet_map.cpp:42-50: bytes by descending count, ties by ascending byte.
static void rank_bytes(const Histogram& h, int order[256]) {
  for (int i = 0; i < 256; ++i) order[i] = i;
  std::stable_sort(order, order + 256, [&](int a, int b) { return h.counts[a] > h.counts[b]; });
}

bool build_map(int strategy, const Histogram& h, uint32_t sigma_prime, unsigned lowbits,
               uint8_t table[256], uint32_t* sigma_out, std::string* err) {
  int order[256];
  auto bad_sigma = [&]() {
    if (sigma_prime < 2 || sigma_prime > 256) {
      *err = "sigma' must be in [2, 256], got " + std::to_string(sigma_prime);
      return true;
    }
    return false;
  };
  switch (strategy) {
    case kMapIdentity:
      for (int c = 0; c < 256; ++c) table[c] = static_cast<uint8_t>(c);
      *sigma_out = 256;
      return true;
    case kMapFrequency:  // alphabet_map.cpp:78-88
      if (bad_sigma()) return false;
      rank_bytes(h, order);
      for (uint32_t rank = 0; rank < 256; ++rank)
        table[order[rank]] = static_cast<uint8_t>(rank < sigma_prime - 1 ? rank : sigma_prime - 1);
      *sigma_out = sigma_prime;
      return true;
    case kMapBalanced: {  // alphabet_map.cpp:90-102 (greedy LPT, ties to lowest bin)
      if (bad_sigma()) return false;
      rank_bytes(h, order);
      std::vector<uint64_t> load(sigma_prime, 0);
      for (int i = 0; i < 256; ++i) {
        uint32_t best = static_cast<uint32_t>(std::min_element(load.begin(), load.end()) - load.begin());
        table[order[i]] = static_cast<uint8_t>(best);
        load[best] += h.counts[order[i]];
      }
      *sigma_out = sigma_prime;
      return true;
    }
    case kMapLowbits:  // alphabet_map.cpp:104-114
      if (lowbits < 1 || lowbits > 8) {
        *err = "lowbits bit count must be in [1, 8], got " + std::to_string(lowbits);
        return false;
      }
      for (unsigned c = 0; c < 256; ++c) table[c] = static_cast<uint8_t>(c & ((1u << lowbits) - 1));
      *sigma_out = 1u << lowbits;
      return true;
  }
  *err = "unknown mapping strategy " + std::to_string(strategy);
  return false;
}

// ----------------------------------------------------------------- tuner
// Restated from tuner.hpp:30-66 and SPEC.md:427-492; kept bit-identical to
// oracle/mag_oracle.c mo_tune().
double expected_class_size(double sigma_eff, double n_super) {
  if (sigma_eff <= 0) return 0;
  return sigma_eff * (1.0 - std::pow(1.0 - 1.0 / sigma_eff, n_super));
}

double match_probability(double sigma_eff, double n_super) {
  if (sigma_eff <= 0) return 1;
  return 1.0 - std::pow(1.0 - 1.0 / sigma_eff, n_super);
}

uint32_t resolve_sigma_prime(uint32_t sigma_observed, uint32_t user_choice) {
  if (user_choice) return user_choice;
  if (sigma_observed <= 64) return sigma_observed < 2 ? 2 : sigma_observed;
  return 256;
}

static double log_base(double x, double b) { return std::log(x) / std::log(b); }

static bool q_feasible(uint32_t sp, uint64_t m, unsigned q) {
  if (q < 1 || q > 8) return false;
  if (m < 2ull * q - 1) return false;
  return std::pow(static_cast<double>(sp), static_cast<double>(q)) <= static_cast<double>(1u << 24);
}

unsigned choose_q(const TuningInput& ti) {
  const double rm = static_cast<double>(ti.r) * static_cast<double>(ti.m);
  const double lq = rm > 1 ? log_base(rm, ti.sigma_prime) : 0;
  long q = std::lround(lq);
  q = std::clamp<long>(q, 1, 8);
  while (q > 1 && !q_feasible(ti.sigma_prime, ti.m, static_cast<unsigned>(q))) --q;
  return static_cast<unsigned>(q);
}

double strided_k_seed(const TuningInput& ti, unsigned /*q*/) {
  const double rm = static_cast<double>(ti.r) * static_cast<double>(ti.m);
  const double L = log_base(rm, ti.sigma_prime);
  if (L <= 0) return 1;
  const double rho = L / static_cast<double>(ti.m);
  const double l = log_base(1.0 / rho, ti.sigma_prime);
  if (L + l <= 0) return 1;
  return static_cast<double>(ti.m) / L * l / (L + l);
}

static unsigned alignment_len(const TuningInput& ti, unsigned q, unsigned k) {
  const uint64_t Lq = (ti.m - q + 1) / q;
  const unsigned w = ti.word_bits ? ti.word_bits : 64;
  return static_cast<unsigned>(std::min<uint64_t>(Lq / k, w / k));
}

double predicted_cost(const TuningInput& ti, unsigned q, unsigned k) {
  const double nq = static_cast<double>(ti.n / q);
  const double p = match_probability(std::pow(static_cast<double>(ti.sigma_prime), q),
                                     static_cast<double>(q) * static_cast<double>(ti.r));
  const unsigned mp = alignment_len(ti, q, k);
  return nq / k + nq * std::pow(p, mp) * (2.0 * q - 1) * static_cast<double>(ti.r) *
                      static_cast<double>(ti.m);
}

unsigned choose_k(const TuningInput& ti, unsigned q) {
  const uint64_t Lq = std::max<uint64_t>(1, (ti.m - q + 1) / q);
  const unsigned w = ti.word_bits ? ti.word_bits : 64;
  long k0 = std::lround(strided_k_seed(ti, q));
  k0 = std::clamp<long>(k0, 1, static_cast<long>(Lq));
  const long lo = std::max<long>(1, k0 - 2), hi = std::min<long>(static_cast<long>(Lq), k0 + 2);
  unsigned best = static_cast<unsigned>(k0);
  double bc = std::numeric_limits<double>::infinity();
  for (long k = lo; k <= hi; ++k) {
    if (static_cast<unsigned>(k) > w) continue;
    const double c = predicted_cost(ti, q, static_cast<unsigned>(k));
    if (c < bc) {
      bc = c;
      best = static_cast<unsigned>(k);
    }
  }
  return best;
}

bool tune(const TuningInput& in, int fixed_q, int fixed_k, TuningResult* out, std::string* err) {
  TuningInput ti = in;
  if (ti.r < 1 || ti.m < 1 || ti.sigma < 1) {
    *err = "tuning input needs r, m, sigma >= 1";
    return false;
  }
  if (!ti.word_bits) ti.word_bits = 64;
  ti.sigma_prime = resolve_sigma_prime(ti.sigma, ti.sigma_prime);
  if (ti.sigma_prime < 2 || ti.sigma_prime > 256) {
    *err = "sigma' must be in [2, 256]";
    return false;
  }
  const unsigned q0 = fixed_q > 0 ? static_cast<unsigned>(fixed_q) : choose_q(ti);
  if (!q_feasible(ti.sigma_prime, ti.m, q0)) {
    *err = "q = " + std::to_string(q0) + " is infeasible (q <= 8, sigma'^q <= 2^24, m >= 2q-1)";
    return false;
  }
  unsigned qlo = q0, qhi = q0;
  if (fixed_q <= 0) {  // tuner.hpp:63-64 joint local grid around the seeds
    qlo = q0 > 2 ? q0 - 2 : 1;
    qhi = q0 + 2;
  }
  unsigned bq = q0, bk = 1;
  double bc = std::numeric_limits<double>::infinity();
  for (unsigned q = qlo; q <= qhi; ++q) {
    if (!q_feasible(ti.sigma_prime, ti.m, q)) continue;
    unsigned k;
    if (fixed_k > 0) {
      const uint64_t Lq = (ti.m - q + 1) / q;
      if (static_cast<uint64_t>(fixed_k) > Lq || static_cast<unsigned>(fixed_k) > ti.word_bits)
        continue;
      k = static_cast<unsigned>(fixed_k);
    } else {
      k = choose_k(ti, q);
    }
    const double c = predicted_cost(ti, q, k);
    if (c < bc) {
      bc = c;
      bq = q;
      bk = k;
    }
  }
  if (!std::isfinite(bc)) {
    *err = "no feasible (q, k)";
    return false;
  }
  const double rm = static_cast<double>(ti.r) * static_cast<double>(ti.m);
  out->q = bq;
  out->k = bk;
  out->sigma_prime = ti.sigma_prime;
  out->rho = (rm > 1 ? log_base(rm, ti.sigma_prime) : 0) / static_cast<double>(ti.m);
  out->predicted_p = match_probability(std::pow(static_cast<double>(ti.sigma_prime), bq),
                                       static_cast<double>(bq) * static_cast<double>(ti.r));
  out->predicted_cost = bc;
  return true;
}

// ------------------------------------------------------------------ plan
namespace {

constexpr uint32_t kChunkTarget = 1536;   // gram bytes per ring slot
constexpr uint32_t kSliceTarget = 32768;  // text bytes per warp work item
constexpr uint32_t kDefaultRing = 2;
constexpr uint32_t kDefaultWarps = kMaxWarps - 1;  // staged plans: 15 warps (calibrated in round 1)

unsigned pow2ceil_log2(unsigned x) {
  unsigned l = 0;
  while ((1u << l) < x) ++l;
  return l;
}

// Probability that a text gram hits an admitted entry at one class position:
// exact membership (uniform text over the pattern alphabet) plus hash
// collisions into 2^table_bits entries.
double est_position_p(double admissions, double universe, double entries) {
  double distinct, exact;
  if (universe > 1e15) {
    distinct = admissions;
    exact = 0;
  } else {
    distinct = universe * (1.0 - std::exp(-admissions / universe));
    exact = distinct / universe;
  }
  if (entries <= 1) return 1.0;
  const double coll = 1.0 - std::exp(-distinct / entries);
  return exact + (1.0 - exact) * coll;
}

double prefilter_fp(double keys, unsigned pf_bits) {
  const double f = 1.0 - std::exp(-2.0 * keys / std::ldexp(1.0, static_cast<int>(pf_bits)));
  return f * f;
}

// Cost model in thread-instructions per text byte (calibrated on B200, see
// DESIGN.md): per sample gram+lookup, per extra m' a shuffle, per candidate
// a queue slot, per verified start a rolled key + prefilter, per prefilter
// pass an L2 bucket probe.
constexpr double kCostSample = 30, kCostShift = 3, kCostCand = 30, kCostStart = 45,
                 kCostWindow = 60, kCostScreen = 25, kCostProbe = 80, kCostVerifyAll = 45, kCostCompare = 40,
                 kCostChunk = 4800,  // per staged chunk (loader + bookkeeping), thread-instr
                 kCostProbeBit = 3,  // per extra probe bit of a multi-probe gram
                 kCostPf = 15,       // shared-memory prefilter test
                 kCostDirectHit = 120,  // direct kernel: a filter hit issues one L2 screen load
                 kCostRollPos = 24,   // roll kernel: roll + one Bloom word per position
                 kCostRollProbe = 1.5,  // each Bloom probe
                 kCostRollBatch = 6,  // a verification batch (expansion, keys, slot loads) per 64 bytes of lane work
                 kCostRollWarm = 2,   // prefix warm-up (q bytes per 32-position run)
                 kCostRollCand = 800;  // expansion + start key + verification-slot round trip of a hit
// Round-1 B200 calibration: the staged kernel's measured cost per
// text byte is ~4x the instruction model above plus a fixed ~15 (ring
// bookkeeping, queue drains, verification latency); the direct kernel's
// per-sample filter work scales the same way, and one direct-kernel filter
// hit (L2 screen load + deferred resolve) costs ~120.
constexpr double kStagedScale = 4, kStagedFloor = 15;
constexpr double kCostWalkEntry = 1500;  // a verification entry walked beyond the survivor's first
double staged_scale(double model) { return kStagedScale * model + kStagedFloor; }

// Expected pattern-table entries sharing a probed key (exact byte compares)
// when `keys` keys of v bytes are drawn over the pattern alphabet.
double key_hits(double keys, double sigma, unsigned v) {
  const double universe = std::pow(sigma, static_cast<double>(v));
  return universe > 1e15 ? 0.0 : keys / universe;
}

uint32_t gcd32(uint32_t a, uint32_t b) {
  while (b) {
    const uint32_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

// Chunk / slice / slot sizes of the warp-streaming kernel.
void finish_geometry(const PatternData& pd, const PlanRequest& rq, Plan* P) {
  const ScanPlan& sp = P->sp;
  const uint32_t ov = sp.m_prime ? sp.m_prime - 1 : 0;
  const uint32_t bps = sp.verify_all || sp.overlapping ? 1 : sp.q * sp.k;  // bytes per sample
  const uint32_t target = rq.tile_bytes > 0 ? static_cast<uint32_t>(rq.tile_bytes)
                                            : (P->chunk_target ? P->chunk_target : kChunkTarget);
  // interior chunks advance by a multiple of 16 bytes (aligned TMA windows)
  const uint32_t m16 = 16 / gcd32(16, bps);
  uint32_t c = std::max<uint32_t>(32, target / bps / m16 * m16);
  c = (c + m16 - 1) / m16 * m16;
  // k = 1 strided chunks record hits in a <= 1024-bit bitmap; m' = 1 chunks
  // tile into whole 64-sample steps
  if (!sp.overlapping && !sp.verify_all && sp.k == 1) {
    c = std::min<uint32_t>(c, 1024);
    if (sp.m_prime == 1 && c >= 64 && 64 % m16 == 0) c = c / 64 * 64;
  }
  P->chunk_samples = c;
  const uint64_t chunk_bytes = static_cast<uint64_t>(c) * bps;
  P->slice_samples = static_cast<uint64_t>(c) *
                     std::max<uint64_t>(1, (kSliceTarget + chunk_bytes / 2) / chunk_bytes);
  // pattern reach after the last gram: full patterns up to 1 KiB stay in the
  // slot, longer ones are compared from global memory; >= 16 + 4 key bytes
  P->back = static_cast<uint32_t>(std::min<uint64_t>(pd.maxlen, 1024) + 24);
  const uint64_t qm1 = sp.overlapping || sp.verify_all ? 0 : sp.q - 1;
  const uint64_t extra = sp.overlapping ? sp.q : 0;
  P->full_bytes = static_cast<uint32_t>(
      align16(chunk_bytes + static_cast<uint64_t>(ov) * bps + qm1 + extra + P->back + 15));
  P->slot_bytes = P->full_bytes + 32;
  P->ring = rq.stages > 0 ? static_cast<uint32_t>(rq.stages) : kDefaultRing;
  P->nwarps = rq.warps > 0 ? std::min<uint32_t>(rq.warps, kMaxWarps) : kDefaultWarps;
}

size_t fixed_smem(const Plan& P) {
  ScanPlan z = P.sp;
  z.table_in_smem = 0;
  z.pf_bits = 0;
  return smem_layout(z, P.slot_bytes, P.ring, P.nwarps).total;
}

void set_entry_geometry(ScanPlan& sp) {
  const unsigned bits = sp.k * sp.m_prime;
  sp.entry_log2 = pow2ceil_log2(std::max(1u, bits));
  uint64_t match = 0;
  for (unsigned j = 0; j < sp.k; ++j) match |= 1ull << (j * sp.m_prime + sp.m_prime - 1);
  sp.match_mask = match;
  if (sp.probes > 1 && !sp.roll) sp.entries = static_cast<uint64_t>(sp.blocks) * 64;
  const uint64_t tbits = sp.entries << sp.entry_log2;
  sp.table_bytes = align16(std::max<uint64_t>(16, (tbits + 7) / 8));
}

}  // namespace

int make_plan(const PatternData& pd, const Histogram& h, const PlanRequest& rq, Plan* P,
              std::string* err) {
  constexpr int kOk = 0, kBadConfig = 5;
  *P = Plan{};
  ScanPlan& sp = P->sp;
  P->variant = rq.variant;
  if (rq.variant == 3 || rq.variant == 4) {
    *err = "variants naive/ac are CPU oracles; this GPU library runs mag, smag and shiftor_og";
    return kBadConfig;
  }
  if (rq.variant < 0 || rq.variant > 4) {
    *err = "unknown variant " + std::to_string(rq.variant);
    return kBadConfig;
  }
  if (pd.r > kMaxPatterns) {
    *err = "at most 2^24 patterns are supported";
    return kBadConfig;
  }
  sp.overlapping = rq.variant == 2;
  sp.probes = 1;
  sp.smag = rq.variant == 1;
  sp.m = static_cast<uint32_t>(std::min<size_t>(pd.m, 0xffffffffu));
  sp.maxlen = static_cast<uint32_t>(std::min<size_t>(pd.maxlen, 0xffffffffu));
  sp.r = static_cast<uint32_t>(pd.r);
  sp.key_len = static_cast<uint32_t>(std::min<size_t>(pd.m, 16));
  const uint32_t sigma_obs = std::max(1u, h.distinct());
  const size_t m = pd.m;
  const unsigned w = rq.word_bits > 0 ? std::min(64, rq.word_bits) : 64;

  uint32_t best_halo = 0;   // roll plans: staged bytes past a step
  uint32_t best_roll_warps = 0, best_roll_step = kRollStep;
  uint32_t best_warps = 0;  // direct plans: warps per CTA the planner chose
  const bool reference_mode = rq.gram_mode == 0 ||
                              (rq.gram_mode < 0 && (rq.q || rq.k || rq.sigma_prime ||
                                                     rq.mapping != -1));
  if (reference_mode) {
    // ---- the reference engine's own parameter path (engine.hpp:22-33)
    sp.gram_mode = kGramExact;
    int mapping = rq.mapping;
    uint32_t sigma_req = static_cast<uint32_t>(std::max(0, rq.sigma_prime));
    uint32_t sprime = resolve_sigma_prime(sigma_obs, sigma_req);
    if (mapping == -1) mapping = sprime < 256 ? kMapBalanced : kMapIdentity;  // mag.h:47
    uint32_t sp_out = 0;
    if (!build_map(mapping, h, sprime, static_cast<unsigned>(std::max(0, rq.lowbits)), P->map,
                   &sp_out, err))
      return kBadConfig;
    P->mapping = mapping;
    sp.sigma_prime = sp_out;
    TuningInput ti;
    ti.sigma = sigma_obs;
    ti.sigma_prime = sp_out;
    ti.r = pd.r;
    ti.m = m;
    ti.word_bits = w;
    unsigned q = rq.q > 0 ? static_cast<unsigned>(rq.q) : 0;
    unsigned k = rq.k > 0 ? static_cast<unsigned>(rq.k) : 0;
    if (!q || (!k && !sp.overlapping)) {
      TuningResult tr;
      std::string terr;
      if (tune(ti, rq.q, sp.overlapping ? 1 : rq.k, &tr, &terr)) {
        if (!q) q = tr.q;
        if (!k) k = tr.k;
      } else if (!q) {
        q = 1;
      }
    }
    if (sp.overlapping) k = 1;
    if (!k) k = 1;
    // GramConfig (qgram.cpp:9-19)
    if (q < 1 || q > 8) {
      *err = "q must be in [1, 8], got " + std::to_string(q);
      return kBadConfig;
    }
    uint64_t space = 1;
    for (unsigned i = 0; i < q; ++i) {
      space *= sp_out;
      if (space > (1u << 24)) {
        *err = "sigma'^q exceeds the table budget (" + std::to_string(sp_out) + "^" +
               std::to_string(q) + " > 2^24); lower q or reduce the alphabet";
        return kBadConfig;
      }
    }
    sp.entries = space;
    sp.q = q;
    sp.k = k;
  } else {
    // ---- GPU planner: hashed q-gram alphabet sized to shared memory
    sp.gram_mode = kGramHashed;
    P->mapping = kMapIdentity;
    for (int c = 0; c < 256; ++c) P->map[c] = static_cast<uint8_t>(c);
    sp.sigma_prime = 256;
    // shared memory left for table + prefilter once the warp rings (of a
    // given chunk size) are in
    auto room_for = [&](unsigned q, unsigned k, unsigned mp, int va, uint32_t chunk, int og = -1) {
      Plan probe = *P;
      if (og >= 0) probe.sp.overlapping = og;
      probe.sp.q = q;
      probe.sp.k = k;
      probe.sp.m_prime = mp;
      probe.sp.verify_all = va;
      probe.chunk_target = chunk;
      finish_geometry(pd, rq, &probe);
      const size_t f = fixed_smem(probe) + 1024;
      return rq.smem_limit > f ? rq.smem_limit - f : size_t(0);
    };
    static const uint32_t kChunks[] = {4096, 3072, 2048, 1536, 1024, 768, 512};
    static const unsigned kPf[] = {0, 16, 17, 18, 19, 20, 21};
    const double keys = static_cast<double>(pd.r);
    struct Cand {
      double cost = std::numeric_limits<double>::infinity();
      unsigned q = 1, k = 1, mp = 1, tb = 0, pf = 0, H = 1;
      uint32_t chunk = kChunkTarget;
      int direct = 0;
      int roll = 0;
      int pack2 = 0;
      uint32_t pack_shift = 0;
      uint32_t roll_words = 0, halo = 0, ddepth = 0, warps = 0;
      uint32_t blocks = 0;
      bool va = true;
      int og = 0;
      double cpb = 1;
      double slope = 0;  // d cost / d (candidates per byte): what a measured rate re-prices
      double surv_slope = 0;  // direct: d cost / d (screen survivors per byte)
    } best;
    best.og = sp.overlapping;
    auto pf_bytes = [](unsigned pf) { return pf ? align16((size_t(1) << pf) / 8) : size_t(16); };
    const bool allow_staged = rq.kernel == 0 || rq.kernel == 1;
    // verify-all baseline
    for (unsigned pf : kPf) {
      if (!allow_staged) break;
      for (uint32_t chunk : kChunks) {
        if (rq.tile_bytes > 0 && chunk != kChunks[0]) break;
        if (pf_bytes(pf) > room_for(1, 1, 1, 1, chunk)) continue;
        const double cost = staged_scale(kCostVerifyAll + kCostChunk / chunk +
                            (pf ? prefilter_fp(keys, pf) : 1.0) * kCostProbe +
                            key_hits(keys, sigma_obs, static_cast<unsigned>(std::min<size_t>(m, 16))) *
                                kCostCompare);
        if (cost < best.cost) {
          best.cost = cost;
          best.pf = pf;
          best.chunk = chunk;
          best.cpb = 1;
          best.slope = 0;
        }
        break;  // largest chunk that fits
      }
    }
    // machines: the requested variant's, and for mag (whose result set is
    // parameter-invariant) also the overlapping one (q-gram per byte, window 1)
    const int og_lo = rq.variant == 2 ? 1 : 0, og_hi = rq.variant == 1 ? 0 : 1;
    for (int og = og_lo; og <= og_hi && rq.table_bits >= 0 && allow_staged; ++og) {
      const unsigned qmax = og ? static_cast<unsigned>(std::min<size_t>(16, m))
                                           : static_cast<unsigned>(std::min<size_t>(16, (m + 1) / 2));
      for (unsigned q = 1; q <= qmax; ++q) {
        if (rq.q > 0 && q != static_cast<unsigned>(rq.q)) continue;
        const size_t L = og ? m - q + 1 : (m - q + 1) / q;
        if (L < 1) continue;
        const double universe = std::pow(static_cast<double>(sigma_obs), static_cast<double>(q));
        const unsigned kmax = og ? 1 : static_cast<unsigned>(std::min<size_t>(L, w));
        for (unsigned k = 1; k <= kmax; ++k) {
          if (rq.k > 0 && !og && k != static_cast<unsigned>(rq.k)) continue;
          const unsigned mpmax = static_cast<unsigned>(std::min<size_t>(L / k, w / k));
          for (unsigned mp = 1; mp <= mpmax; ++mp) {
            const unsigned el = pow2ceil_log2(std::max(1u, k * mp));
            const double sample_cost = (kCostSample + (mp - 1) * kCostShift) /
                                       (og ? 1.0 : static_cast<double>(k * q));
            const bool wkey = !og && q > 1;
            const double nkeys = wkey ? keys * q : keys;
            const double hits = key_hits(nkeys, sigma_obs,
                                         static_cast<unsigned>(wkey ? std::min<size_t>(16, m - q + 1)
                                                                    : std::min<size_t>(16, m)));
            for (unsigned tbits = 12; tbits <= 24; ++tbits) {
             if (rq.table_bits > 0 && tbits != static_cast<unsigned>(rq.table_bits)) continue;
             const unsigned hmax = (mp == 1 && k == 1 && tbits >= 8) ? 4 : 1;
             for (unsigned H = 1; H <= hmax; ++H) {
              if (rq.probes > 0 && H != static_cast<unsigned>(rq.probes)) continue;
              const size_t tbytes = align16((size_t(1) << (tbits + el)) / 8);
              const double adm = og ? keys : keys * q;
              double p = est_position_p(adm, universe, std::ldexp(1.0, static_cast<int>(tbits)));
              if (H > 1) {  // probes inside a 32-entry block (est. as a plain Bloom filter)
                const double distinct = universe > 1e15 ? adm : universe * (1.0 - std::exp(-adm / universe));
                const double exact = universe > 1e15 ? 0.0 : distinct / universe;
                const double fill = 1.0 - std::exp(-static_cast<double>(H) * distinct / std::ldexp(1.0, static_cast<int>(tbits)));
                p = exact + (1.0 - exact) * std::pow(fill, static_cast<double>(H));
              }
              const double pm = std::pow(p, static_cast<double>(mp));
              // candidates per byte, and verified starts per byte
              const double cpb = og ? pm : pm / q;
              for (unsigned pf : kPf) {
                uint32_t chunk = 0;
                for (uint32_t c : kChunks) {
                  if (rq.tile_bytes > 0 && c != kChunks[0]) break;
                  if (tbytes + pf_bytes(pf) <= room_for(q, k, mp, 0, c, og)) {
                    chunk = c;
                    break;
                  }
                }
                if (!chunk) continue;
                const double fp = pf ? prefilter_fp(nkeys, pf) : 1.0;
                double cost = sample_cost + (H - 1) * kCostProbeBit / (og ? 1.0 : static_cast<double>(k * q)) + kCostChunk / chunk;
                // per candidate: window keys pay one batched key + L2 screen,
                // start keys one probe per verified start (q starts per strided candidate)
                const double per_cand =
                    wkey ? kCostCand + kCostWindow + (pf ? kCostPf : 0.0) +
                               fp * (kCostScreen + 0.01 * kCostProbe) + hits * kCostCompare
                         : kCostCand + (og ? 1.0 : static_cast<double>(q)) *
                                           (kCostStart + fp * kCostProbe + hits * kCostCompare);
                cost += cpb * per_cand;
                cost = staged_scale(cost);
                if (cost < best.cost * 0.999) {
                  best.cost = cost;
                  best.q = q;
                  best.k = k;
                  best.mp = mp;
                  best.tb = tbits;
                  best.H = H;
                  best.pf = pf;
                  best.chunk = chunk;
                  best.va = false;
                  best.og = og;
                  best.cpb = cpb;
                  best.slope = kStagedScale * per_cand;
                }
              }
             }
            }
          }
        }
      }
    }
    // direct stream kernel (q = 16 or 8 byte aligned samples): no gram
    // staging, the table takes the smem; an occurrence (m >= 2q - 1) always
    // covers one whole aligned sample, at one of q shifts
    for (unsigned q : {16u, 8u}) {
      // rq.stages selects the ring depth (2..4; single-probe q = 16 tables only)
      const bool depth_ok = rq.stages == 0 || (q == 16 && rq.stages >= 2 && rq.stages <= 4 && rq.probes <= 1);
      if (!((rq.kernel == 0 || rq.kernel == 2) && rq.table_bits >= 0 && !sp.overlapping && m >= 2 * q - 1 &&
            (rq.q == 0 || rq.q == static_cast<int>(q)) && rq.k <= 1 && depth_ok && rq.tile_bytes == 0))
        continue;
      // Round 1 measured W = 16 at 13/14/15/16 warps: cfg4 2,551/2,604/2,686/1,934
      // GB/s (a 16th scanning warp leaves L1 ~17 KB for the screen and bucket
      // loads), cfg2 15 vs 16 = 4,802 vs 4,689 GB/s.
      // Round 2, W = 8: 16 warps 3,428 vs 15 warps 3,317 GB/s on cfg3.
      const uint32_t warps = rq.warps > 0 ? std::min<uint32_t>(rq.warps, kMaxWarps)
                                          : (q == 8 ? kMaxWarps : kMaxWarps - 1);
      // ring depth: multi-probe tables run 4-deep rings; single-probe q = 16
      // tables default to 2-deep rings, whose freed 32 KB doubles the table
      // (2^20 bits: measured +4% cfg2, +16% cfg4 over 4-deep / 2^19)
      auto room_at = [&](uint32_t depth) {
        ScanPlan z{};
        z.q = q;
        z.ddepth = depth;
        const size_t fixed = direct_smem(z, warps);  // the kernel has no static shared memory
        return rq.smem_limit > fixed ? rq.smem_limit - fixed : size_t(0);
      };
      const uint32_t depth1 = rq.stages ? static_cast<uint32_t>(rq.stages) : (q == 16 && warps <= 16 ? 2u : 0u);
      const size_t room = room_at(rq.stages ? static_cast<uint32_t>(rq.stages) : 0u);
      const size_t room1 = room_at(depth1);
      // tables of at most ~64 bits per admitted gram (every CTA loads its copy)
      const double adm = keys * q;
      const size_t cap_bits = std::max<size_t>(size_t(1) << 14, static_cast<size_t>(adm * 64));
      const uint32_t blocks = static_cast<uint32_t>(std::min<size_t>({room / 8, size_t(1) << 22, cap_bits / 64}));
      const double universe = std::pow(static_cast<double>(sigma_obs), static_cast<double>(q));
      const double distinct = universe > 1e15 ? adm : universe * (1.0 - std::exp(-adm / universe));
      const double exact = universe > 1e15 ? 0.0 : distinct / universe;
      const double hits = key_hits(adm, sigma_obs, q);
      // single probe: largest power-of-two table that fits
      unsigned tb1 = 6;
      while (tb1 < 26 && (size_t(1) << (tb1 + 1)) / 8 <= room1 && (size_t(1) << tb1) < cap_bits) ++tb1;
      for (unsigned H = 1; H <= (q == 8 ? 4u : kMaxProbes); ++H) {
        if (rq.probes > 0 && H != static_cast<unsigned>(rq.probes)) continue;
        if (H > 1 && blocks == 0) break;  // multi-probe tables run 4-deep rings: no room left
        if (H == 1 && room1 < 2048) continue;
        if (rq.stages != 0 && H > 1) continue;
        const double bits = H == 1 ? std::ldexp(1.0, static_cast<int>(tb1)) : 64.0 * blocks;
        const double fill = 1.0 - std::exp(-static_cast<double>(H) * distinct / bits);
        const double p = exact + (1.0 - exact) * std::pow(fill, static_cast<double>(H));
        const double cpb = p / q;
        // a filter hit only issues its L2 screen load (resolved a step later);
        // ~1/128 of them, plus the true starts, reach a bucket walk
        const double per_surv = kCostCand + kCostProbe + hits * kCostCompare;
        const double per_cand = kCostDirectHit + 0.008 * per_surv;
        const double cost = kStagedScale * (kCostSample + 2 * H * kCostProbeBit) / q + cpb * per_cand;
        if (cost < best.cost * 0.999) {
          best.cost = cost;
          best.q = q;
          best.k = 1;
          best.mp = 1;
          best.tb = 0;
          best.H = H;
          best.pf = 0;
          best.chunk = kChunkTarget;
          best.va = false;
          best.cpb = cpb;
          best.slope = kCostDirectHit;
          best.surv_slope = per_surv;
          best.direct = 1;
          best.og = 0;
          best.blocks = H > 1 ? blocks : 0;
          best.tb = H > 1 ? 0 : tb1;
          best.ddepth = H > 1 ? static_cast<uint32_t>(rq.stages) : depth1;
          best.warps = warps;
        }
      }
    }
    // dense rolling-hash scan: every position, whole-prefix (q <= m) keys in a
    // shared-memory Bloom filter; for pattern sets that saturate gram filters
    if ((rq.kernel == 0 || rq.kernel == 3) && rq.table_bits >= 0 && rq.variant != 1 && m >= 8 &&
        rq.k <= 1 && rq.stages == 0 && rq.tile_bytes == 0) {
      static const unsigned kRollQ[] = {32, 24, 20, 16, 12, 8};
      unsigned q = 0;
      for (unsigned c : kRollQ)
        if (c <= m && (rq.q == 0 || static_cast<unsigned>(rq.q) == c)) {
          q = c;
          break;
        }
      // equal-length sets of <= 12 bytes run the pipelined kernel: up to 24 warps
      const bool eq_set = pd.maxlen == pd.m && pd.m <= 12;
      // (cfg5, 15 / 16 / 20 warps: 690 / 718 / 655 GB/s; the finish grid waits for a CTA to leave)
      const uint32_t warps = rq.warps > 0 ? std::min<uint32_t>(rq.warps, eq_set ? kRollMaxWarps : kMaxWarps)
                                          : (eq_set ? kMaxWarps : kMaxWarps - 1);
      best_roll_warps = warps;
      const uint32_t v4 = (32 + q - 1 + 15) / 16;
      const uint32_t halo = static_cast<uint32_t>(
          align16(std::max<size_t>(16 * v4, std::min<size_t>(pd.maxlen, 240) + 8)));
      const uint32_t rstep = eq_set ? kRollStepEq : kRollStep;
      best_roll_step = rstep;
      const size_t fixed = roll_smem(0, halo, warps, rstep) + 1024;
      // Bloom words: what shared memory leaves, but no more than ~2 Kibit per
      // pattern (every CTA loads the table: small sets keep it small)
      const size_t room_words = rq.smem_limit > fixed ? (rq.smem_limit - fixed) / 16 * 4 : 0;
      const uint32_t words = static_cast<uint32_t>(
          std::min<size_t>(room_words, std::max<size_t>(4096, (64 * pd.r + 3) / 4 * 4)));
      const double universe = std::pow(static_cast<double>(sigma_obs), static_cast<double>(q));
      const double exact = universe > 1e15 ? 0.0 : std::min(1.0, keys / universe);
      for (unsigned H = 1; q && room_words >= 1024 && H <= 3; ++H) {
        if (rq.probes > 0 && H != static_cast<unsigned>(rq.probes)) continue;
        const double bits = 32.0 * words;
        const double fill = 1.0 - std::exp(-static_cast<double>(H) * keys / bits);
        const double fp = std::min(1.0, 1.4 * std::pow(fill, static_cast<double>(H)));  // blocked penalty
        const double cpb = exact + (1.0 - exact) * fp;
        // a step (2048 positions) with any hit pays one verification batch
        const double batch = 1.0 - std::exp(-cpb * rstep);
        const double cost = kCostRollPos + H * kCostRollProbe + kCostRollWarm * q / 32.0 + cpb * kCostRollCand +
                            batch * kCostRollBatch;
        if (cost < best.cost * 0.999) {
          best = Cand{};
          best.cost = cost;
          best.q = q;
          best.H = H;
          best.va = false;
          best.og = 1;
          best.cpb = cpb;
          best.slope = kCostRollCand;
          best.roll = 1;
          best.roll_words = words;
          best.halo = halo;
          best.chunk = rstep;
        }
      }
    }
    // pack2: the pattern alphabet has <= 4 symbols and some shift s makes
    // b -> (b >> s) & 3 injective on it (DNA: s = 1).  Forced only
    // (scan_kernel = 4): on cfg5 its 10-symbol level 1 passes 10% of the
    // positions and measured 211 GB/s against the rolling-hash scan's 473.
    int pack_shift = -1;
    {
      bool used[256] = {false};
      for (size_t i = 0; i < pd.r; ++i)
        for (uint32_t j = 0; j < pd.len[i]; ++j) used[pd.pattern(i)[j]] = true;
      int distinct = 0;
      for (int c = 0; c < 256; ++c) distinct += used[c];
      for (int s = 0; s <= 6 && distinct <= 4 && pack_shift < 0; ++s) {
        unsigned seen = 0;
        bool ok = true;
        for (int c = 0; c < 256 && ok; ++c)
          if (used[c]) {
            const unsigned v = 1u << ((c >> s) & 3);
            ok = !(seen & v);
            seen |= v;
          }
        if (ok) pack_shift = s;
      }
    }
    const bool pack_ok = pack_shift >= 0 && m >= 10 && rq.table_bits >= 0 && rq.variant != 1 && rq.k <= 1 &&
                         rq.stages == 0 && rq.tile_bytes == 0 && rq.q == 0;
    if (pack_ok && rq.kernel == 4) {
      best = Cand{};
      best.cost = 0;
      best.q = static_cast<unsigned>(std::min<size_t>(m, 16));
      best.va = false;
      best.og = 1;
      best.pack2 = 1;
      best.pack_shift = static_cast<uint32_t>(pack_shift);
      best.halo = 32;
      best.chunk = kPack2Step;
      // level-1 candidates: keys' distinct 10-symbol prefixes over 2^20
      best.cpb = std::min(1.0, 1.0 - std::exp(-static_cast<double>(pd.r) / std::ldexp(1.0, kPack2L1Bits)));
    }
    if (rq.kernel != 0 && !std::isfinite(best.cost)) {
      *err = "the requested scan kernel cannot run this pattern set / option combination";
      return kBadConfig;
    }
    sp.overlapping = best.og;
    if (best.va) {
      sp.q = 1;
      sp.k = 1;
      sp.m_prime = 1;
      sp.table_bits = 0;
      sp.entries = 1;
      sp.verify_all = 1;
    } else {
      sp.q = best.q;
      sp.k = best.k;
      sp.m_prime = best.mp;
      sp.table_bits = best.tb;
      sp.entries = 1ull << best.tb;
      sp.probes = best.H;
      sp.blocks = best.H > 1 ? (best.direct ? best.blocks : static_cast<uint32_t>((1ull << best.tb) / 64)) : 0;
      sp.direct = best.direct;
      sp.ddepth = best.ddepth;
      best_warps = best.warps;
      sp.roll = best.roll;
      sp.pack2 = best.pack2;
      sp.pack_shift = best.pack_shift;
      best_halo = best.halo;
      if (best.roll) {
        sp.roll_words = best.roll_words;
        sp.entries = static_cast<uint64_t>(best.roll_words) * 32;
        sp.table_bits = 0;
        sp.blocks = 0;
      }
      if (best.pack2) {  // level-1 bitmap of the first 10 symbols' codes
        sp.table_bits = kPack2L1Bits;
        sp.entries = 1ull << kPack2L1Bits;
        sp.blocks = 0;
        sp.probes = 1;
      }
    }
    sp.pf_bits = best.pf;
    P->chunk_target = best.chunk;
    P->pred_cand_per_byte = best.cpb;
    P->pred_cost = best.cost;
    P->cost_slope = best.slope;
    P->surv_slope = best.surv_slope;
    P->pred_surv_per_byte = best.direct ? 0.008 * best.cpb : 0.0;
  }

  // ---- machine shape (filter.hpp:27-31, superimpose.cpp:11-21)
  const unsigned q = sp.q;
  size_t L;
  if (sp.overlapping) {
    if (m < q) {
      *err = "m = " + std::to_string(m) + " is shorter than q; lower q";
      return kBadConfig;
    }
    L = m - q + 1;
    sp.k = 1;
  } else {
    if (m < 2 * static_cast<size_t>(q) - 1) {
      *err = "m = " + std::to_string(m) + " is below 2q-1 = " + std::to_string(2 * q - 1) +
             "; lower q so every shift yields at least one gram";
      return kBadConfig;
    }
    L = (m - q + 1) / q;
  }
  if (sp.k < 1 || sp.k > L || sp.k > w) {
    *err = "k = " + std::to_string(sp.k) + " is infeasible for L = " + std::to_string(L) +
           " and w = " + std::to_string(w);
    return kBadConfig;
  }
  if (reference_mode || sp.m_prime == 0)
    sp.m_prime = static_cast<uint32_t>(std::min<size_t>(L / sp.k, w / sp.k));
  set_entry_geometry(sp);
  finish_geometry(pd, rq, P);
  if (sp.direct) {  // direct kernel: slices of whole steps, ~32 KiB of text
    const uint64_t step = direct_step_bytes(sp.q) / sp.q;
    P->slice_samples = step * std::max<uint64_t>(1, 32768 / direct_step_bytes(sp.q));
  }
  if (sp.pack2) {  // pack2 geometry: 2 KiB steps, 16 steps per slice
    P->chunk_samples = kPack2Step;
    P->slice_samples = static_cast<uint64_t>(kPack2Step) * 16;
    P->back = best_halo;
    P->ring = kPack2Depth;
    P->nwarps = rq.warps > 0 ? std::min<uint32_t>(rq.warps, kMaxWarps) : kMaxWarps - 1;
  }
  if (sp.roll) {  // roll kernel geometry: 2 KiB steps, 16 steps per slice
    sp.roll_step = best_roll_step;
    P->chunk_samples = best_roll_step;
    P->slice_samples = 32768;  // whole steps either way
    P->back = best_halo;
    P->ring = kRollDepth;
    // more than 16 warps: only the 3-probe equal-length kernels are built with
    // the wider launch bounds (scan_roll.cu launch_roll_qhe)
    P->nwarps = best_roll_warps ? best_roll_warps : kMaxWarps - 1;
    if (sp.probes != 3) P->nwarps = std::min<uint32_t>(P->nwarps, kMaxWarps);
  }

  // ---- shared-memory placement
  const size_t fixed = fixed_smem(*P);
  if (reference_mode) {
    // prefilter first (>= 2^12 bits), then the table if it fits
    unsigned pf = 12;
    const size_t room = rq.smem_limit > fixed + 4096 ? rq.smem_limit - fixed - 4096 : 0;
    sp.table_in_smem = sp.table_bytes + (size_t(1) << pf) / 8 <= room;
    const size_t left = room - (sp.table_in_smem ? sp.table_bytes : 0);
    const size_t nkeys = std::max<size_t>(pd.r, 1) * (!sp.overlapping && sp.q > 1 ? sp.q : 1);
    while (pf < 22 && (size_t(1) << (pf + 1)) / 8 <= left && (size_t(1) << pf) < 16 * nkeys) ++pf;
    sp.pf_bits = pf;
  } else {
    sp.table_in_smem = sp.verify_all ? 0 : 1;
    if (sp.direct)
      P->nwarps = best_warps ? best_warps
                             : (rq.warps > 0 ? std::min<uint32_t>(rq.warps, kMaxWarps) : kMaxWarps - 1);
  }
  sp.window_key = !sp.overlapping && !sp.verify_all && sp.q > 1;
  sp.wkey_len = sp.window_key ? static_cast<uint32_t>(std::min<size_t>(16, m - sp.q + 1)) : 0;
  if (sp.direct) sp.wkey_len = sp.q;  // the window key is the aligned sample itself
  sp.key_gram = sp.direct;
  sp.l2_bits = 0;
  if (sp.window_key) {  // ~128 bits per key: ~0.8% of screened keys walk a bucket
    unsigned lb = 16;
    while (lb < 30 && (size_t(1) << lb) < 128 * pd.r * sp.q) ++lb;
    sp.l2_bits = lb;
  }
  {
    const size_t keys = sp.window_key ? pd.r * sp.q : pd.r;
    unsigned bb = 4;
    while ((size_t(1) << bb) < 2 * keys && bb < 27) ++bb;
    sp.bucket_bits = bb;
  }
  // oversized rings (long patterns, wide windows): fewer warps per CTA
  while (!sp.direct && plan_smem(*P) > rq.smem_limit && P->nwarps > 1) P->nwarps /= 2;
  const size_t total = plan_smem(*P);
  if (total > rq.smem_limit) {
    *err = "plan needs " + std::to_string(total) + " bytes of shared memory (limit " +
           std::to_string(rq.smem_limit) + ")";
    return kBadConfig;
  }
  return kOk;
}

size_t plan_smem(const Plan& p) {
  if (p.sp.direct) return direct_smem(p.sp, p.nwarps);
  if (p.sp.pack2) return pack2_smem(p.sp.table_bytes, p.back, p.nwarps);
  if (p.sp.roll) return roll_smem(p.sp.roll_words, p.back, p.nwarps, p.sp.roll_step);
  return smem_layout(p.sp, p.slot_bytes, p.ring, p.nwarps).total;
}

// --------------------------------------------------------------- tables
static inline uint32_t gram_index_host(const Plan& P, const uint8_t* g) {
  const ScanPlan& sp = P.sp;
  if (sp.gram_mode == kGramExact) {
    uint32_t code = P.map[g[sp.q - 1]];
    for (int i = static_cast<int>(sp.q) - 2; i >= 0; --i) code = code * sp.sigma_prime + P.map[g[i]];
    return code;
  }
  return gram_slot(hash_gram_bytes(g, sp.q), sp.table_bits);
}

// Entries of a gram under multi-probe hashing (probes >= 2).
static inline uint64_t probe_entry(const ScanPlan& sp, uint32_t h, unsigned i) {
  return static_cast<uint64_t>(bloom_block(h, sp.blocks)) * 64 + bloom_bit(bloom_mix(h), i);
}

// Single-probe direct tables keep entry idx at bit (idx - 1) & 31 of word
// idx >> 5: the kernel's wrap-mode funnel shift by idx lands it at bit 31
// (scan_direct.cu rejects()).
static inline bool rotated_entries(const Plan& P) { return P.sp.direct && P.sp.probes <= 1; }

static inline void clear_bit(const Plan& P, std::vector<uint8_t>* t, uint64_t idx, unsigned b) {
  const unsigned el = P.sp.entry_log2;
  if (rotated_entries(P)) {
    uint32_t* w = reinterpret_cast<uint32_t*>(t->data());
    w[idx >> 5] &= ~(1u << ((idx - 1) & 31));
  } else if (el == 6) {
    uint64_t* w = reinterpret_cast<uint64_t*>(t->data());
    w[idx] &= ~(1ull << b);
  } else {
    uint32_t* w = reinterpret_cast<uint32_t*>(t->data());
    const uint64_t wi = idx >> (5 - el);
    const unsigned sh = static_cast<unsigned>((idx & ((32u >> el) - 1u)) << el);
    w[wi] &= ~(1u << (sh + b));
  }
}

uint64_t mask_entry(const Plan& P, const std::vector<uint8_t>& t, uint64_t idx) {
  const unsigned el = P.sp.entry_log2;
  if (rotated_entries(P))
    return ((reinterpret_cast<const uint32_t*>(t.data())[idx >> 5] >> ((idx - 1) & 31)) & 1u) | ~1ull;
  if (el == 6) return reinterpret_cast<const uint64_t*>(t.data())[idx];
  const uint32_t* w = reinterpret_cast<const uint32_t*>(t.data());
  const uint64_t wi = idx >> (5 - el);
  const unsigned sh = static_cast<unsigned>((idx & ((32u >> el) - 1u)) << el);
  const unsigned bits = 1u << el;
  const uint64_t v = (w[wi] >> sh) & (bits == 32 ? 0xffffffffull : ((1ull << bits) - 1));
  // widen: bits past the entry read as 1 (never admitted)
  return v | (bits >= 64 ? 0 : (~0ull << bits));
}

// superimpose.hpp:33-47 admissions streamed into masks (filter.hpp:27-31):
// class position c goes to alignment c % k, position c / k (P^j[i]=P[j+ik]).
void build_masks(const Plan& P, const PatternData& pd, std::vector<uint8_t>* table) {
  const ScanPlan& sp = P.sp;
  table->assign(sp.table_bytes, 0xff);
  if (sp.verify_all) {
    table->assign(sp.table_bytes, 0);
    return;
  }
  if (sp.pack2) {  // level-1 bitmap: codes of the patterns' first 10 symbols (bit set = present)
    table->assign(sp.table_bytes, 0);
    uint32_t* w = reinterpret_cast<uint32_t*>(table->data());
    for (size_t i = 0; i < pd.r; ++i) {
      const uint32_t c = pack2_code(pd.pattern(i), kPack2L1Bits / 2, sp.pack_shift);
      w[c >> 5] |= 1u << (c & 31);
    }
    return;
  }
  if (sp.roll) {  // Bloom words of the patterns' q-byte prefix hashes (bit set = present)
    table->assign(sp.table_bytes, 0);
    uint32_t* w = reinterpret_cast<uint32_t*>(table->data());
    for (size_t i = 0; i < pd.r; ++i) {
      const uint32_t h = roll_hash_bytes(pd.pattern(i), sp.q);
      const uint32_t wi = roll_word(h, sp.roll_words);
      for (unsigned j = 0; j < sp.probes; ++j)
        w[wi] |= 1u << (31u - (roll_probe_shift(h, static_cast<int>(j)) & 31u));
    }
    return;
  }
  const size_t m = pd.m;
  const unsigned q = sp.q;
  const size_t L = sp.overlapping ? m - q + 1 : (m - q + 1) / q;
  const unsigned shifts = sp.overlapping ? 1 : q;
  for (size_t i = 0; i < pd.r; ++i) {
    const uint8_t* p = pd.pattern(i);
    for (unsigned s = 0; s < shifts; ++s) {
      for (size_t c = 0; c < L; ++c) {
        const size_t align = c % sp.k, pos = c / sp.k;
        if (pos >= sp.m_prime) continue;
        const uint8_t* g = sp.overlapping ? p + c : p + s + c * q;
        if (sp.probes > 1) {
          const uint32_t hh = hash_gram_bytes(g, q);
          for (unsigned i = 0; i < sp.probes; ++i) clear_bit(P, table, probe_entry(sp, hh, i), 0);
          continue;
        }
        clear_bit(P, table, gram_index_host(P, g),
                  static_cast<unsigned>(align * sp.m_prime + pos));
      }
    }
  }
}

void build_pattern_table(const Plan& P, const PatternData& pd, PatternTable* pt) {
  const ScanPlan& sp = P.sp;
  const size_t r = pd.r;
  // (key, pattern | shift << 24): one per pattern, or one per (pattern,
  // shift) with window keys; bucket order = (shift descending, pattern
  // ascending) so hits come out in (start, pattern) order.
  struct Ent {
    uint32_t key, tag;
  };
  std::vector<Ent> ents;
  if (sp.window_key) {
    ents.reserve(r * sp.q);
    for (int s = static_cast<int>(sp.q) - 1; s >= 0; --s)
      for (size_t i = 0; i < r; ++i)
        ents.push_back({sp.key_gram ? hash_gram_bytes(pd.pattern(i) + s, sp.q)
                                    : key_bytes(pd.pattern(i) + s, sp.wkey_len),
                        static_cast<uint32_t>(i) | (static_cast<uint32_t>(s) << kPidBits)});
  } else {
    ents.reserve(r);
    for (size_t i = 0; i < r; ++i)
      ents.push_back({key_bytes(pd.pattern(i), sp.key_len), static_cast<uint32_t>(i)});
  }
  // prefilter: two probes per key (scan_kernels.cu prefilter_pass)
  const size_t pf_words = std::max<size_t>(4, (size_t(1) << sp.pf_bits) / 32);
  pt->prefilter.assign(align16(pf_words * 4) / 4, 0);
  if (sp.pf_bits) {
    for (const Ent& e : ents) {
      const uint32_t i1 = e.key >> (32 - sp.pf_bits);
      const uint32_t i2 = ((e.key ^ (e.key >> 15)) * 0x2C1B3C6Du) >> (32 - sp.pf_bits);
      pt->prefilter[i1 >> 5] |= 1u << (i1 & 31);
      pt->prefilter[i2 >> 5] |= 1u << (i2 & 31);
    }
  }
  // L2 screen bitmap (window keys): top key bits
  pt->l2map.assign(sp.l2_bits ? std::max<size_t>(4, (size_t(1) << sp.l2_bits) / 32) : 4, 0);
  if (sp.l2_bits) {
    // direct plans: bit b sits at (b - 1) & 31 of word b >> 5, so the kernel's
    // rotate by the key lands it at bit 31 (scan_direct.cu resolve())
    const uint32_t rot = sp.direct ? 31u : 0u;
    for (const Ent& e : ents) {
      const uint32_t b = screen_bit(e.key, sp.l2_bits);
      pt->l2map[b >> 5] |= 1u << ((b + rot) & 31);
    }
  }
  // roll plans: open addressing by the start key, linear probing; patterns
  // inserted in id order, so equal keys are met in id order along a probe run
  pt->vtab.assign(8 * 16, 0);
  pt->vmask = 0;
  if (sp.pack2) {  // level 2: open addressing by the exact code of the first kb = q symbols
    size_t slots = 16;  // load factor <= 1/8: a missing key's home slot is empty 7 times in 8
    uint32_t bits = 4;
    while (slots < 8 * r) {
      slots <<= 1;
      ++bits;
    }
    pt->vmask = static_cast<uint32_t>(slots - 1);
    pt->vbits = bits;
    pt->vtab.assign(8 * slots, 0);
    for (size_t i = 0; i < slots; ++i) pt->vtab[8 * i + 1] = 0xffffffffu;
    for (size_t i = 0; i < r; ++i) {
      const uint32_t code = pack2_code(pd.pattern(i), sp.q, sp.pack_shift);
      size_t s = pack2_home(code, bits);
      while (pt->vtab[8 * s + 1] != 0xffffffffu) s = (s + 1) & pt->vmask;
      uint32_t* e = &pt->vtab[8 * s];
      e[0] = code;
      e[1] = static_cast<uint32_t>(i);
      e[2] = pd.len[i];
      e[3] = static_cast<uint32_t>(pd.off[i] / 16);
      std::memcpy(e + 4, pd.pattern(i), 16);
    }
    for (size_t i = 0; i < slots; ++i)
      if (pt->vtab[8 * i + 1] != 0xffffffffu && pt->vtab[8 * ((i + 1) & pt->vmask) + 1] != 0xffffffffu)
        pt->vtab[8 * i + 2] |= 0x80000000u;
  }
  if (sp.roll && sp.roll_step == static_cast<uint32_t>(kRollStepEq)) {
    // Equal-length sets of m <= 12 bytes: 32-byte sectors of two 16-byte
    // entries {pattern (zero padded to 12 bytes), pid | F << 31}; empty
    // entries have the pid word 0xffffffff.  Pass 1 places every pattern in
    // its home sector while that has room (id order: entry 0 before entry
    // 1); pass 2 moves the others to the next sector with room and sets F
    // in the HOME sector's entry 0: "patterns of this home live further
    // along" — the only case in which the kernel walks on (~0.4% of the
    // patterns at <= 0.125 patterns per sector).
    size_t sectors = 16;
    // cfg5 (r = 100k), sectors >= 4r / 8r / 16r: 774 / 805 / 812 GB/s (fewer
    // overflowing home sectors, hence fewer walks); 8r = 32 MiB stays a
    // quarter of L2
    while (sectors < (r <= (size_t(1) << 20) ? 8 : 4) * r) sectors <<= 1;
    pt->vmask = static_cast<uint32_t>(sectors - 1);
    pt->vtab.assign(8 * sectors, 0);
    for (size_t i = 0; i < 2 * sectors; ++i) pt->vtab[4 * i + 3] = 0xffffffffu;
    auto put = [&](size_t sec, size_t i) -> bool {
      for (int e = 0; e < 2; ++e) {
        uint32_t* w = &pt->vtab[8 * sec + 4 * e];
        if (w[3] != 0xffffffffu) continue;
        std::memcpy(w, pd.pattern(i), 12);  // patterns are zero padded to 16 bytes
        w[3] = static_cast<uint32_t>(i);
        return true;
      }
      return false;
    };
    std::vector<uint8_t> placed(r, 0);
    std::vector<uint32_t> keys(r);
    for (size_t i = 0; i < r; ++i) {
      keys[i] = key_bytes(pd.pattern(i), sp.key_len);
      placed[i] = put(keys[i] & pt->vmask, i);
    }
    for (size_t i = 0; i < r; ++i) {
      if (placed[i]) continue;
      const size_t home = keys[i] & pt->vmask;
      size_t sec = home;
      do sec = (sec + 1) & pt->vmask; while (!put(sec, i));
      pt->vtab[8 * home + 3] |= 0x80000000u;
    }
  } else if (sp.roll) {
    size_t slots = 16;
    while (slots < 4 * r) slots <<= 1;  // load factor <= 1/4
    pt->vmask = static_cast<uint32_t>(slots - 1);
    pt->vtab.assign(8 * slots, 0);
    for (size_t i = 0; i < slots; ++i) pt->vtab[8 * i + 1] = 0xffffffffu;
    auto put = [&](size_t s, size_t i, uint32_t key) {
      uint32_t* e = &pt->vtab[8 * s];  // {len | F << 31, pid, key, pattern offset / 16}
      e[0] = pd.len[i];
      e[1] = static_cast<uint32_t>(i);
      e[2] = key;
      e[3] = static_cast<uint32_t>(pd.off[i] / 16);
      std::memcpy(e + 4, pd.pattern(i), 16);  // patterns are zero padded to 16 bytes
    };
    // Pass 1: every home slot goes to the first (lowest id) pattern that
    // hashes there, so a lookup of a key whose home holds one pattern is ONE
    // L2 round trip.  Pass 2: the others, in id order, probe linearly from
    // their home (equal keys are therefore met in id order along a run) and
    // set bit 31 of their HOME slot's len word: "patterns of this home live
    // further along" — the only case in which the kernel walks on.
    std::vector<uint32_t> keys(r);
    std::vector<uint8_t> placed(r, 0);
    for (size_t i = 0; i < r; ++i) {
      keys[i] = key_bytes(pd.pattern(i), sp.key_len);
      const size_t s = keys[i] & pt->vmask;
      if (pt->vtab[8 * s + 1] == 0xffffffffu) {
        put(s, i, keys[i]);
        placed[i] = 1;
      }
    }
    for (size_t i = 0; i < r; ++i) {
      if (placed[i]) continue;
      const size_t home = keys[i] & pt->vmask;
      size_t s = home;
      while (pt->vtab[8 * s + 1] != 0xffffffffu) s = (s + 1) & pt->vmask;
      put(s, i, keys[i]);
      pt->vtab[8 * home] |= 0x80000000u;
    }
  }
  // buckets by low key bits, stable within a bucket
  const size_t nb = size_t(1) << sp.bucket_bits;
  pt->bucket_start.assign(nb + 1, 0);
  for (const Ent& e : ents) pt->bucket_start[(e.key & (nb - 1)) + 1]++;
  for (size_t b = 0; b < nb; ++b) pt->bucket_start[b + 1] += pt->bucket_start[b];
  std::vector<uint32_t> cursor(pt->bucket_start.begin(), pt->bucket_start.end() - 1);
  pt->entries.assign(2 * std::max<size_t>(ents.size(), 1), 0);
  for (const Ent& e : ents) {
    const uint32_t x = cursor[e.key & (nb - 1)]++;
    pt->entries[2 * x] = e.key;
    pt->entries[2 * x + 1] = e.tag;
  }
}

FilterRates measure_filter(const Plan& P, const PatternData& pd, const std::vector<uint8_t>& table,
                           const uint8_t* text, size_t n) {
  const ScanPlan& sp = P.sp;
  FilterRates R;
  if (n == 0) return R;
  if (sp.verify_all) {
    R.candidates = 1.0;
    return R;
  }
  // Verification keys of the plan (build_pattern_table), sorted: a candidate
  // whose key is among them is a survivor, and walks every entry sharing it.
  const bool wkey = sp.window_key != 0;
  const unsigned klen = sp.direct ? sp.q : (wkey ? sp.wkey_len : sp.key_len);
  std::vector<uint32_t> keys;
  // (sets beyond 2^25 keys are measured for candidates only: no key index)
  const bool index_keys = pd.r * (wkey ? sp.q : 1u) <= (size_t(1) << 25);
  if (index_keys) {
    const unsigned shifts = wkey ? sp.q : 1;
    keys.reserve(pd.r * shifts);
    for (size_t i = 0; i < pd.r; ++i)
      for (unsigned s = 0; s < shifts; ++s)
        keys.push_back(sp.key_gram ? hash_gram_bytes(pd.pattern(i) + s, sp.q)
                       : sp.pack2  ? pack2_code(pd.pattern(i), sp.q, sp.pack_shift)
                                   : key_bytes(pd.pattern(i) + s, klen));
    std::sort(keys.begin(), keys.end());
  }
  uint64_t cands = 0, surv = 0, walked = 0;
  // a candidate whose verification key is read at text offset a
  auto verify_at = [&](uint64_t a) {
    if (!index_keys || a + klen > n) return;
    const uint32_t key = sp.key_gram ? hash_gram_bytes(text + a, sp.q)
                         : sp.pack2  ? pack2_code(text + a, sp.q, sp.pack_shift)
                                     : key_bytes(text + a, klen);
    const auto range = std::equal_range(keys.begin(), keys.end(), key);
    if (range.first == range.second) return;
    ++surv;
    walked += static_cast<uint64_t>(range.second - range.first);
  };
  const uint32_t* w32 = reinterpret_cast<const uint32_t*>(table.data());
  if (sp.pack2) {  // level 1: the first 10 symbols' code
    const unsigned sym = kPack2L1Bits / 2;
    for (size_t p = 0; p + sym <= n; ++p) {
      const uint32_t c = pack2_code(text + p, sym, sp.pack_shift);
      if ((w32[c >> 5] >> (c & 31)) & 1u) {
        ++cands;
        verify_at(p);
      }
    }
  } else if (sp.roll) {  // every position's q-byte prefix hash against its Bloom word
    const uint32_t bq = roll_pow(sp.q);
    uint32_t h = n >= sp.q ? roll_hash_bytes(text, sp.q) : 0;
    for (size_t p = 0; p + sp.q <= n; ++p) {
      const uint32_t wd = w32[roll_word(h, sp.roll_words)];
      bool hit = true;
      for (unsigned j = 0; j < sp.probes; ++j)
        hit = hit && ((wd >> (31u - (roll_probe_shift(h, static_cast<int>(j)) & 31u))) & 1u);
      if (hit) {
        ++cands;
        verify_at(p);
      }
      if (p + sp.q < n) h = h * kRollB + text[p + sp.q] - text[p] * bq;
    }
  } else {
    // the Shift-Or machine of filter.hpp:58-73 (direct plans are its
    // q = W, k = m' = 1 case): d = ((d << 1) & keep) | mask[gram]
    uint64_t keep = ~0ull;
    for (unsigned j = 0; j < sp.k; ++j) keep &= ~(1ull << (j * sp.m_prime));
    const uint64_t T = filter_reads(P, n);
    uint64_t d = ~0ull;
    for (uint64_t t = 0; t < T; ++t) {
      const uint64_t u = sp.overlapping ? t : (t + 1) * sp.k - 1;
      const uint8_t* g = text + (sp.overlapping ? u : u * sp.q);
      uint64_t mv;
      if (sp.probes > 1) {
        const uint32_t hh = hash_gram_bytes(g, sp.q);
        mv = 0;
        for (unsigned i = 0; i < sp.probes; ++i) mv |= mask_entry(P, table, probe_entry(sp, hh, i)) & 1ull;
        mv |= ~1ull;
      } else {
        mv = mask_entry(P, table, gram_index_host(P, g));
      }
      d = ((d << 1) & keep) | mv;
      for (uint64_t hits = ~d & sp.match_mask; hits; hits &= hits - 1) {
        ++cands;
        const unsigned j = static_cast<unsigned>(__builtin_ctzll(hits)) / sp.m_prime;
        const uint64_t back = j + static_cast<uint64_t>(sp.m_prime - 1) * sp.k;
        if (u < back) continue;
        const uint64_t ss = u - back;  // the candidate's super start (filter.hpp:66-70)
        if (sp.overlapping || wkey) {
          verify_at(sp.overlapping ? ss : ss * sp.q);  // one start / one window key at the gram boundary
        } else {  // start keys: every start of the window [q ss - (q - 1), q ss]
          for (uint64_t s = 0; s < sp.q && s <= ss * sp.q; ++s) verify_at(ss * sp.q - s);
        }
      }
    }
  }
  R.candidates = static_cast<double>(cands) / static_cast<double>(n);
  R.survivors = static_cast<double>(surv) / static_cast<double>(n);
  R.walked = static_cast<double>(walked) / static_cast<double>(n);
  return R;
}

int make_plan_measured(const PatternData& pd, const Histogram& h, const PlanRequest& rq,
                       const uint8_t* sample, size_t sample_len, Plan* P, std::string* err) {
  const int rc = make_plan(pd, h, rq, P, err);
  if (rc != 0 || !sample || sample_len < 4096 || sample_len < 4 * pd.m) return rc;
  const size_t n = std::min<size_t>(sample_len, size_t(1) << 20);
  auto measure = [&](Plan* pl) {
    std::vector<uint8_t> table;
    build_masks(*pl, pd, &table);
    const FilterRates fr = measure_filter(*pl, pd, table, sample, n);
    pl->meas_cand_per_byte = fr.candidates;
    pl->meas_surv_per_byte = fr.survivors;
    pl->meas_walk_per_byte = fr.walked;
    pl->meas_sample_bytes = n;
    double cost = pl->pred_cost + pl->cost_slope * (pl->meas_cand_per_byte - pl->pred_cand_per_byte);
    // direct plans price the survivors of the L2 screen separately
    if (pl->sp.direct) cost += pl->surv_slope * (pl->meas_surv_per_byte - pl->pred_surv_per_byte);
    // every family: entries walked beyond one per survivor cost a serial L2
    // round trip each, in one lane of the warp (B200: word-Zipf text whose
    // survivors walk ~300 entries ran the direct kernel at 1 GB/s, i.e.
    // ~1,500 per walked entry in this unit)
    cost += kCostWalkEntry * std::max(0.0, pl->meas_walk_per_byte - pl->meas_surv_per_byte);
    pl->meas_cost = std::max(0.0, cost);
  };
  measure(P);
  P->meas_plans = 1;
  // pinned plans are only measured: reference parameters, a forced kernel,
  // fixed q / table / probes / ring options
  const bool pinned = P->sp.gram_mode == kGramExact || rq.kernel != 0 || rq.q || rq.k || rq.table_bits ||
                      rq.probes || rq.stages || rq.tile_bytes || rq.variant == 1;
  if (pinned) return rc;
  struct Family {
    int kernel, q;
  };
  static const Family kFamilies[] = {{1, 0}, {2, 16}, {2, 8}, {3, 0}};
  Plan best = *P;
  uint32_t measured = 1;
  for (const Family& f : kFamilies) {
    PlanRequest r2 = rq;
    r2.kernel = f.kernel;
    r2.gram_mode = 1;  // a fixed q would otherwise select the reference's exact-code path
    r2.q = f.q;
    Plan alt;
    std::string e2;
    if (make_plan(pd, h, r2, &alt, &e2) != 0) continue;
    const bool same = alt.sp.direct == P->sp.direct && alt.sp.roll == P->sp.roll && alt.sp.q == P->sp.q &&
                      alt.sp.k == P->sp.k && alt.sp.m_prime == P->sp.m_prime &&
                      alt.sp.table_bits == P->sp.table_bits && alt.sp.probes == P->sp.probes &&
                      alt.sp.overlapping == P->sp.overlapping && alt.sp.verify_all == P->sp.verify_all;
    if (same) continue;
    measure(&alt);
    ++measured;
    // a clear margin: the calibrated analytic choice stands on near ties
    if (alt.meas_cost < 0.9 * best.meas_cost) best = alt;
  }
  *P = best;
  P->meas_plans = measured;
  return rc;
}

uint64_t filter_reads(const Plan& P, uint64_t n) {
  const ScanPlan& sp = P.sp;
  if (sp.overlapping) return n >= sp.q ? n - sp.q + 1 : 0;
  return (n / sp.q) / sp.k;
}

void sample_offsets(size_t corpus_len, size_t count, size_t length, uint64_t seed,
                    std::vector<uint64_t>* out) {
  uint64_t s = seed;
  const uint64_t span = corpus_len - length + 1;
  out->resize(count);
  for (size_t i = 0; i < count; ++i) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    (*out)[i] = z % span;
  }
}

}  // namespace magb
