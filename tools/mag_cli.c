/*
 * mag_cli — command-line front end over the mag.h C ABI.
 *
 * A plain C caller of the reference interface: it compiles against either
 * this repo's include/mag.h or the reference's proj/include/mag.h unchanged
 * and links libmag_b200.so.  Subcommands:
 *
 *   search --patterns FILE --text FILE [--variant mag|smag|shiftor_og]
 *          [--q N] [--k N] [--sigma-prime N]
 *          [--mapping identity|freq|balance|lowbits:L] [--count]
 *       one "pattern_index\toffset\n" line per occurrence, sorted
 *       (SPEC.md:514-518); --count prints only the total.
 *   bench  --text FILE [--name NAME] [--variant V[,V...]] [--r R[,R...]]
 *          [--m M[,M...]] [--seed S] [--reps N] [--check] [--include-prep]
 *          [--q N] [--k N] [--sigma-prime N] [--mapping M] [--csv]
 *       the section-4 benchmark matrix: for every
 *       (variant x r x m) cell, r patterns of length m sampled from the text
 *       (mag_sample_patterns, seeded), one BenchRow CSV line (SPEC.md:
 *       500-502) under the header below.  mb_per_s = n / seconds / 2^20 of
 *       the median of --reps searches (mag_search_prepared: text already
 *       prepared); --include-prep adds engine creation and mag_prepare_text
 *       to every timed run.  --check verifies every reported occurrence
 *       byte-for-byte, the (offset, pattern_index) order, and the count
 *       against a rolling-hash dictionary scan of the text (exit 1 on a
 *       mismatch).  Defaults: r {10,100,1000,10000}, m {8,16,32,64}, variant
 *       mag.
 *   tune   --sigma S --r R --m M [--n N] [--sigma-prime N] [--word-bits W]
 *       the reference tuner's choice (mag_tune), one "key=value" per line.
 *   gen    --corpus FILE --r R --m M [--seed S]
 *       seeded corpus substrings (mag_sample_patterns), one per line.
 *
 * Pattern files hold one pattern per line (a trailing '\r' is kept: the
 * bytes are the pattern).  Errors: message on stderr, exit code 2 for usage,
 * 1 for library errors (mag_status_string + mag_last_error).
 */
#define _POSIX_C_SOURCE 200809L
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "mag.h"

static int usage(void) {
  fprintf(stderr,
          "usage: mag_cli search --patterns FILE --text FILE [--variant V] [--q N] [--k N]\n"
          "                      [--sigma-prime N] [--mapping M|lowbits:L] [--count]\n"
          "       mag_cli bench --text FILE [--name NAME] [--variant V,..] [--r R,..] [--m M,..]\n"
          "                     [--seed S] [--reps N] [--check] [--include-prep] [--q N] [--k N]\n"
          "                     [--sigma-prime N] [--mapping M|lowbits:L] [--csv]\n"
          "       mag_cli tune --sigma S --r R --m M [--n N] [--sigma-prime N] [--word-bits W]\n"
          "       mag_cli gen --corpus FILE --r R --m M [--seed S]\n");
  return 2;
}

static int lib_error(const char* what, mag_status s) {
  fprintf(stderr, "mag_cli: %s: %s: %s\n", what, mag_status_string(s), mag_last_error());
  return 1;
}

static uint8_t* read_file(const char* path, size_t* len) {
  FILE* f = fopen(path, "rb");
  if (!f) return NULL;
  size_t cap = 1 << 20, n = 0;
  uint8_t* buf = (uint8_t*)malloc(cap);
  while (buf) {
    size_t got = fread(buf + n, 1, cap - n, f);
    n += got;
    if (n < cap) break;
    cap *= 2;
    uint8_t* nb = (uint8_t*)realloc(buf, cap);
    if (!nb) {
      free(buf);
      buf = NULL;
    }
    buf = nb;
  }
  fclose(f);
  *len = n;
  return buf;
}

static const char* arg(int argc, char** argv, const char* name) {
  for (int i = 2; i + 1 < argc; ++i)
    if (!strcmp(argv[i], name)) return argv[i + 1];
  return NULL;
}

static int flag(int argc, char** argv, const char* name) {
  for (int i = 2; i < argc; ++i)
    if (!strcmp(argv[i], name)) return 1;
  return 0;
}

static int parse_variant(const char* v, int* out) {
  if (!strcmp(v, "mag")) *out = MAG_VARIANT_MAG;
  else if (!strcmp(v, "smag")) *out = MAG_VARIANT_SMAG;
  else if (!strcmp(v, "shiftor_og")) *out = MAG_VARIANT_SHIFTOR_OG;
  else if (!strcmp(v, "naive")) *out = MAG_VARIANT_NAIVE;
  else if (!strcmp(v, "ac")) *out = MAG_VARIANT_AC;
  else return 0;
  return 1;
}

static const char* variant_name(int v) {
  static const char* names[] = {"mag", "smag", "shiftor_og", "naive", "ac"};
  return v >= 0 && v < 5 ? names[v] : "?";
}

/* --variant (one name), --q, --k, --sigma-prime, --mapping into o */
static int parse_options(int argc, char** argv, const char* variant, mag_options* o) {
  mag_options_init(o);
  if (variant) {
    int v;
    if (!parse_variant(variant, &v)) return 0;
    o->variant = v;
  }
  const char* x;
  if ((x = arg(argc, argv, "--q"))) o->q = atoi(x);
  if ((x = arg(argc, argv, "--k"))) o->k = atoi(x);
  if ((x = arg(argc, argv, "--sigma-prime"))) o->sigma_prime = atoi(x);
  if ((x = arg(argc, argv, "--mapping"))) {
    if (!strcmp(x, "identity")) o->mapping = MAG_MAPPING_IDENTITY;
    else if (!strcmp(x, "freq")) o->mapping = MAG_MAPPING_FREQUENCY;
    else if (!strcmp(x, "balance")) o->mapping = MAG_MAPPING_BALANCED;
    else if (!strncmp(x, "lowbits:", 8)) {
      o->mapping = MAG_MAPPING_LOWBITS;
      o->lowbits = atoi(x + 8);
    } else {
      return 0;
    }
  }
  return 1;
}

static int cmd_search(int argc, char** argv) {
  const char* pf = arg(argc, argv, "--patterns");
  const char* tf = arg(argc, argv, "--text");
  if (!pf || !tf) return usage();
  mag_options o;
  if (!parse_options(argc, argv, arg(argc, argv, "--variant"), &o)) return usage();
  size_t plen = 0, tlen = 0;
  uint8_t* pbuf = read_file(pf, &plen);
  if (!pbuf) {
    fprintf(stderr, "mag_cli: cannot read %s\n", pf);
    return 2;
  }
  uint8_t* text = read_file(tf, &tlen);
  if (!text) {
    fprintf(stderr, "mag_cli: cannot read %s\n", tf);
    free(pbuf);
    return 2;
  }
  /* one pattern per line; a final line without '\n' counts */
  size_t r = 0;
  for (size_t i = 0; i < plen; ++i) r += pbuf[i] == '\n';
  if (plen && pbuf[plen - 1] != '\n') ++r;
  const uint8_t** pats = (const uint8_t**)malloc((r ? r : 1) * sizeof(*pats));
  size_t* lens = (size_t*)malloc((r ? r : 1) * sizeof(*lens));
  size_t s = 0, j = 0;
  for (size_t i = 0; i <= plen && j < r; ++i) {
    if (i == plen || pbuf[i] == '\n') {
      pats[j] = pbuf + s;
      lens[j] = i - s;
      ++j;
      s = i + 1;
    }
  }
  int rc = 0;
  mag_engine* e = NULL;
  mag_matches* m = NULL;
  mag_status st = mag_engine_create(pats, lens, r, &o, &e);
  if (st != MAG_OK) {
    rc = lib_error("engine", st);
    goto done;
  }
  st = mag_search(e, text, tlen, &m);
  if (st != MAG_OK) {
    rc = lib_error("search", st);
    goto done;
  }
  {
    const size_t cnt = mag_matches_count(m);
    if (flag(argc, argv, "--count")) {
      printf("%zu\n", cnt);
    } else {
      for (size_t i = 0; i < cnt; ++i) {
        uint32_t pid;
        size_t off;
        st = mag_matches_get(m, i, &pid, &off);
        if (st != MAG_OK) {
          rc = lib_error("matches", st);
          break;
        }
        printf("%u\t%zu\n", pid, off);
      }
    }
  }
done:
  mag_matches_destroy(m);
  mag_engine_destroy(e);
  free(pats);
  free(lens);
  free(pbuf);
  free(text);
  return rc;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* comma-separated size_t list; returns the count (0 on a parse error) */
static size_t parse_list(const char* s, size_t* out, size_t cap) {
  size_t n = 0;
  while (s && *s && n < cap) {
    char* end;
    const unsigned long long v = strtoull(s, &end, 10);
    if (end == s || v == 0) return 0;
    out[n++] = (size_t)v;
    if (*end == ',') ++end;
    else if (*end) return 0;
    s = end;
  }
  return n;
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : x > y;
}

/* --check: the occurrence count of r equal-length patterns, by a rolling
 * (Rabin-Karp, mod 2^64) hash of every length-m window looked up in an
 * open-addressing table of the pattern hashes, with a byte compare on every
 * hash hit.  Independent of the library (test path of the CLI only). */
static size_t dictionary_count(const uint8_t* t, size_t n, const uint8_t* const* pats, size_t r,
                               size_t m) {
  if (m > n) return 0;
  const uint64_t B = 0x100000001b3ull;
  uint64_t Bm = 1;
  for (size_t i = 0; i < m; ++i) Bm *= B;
  size_t cap = 16;
  while (cap < 2 * r) cap <<= 1;
  uint64_t* hk = (uint64_t*)calloc(cap, sizeof(uint64_t));
  size_t* hv = (size_t*)malloc(cap * sizeof(size_t));
  uint8_t* used = (uint8_t*)calloc(cap, 1);
  for (size_t p = 0; p < r; ++p) {
    uint64_t h = 0;
    for (size_t i = 0; i < m; ++i) h = h * B + pats[p][i];
    size_t s = (size_t)(h * 0x9e3779b97f4a7c15ull >> 17) & (cap - 1);
    while (used[s]) s = (s + 1) & (cap - 1);
    used[s] = 1;
    hk[s] = h;
    hv[s] = p;
  }
  size_t count = 0;
  uint64_t h = 0;
  for (size_t i = 0; i < m; ++i) h = h * B + t[i];
  for (size_t a = 0;; ++a) {
    for (size_t s = (size_t)(h * 0x9e3779b97f4a7c15ull >> 17) & (cap - 1); used[s]; s = (s + 1) & (cap - 1))
      if (hk[s] == h && !memcmp(pats[hv[s]], t + a, m)) ++count;
    if (a + m >= n) break;
    h = h * B + t[a + m] - Bm * t[a];
  }
  free(hk);
  free(hv);
  free(used);
  return count;
}

/* every reported occurrence is genuine and strictly (offset, pattern) ordered */
static int check_matches(const mag_matches* mm, const uint8_t* t, size_t n, const uint8_t* const* pats,
                         size_t m, size_t want) {
  const size_t cnt = mag_matches_count(mm);
  if (cnt != want) {
    fprintf(stderr, "mag_cli: check: %zu occurrences, the dictionary scan finds %zu\n", cnt, want);
    return 0;
  }
  size_t lo = 0;
  uint32_t lp = 0;
  for (size_t i = 0; i < cnt; ++i) {
    uint32_t pid;
    size_t off;
    if (mag_matches_get(mm, i, &pid, &off) != MAG_OK || off + m > n || memcmp(pats[pid], t + off, m) ||
        (i && (off < lo || (off == lo && pid <= lp)))) {
      fprintf(stderr, "mag_cli: check: occurrence %zu (pattern %u at %zu) is wrong or out of order\n", i,
              pid, off);
      return 0;
    }
    lo = off;
    lp = pid;
  }
  return 1;
}

static const char* mapping_name(int mapping, int lowbits, char* buf, size_t cap) {
  switch (mapping) {
    case MAG_MAPPING_IDENTITY: return "identity";
    case MAG_MAPPING_FREQUENCY: return "freq";
    case MAG_MAPPING_BALANCED: return "balance";
    case MAG_MAPPING_LOWBITS: snprintf(buf, cap, "lowbits:%d", lowbits); return buf;
  }
  return "auto";
}

static int cmd_bench(int argc, char** argv) {
  const char* tf = arg(argc, argv, "--text");
  if (!tf) tf = arg(argc, argv, "--corpus");
  if (!tf) return usage();
  size_t rs[64], ms[64];
  size_t nr = parse_list(arg(argc, argv, "--r") ? arg(argc, argv, "--r") : "10,100,1000,10000", rs, 64);
  size_t nm = parse_list(arg(argc, argv, "--m") ? arg(argc, argv, "--m") : "8,16,32,64", ms, 64);
  if (!nr || !nm) return usage();
  int variants[8];
  size_t nv = 0;
  {
    const char* vl = arg(argc, argv, "--variant");
    char buf[256];
    snprintf(buf, sizeof buf, "%s", vl ? vl : "mag");
    for (char* tok = strtok(buf, ","); tok && nv < 8; tok = strtok(NULL, ","))
      if (!parse_variant(tok, &variants[nv++])) return usage();
  }
  mag_options o;
  if (!parse_options(argc, argv, NULL, &o)) return usage();
  const char* x;
  const uint64_t seed = (x = arg(argc, argv, "--seed")) ? strtoull(x, NULL, 10) : 0;
  int reps = (x = arg(argc, argv, "--reps")) ? atoi(x) : 3;
  if (reps < 1 || reps > 1000) return usage();
  const int check = flag(argc, argv, "--check"), prep = flag(argc, argv, "--include-prep");
  const char* name = arg(argc, argv, "--name");
  if (!name) {
    name = strrchr(tf, '/');
    name = name ? name + 1 : tf;
  }
  size_t n = 0;
  uint8_t* text = read_file(tf, &n);
  if (!text) {
    fprintf(stderr, "mag_cli: cannot read %s\n", tf);
    return 2;
  }
  printf("dataset,variant,r,m,q,k,sigma_prime,mapping,mb_per_s,filter_reads,candidates,occurrences\n");
  int rc = 0;
  double* times = (double*)malloc((size_t)reps * sizeof(double));
  for (size_t vi = 0; vi < nv && !rc; ++vi) {
    for (size_t ri = 0; ri < nr && !rc; ++ri) {
      for (size_t mi = 0; mi < nm && !rc; ++mi) {
        const size_t r = rs[ri], m = ms[mi];
        mag_patterns* ps = NULL;
        mag_engine* e = NULL;
        mag_prepared* p = NULL;
        mag_matches* mm = NULL;
        const uint8_t** pats = (const uint8_t**)malloc(r * sizeof(*pats));
        size_t* lens = (size_t*)malloc(r * sizeof(*lens));
        o.variant = variants[vi];
        mag_status st = mag_sample_patterns(text, n, r, m, seed, &ps);
        if (st != MAG_OK) {
          rc = lib_error("gen", st);
          goto cell_done;
        }
        for (size_t i = 0; i < r; ++i) mag_patterns_get(ps, i, &pats[i], &lens[i]);
        for (int rep = 0; rep < reps; ++rep) {
          double t0 = now_s();
          if (!e || prep) {
            mag_matches_destroy(mm);
            mag_prepared_destroy(p);
            mag_engine_destroy(e);
            mm = NULL;
            p = NULL;
            e = NULL;
            if ((st = mag_engine_create(pats, lens, r, &o, &e)) != MAG_OK) {
              rc = lib_error("engine", st);
              goto cell_done;
            }
            if ((st = mag_prepare_text(e, text, n, &p)) != MAG_OK) {
              rc = lib_error("prepare", st);
              goto cell_done;
            }
          }
          if (!prep) t0 = now_s();
          mag_matches_destroy(mm);
          mm = NULL;
          if ((st = mag_search_prepared(e, p, &mm)) != MAG_OK) {
            rc = lib_error("search", st);
            goto cell_done;
          }
          mag_matches_count(mm);
          times[rep] = now_s() - t0;
        }
        qsort(times, (size_t)reps, sizeof(double), cmp_double);
        {
          mag_engine_info info;
          mag_metrics met;
          char mb[32];
          if ((st = mag_engine_get_info(e, &info)) != MAG_OK || (st = mag_matches_metrics(mm, &met)) != MAG_OK) {
            rc = lib_error("metrics", st);
            goto cell_done;
          }
          const double secs = times[reps / 2] > 1e-9 ? times[reps / 2] : 1e-9;
          printf("%s,%s,%zu,%zu,%d,%d,%d,%s,%.3f,%llu,%llu,%zu\n", name, variant_name(info.variant), r, m,
                 info.q, info.k, info.sigma_prime, mapping_name(info.mapping, o.lowbits, mb, sizeof mb),
                 (double)n / secs / 1048576.0, (unsigned long long)met.filter_reads,
                 (unsigned long long)met.candidates, mag_matches_count(mm));
          fflush(stdout);
          if (check && !check_matches(mm, text, n, pats, m, dictionary_count(text, n, pats, r, m))) rc = 1;
        }
      cell_done:
        mag_matches_destroy(mm);
        mag_prepared_destroy(p);
        mag_engine_destroy(e);
        mag_patterns_destroy(ps);
        free(pats);
        free(lens);
      }
    }
  }
  free(times);
  free(text);
  return rc;
}

static int cmd_tune(int argc, char** argv) {
  const char *a = arg(argc, argv, "--sigma"), *r = arg(argc, argv, "--r"), *m = arg(argc, argv, "--m");
  if (!a || !r || !m) return usage();
  mag_tuning_input ti;
  memset(&ti, 0, sizeof ti);
  ti.sigma = (uint32_t)strtoul(a, NULL, 10);
  ti.r = strtoull(r, NULL, 10);
  ti.m = strtoull(m, NULL, 10);
  const char* x;
  ti.n = (x = arg(argc, argv, "--n")) ? strtoull(x, NULL, 10) : (1u << 20);
  if ((x = arg(argc, argv, "--sigma-prime"))) ti.sigma_prime = (uint32_t)strtoul(x, NULL, 10);
  if ((x = arg(argc, argv, "--word-bits"))) ti.word_bits = (uint32_t)strtoul(x, NULL, 10);
  mag_tuning_result out;
  mag_status st = mag_tune(&ti, &out);
  if (st != MAG_OK) return lib_error("tune", st);
  printf("q=%d\nk=%d\nsigma_prime=%d\nrho=%.6g\npredicted_p=%.6g\npredicted_cost=%.6g\n", out.q, out.k,
         out.sigma_prime, out.rho, out.predicted_p, out.predicted_cost);
  return 0;
}

static int cmd_gen(int argc, char** argv) {
  const char *c = arg(argc, argv, "--corpus"), *r = arg(argc, argv, "--r"), *m = arg(argc, argv, "--m");
  if (!c || !r || !m) return usage();
  const char* x = arg(argc, argv, "--seed");
  const uint64_t seed = x ? strtoull(x, NULL, 10) : 0;
  size_t n = 0;
  uint8_t* corpus = read_file(c, &n);
  if (!corpus) {
    fprintf(stderr, "mag_cli: cannot read %s\n", c);
    return 2;
  }
  mag_patterns* ps = NULL;
  mag_status st = mag_sample_patterns(corpus, n, strtoull(r, NULL, 10), strtoull(m, NULL, 10), seed, &ps);
  int rc = 0;
  if (st != MAG_OK) {
    rc = lib_error("gen", st);
  } else {
    for (size_t i = 0; i < mag_patterns_count(ps); ++i) {
      const uint8_t* b;
      size_t len;
      if (mag_patterns_get(ps, i, &b, &len) != MAG_OK) break;
      fwrite(b, 1, len, stdout);
      fputc('\n', stdout);
    }
  }
  mag_patterns_destroy(ps);
  free(corpus);
  return rc;
}

int main(int argc, char** argv) {
  if (argc < 2) return usage();
  if (!strcmp(argv[1], "search")) return cmd_search(argc, argv);
  if (!strcmp(argv[1], "bench")) return cmd_bench(argc, argv);
  if (!strcmp(argv[1], "tune")) return cmd_tune(argc, argv);
  if (!strcmp(argv[1], "gen")) return cmd_gen(argc, argv);
  return usage();
}
