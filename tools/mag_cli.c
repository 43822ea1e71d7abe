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
 *   tune   --sigma S --r R --m M [--n N] [--sigma-prime N] [--word-bits W]
 *       the reference tuner's choice (mag_tune), one "key=value" per line.
 *   gen    --corpus FILE --r R --m M [--seed S]
 *       seeded corpus substrings (mag_sample_patterns), one per line.
 *
 * Pattern files hold one pattern per line (a trailing '\r' is kept: the
 * bytes are the pattern).  Errors: message on stderr, exit code 2 for usage,
 * 1 for library errors (mag_status_string + mag_last_error).
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "mag.h"

static int usage(void) {
  fprintf(stderr,
          "usage: mag_cli search --patterns FILE --text FILE [--variant V] [--q N] [--k N]\n"
          "                      [--sigma-prime N] [--mapping M|lowbits:L] [--count]\n"
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

static int cmd_search(int argc, char** argv) {
  const char* pf = arg(argc, argv, "--patterns");
  const char* tf = arg(argc, argv, "--text");
  if (!pf || !tf) return usage();
  mag_options o;
  mag_options_init(&o);
  const char* v = arg(argc, argv, "--variant");
  if (v) {
    if (!strcmp(v, "mag")) o.variant = MAG_VARIANT_MAG;
    else if (!strcmp(v, "smag")) o.variant = MAG_VARIANT_SMAG;
    else if (!strcmp(v, "shiftor_og")) o.variant = MAG_VARIANT_SHIFTOR_OG;
    else if (!strcmp(v, "naive")) o.variant = MAG_VARIANT_NAIVE;
    else if (!strcmp(v, "ac")) o.variant = MAG_VARIANT_AC;
    else return usage();
  }
  const char* x;
  if ((x = arg(argc, argv, "--q"))) o.q = atoi(x);
  if ((x = arg(argc, argv, "--k"))) o.k = atoi(x);
  if ((x = arg(argc, argv, "--sigma-prime"))) o.sigma_prime = atoi(x);
  if ((x = arg(argc, argv, "--mapping"))) {
    if (!strcmp(x, "identity")) o.mapping = MAG_MAPPING_IDENTITY;
    else if (!strcmp(x, "freq")) o.mapping = MAG_MAPPING_FREQUENCY;
    else if (!strcmp(x, "balance")) o.mapping = MAG_MAPPING_BALANCED;
    else if (!strncmp(x, "lowbits:", 8)) {
      o.mapping = MAG_MAPPING_LOWBITS;
      o.lowbits = atoi(x + 8);
    } else {
      return usage();
    }
  }
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
  if (!strcmp(argv[1], "tune")) return cmd_tune(argc, argv);
  if (!strcmp(argv[1], "gen")) return cmd_gen(argc, argv);
  return usage();
}
