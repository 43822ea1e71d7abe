"""GPU parity: the sm_100a search path (through the C ABI) against the
reference's own compiled oracles and the C restatement.

Bar: bit-exact (offset, pattern_index) sets; identical filter counters
(reads, candidates) to the restated reference machine at identical
(variant, q, k, sigma', map, w, gram mode).
"""
import numpy as np
import pytest

from pyoracle import as_pairs

pytestmark = pytest.mark.gpu


def gpu_pairs(engine, text):
    m = engine.search(text)
    return m.pairs(), m.metrics()


def rand_instance(rng, sig=None, n=None, r=None, m=None, unequal=True, copy_frac=0.5, base=97):
    sig = sig or int(rng.choice([2, 4, 16, 64, 200]))
    n = int(rng.integers(0, 20000)) if n is None else n
    r = r or int(rng.integers(1, 40))
    m = m or int(rng.integers(1, 40))
    text = (rng.integers(0, sig, n) + base).astype(np.uint8)
    pats = []
    for _ in range(r):
        L = m + (int(rng.integers(0, 5)) if unequal else 0)
        if n > L and rng.random() < copy_frac:
            s = int(rng.integers(0, n - L + 1))
            pats.append(text[s:s + L].tobytes())
        else:
            pats.append((rng.integers(0, sig, L) + base).astype(np.uint8).tobytes())
    return text, pats


def test_spec_examples(mag, ref):
    # SPEC.md:55-57, 65-66, 382, 516 (results as (offset, pattern_index))
    cases = [
        (b"xabbacy", [b"abba", b"bbac"], [(1, 0), (2, 1)]),
        (b"aaa", [b"aa"], [(0, 0), (1, 0)]),
        (b"abab", [b"zz"], []),
        (b"ushers", [b"he", b"she", b"his"], [(1, 1), (2, 0)]),
        (b"", [b"ab"], []),
        (b"zabbaz", [b"abba"], [(1, 0)]),
    ]
    for text, pats, want in cases:
        assert as_pairs(*ref.naive(text, pats)) == want
        for variant in ("mag", "smag", "shiftor_og"):
            e = mag.Engine(pats, variant=variant)
            got, _ = gpu_pairs(e, text)
            assert got == want, (text, pats, variant, e.plan())
        # the reference's own parameter path (exact grams, q = 1)
        e = mag.Engine(pats, q=1, k=1, mapping="identity")
        assert gpu_pairs(e, text)[0] == want


def test_random_auto_plans(mag, ref):
    rng = np.random.default_rng(11)
    for it in range(120):
        text, pats = rand_instance(rng)
        want = as_pairs(*ref.ac(text, pats))
        variant = ["mag", "smag", "shiftor_og"][it % 3]
        e = mag.Engine(pats, variant=variant)
        got, met = gpu_pairs(e, text)
        assert got == want, (it, variant, e.plan())


@pytest.mark.parametrize("mapping", ["identity", "freq", "balance", "lowbits"])
def test_reference_parameters_and_counters(mag, ref, port, mapping):
    """Exact-gram plans with explicit (q, k, sigma', map): same matches as the
    reference oracles, same filter reads/candidates as the restated machine."""
    rng = np.random.default_rng(hash(mapping) & 0xffff)
    for it in range(40):
        sig = int(rng.choice([2, 4, 16, 64]))
        text, pats = rand_instance(rng, sig=sig, m=int(rng.integers(2, 33)))
        mm = min(len(p) for p in pats)
        variant = ["mag", "smag", "shiftor_og"][it % 3]
        if variant == "shiftor_og":
            qmax = min(8, mm)
        else:
            qmax = min(8, (mm + 1) // 2)
        q = int(rng.integers(1, qmax + 1))
        kk = 0 if variant == "shiftor_og" else int(rng.integers(1, (mm - q + 1) // q + 1))
        kw = dict(variant=variant, q=q, k=kk, mapping=mapping)
        if mapping == "lowbits":
            kw["lowbits"] = int(rng.integers(1, 9))
            if (1 << kw["lowbits"]) ** q > (1 << 24):
                continue
        elif mapping in ("freq", "balance"):
            kw["sigma_prime"] = int(rng.integers(2, 17))
            if kw["sigma_prime"] ** q > (1 << 24):
                continue
        elif 256 ** q > (1 << 24):
            continue
        e = mag.Engine(pats, **kw)
        got, met = gpu_pairs(e, text)
        want = as_pairs(*ref.ac(text, pats))
        assert got == want, (it, kw)
        info = e.info()
        table, sp = e.alphabet()
        P = port.params(variant={"mag": 0, "smag": 1, "shiftor_og": 2}[variant], gram_mode=0, q=info.q,
                        k=info.k, sigma_prime=sp, table=table)
        o, p, reads, cands = port.search(text, pats, P)
        assert as_pairs(o, p) == want
        assert (met.filter_reads, met.candidates) == (reads, cands), (it, kw)


def test_hashed_counters_match_port(mag, ref, port):
    rng = np.random.default_rng(5)
    for it in range(40):
        text, pats = rand_instance(rng, sig=4, n=int(rng.integers(1000, 60000)), r=int(rng.integers(1, 300)),
                                   m=int(rng.integers(4, 40)), base=65)
        variant = ["mag", "shiftor_og"][it % 2]
        e = mag.Engine(pats, variant=variant)
        pl = e.plan()
        got, met = gpu_pairs(e, text)
        assert got == as_pairs(*ref.ac(text, pats))
        if pl["verify_all"]:
            assert met.candidates == met.filter_reads
            continue
        if pl["roll"]:
            from pyoracle import roll_candidates
            assert met.filter_reads == max(0, text.size - pl["q"] + 1)
            assert met.candidates == roll_candidates(text, pats, pl["q"], pl["table_bytes"] // 4, pl["probes"])
            continue
        assert not pl["pack2"], pl  # never planned automatically
        P = port.params(variant=0 if pl["variant"] == 0 else 2, gram_mode=1, q=pl["q"], k=pl["k"],
                        table_bits=pl["table_bits"], word_bits=pl["k"] * pl["m_prime"], probes=pl["probes"],
                        blocks=pl["blocks"])
        o, p, reads, cands = port.search(text, pats, P)
        assert (met.filter_reads, met.candidates) == (reads, cands), (it, pl)


def test_edge_cases(mag, ref):
    cases = []
    cases.append((b"", [b"a"]))                       # empty text
    cases.append((b"abc", [b"abcd"]))                 # n < m
    cases.append((b"ab", [b"abcdefgh"]))              # n < q for most plans
    cases.append((b"abcabc", [b"abc", b"abc", b"bc"]))  # duplicates keep both ids
    cases.append((b"xyzxyz", [b"xyz", b"yzxyz"]))     # match at 0 and at n-m
    cases.append((b"a" * 5000, [b"a", b"aa", b"aaa"]))  # every position, every pattern
    cases.append((b"a" * 70000, [b"aaaa"] * 7))       # dense + duplicates: output overflow path
    for text, pats in cases:
        want = as_pairs(*ref.naive(text, pats))
        for variant in ("mag", "smag", "shiftor_og"):
            e = mag.Engine(pats, variant=variant)
            assert gpu_pairs(e, text)[0] == want, (text[:20], pats, variant)


def test_tile_boundaries(mag, ref):
    """Texts whose occurrences straddle tile and warp-slice boundaries."""
    rng = np.random.default_rng(7)
    for tile in (256, 1024, 8192):
        for it in range(6):
            n = tile * int(rng.integers(1, 6)) + int(rng.integers(-40, 40))
            text, pats = rand_instance(rng, sig=4, n=max(n, 0), r=20, m=int(rng.integers(5, 30)), base=65)
            # plant occurrences right around every tile boundary
            text = text.copy()
            for b in range(tile, text.size, tile):
                p = pats[int(rng.integers(0, len(pats)))]
                s = max(0, b - int(rng.integers(0, len(p))))
                if s + len(p) <= text.size:
                    text[s:s + len(p)] = np.frombuffer(p, dtype=np.uint8)
            want = as_pairs(*ref.ac(text, pats))
            for variant in ("mag", "shiftor_og"):
                e = mag.Engine(pats, variant=variant, tile_bytes=tile, warps=int(rng.choice([1, 4, 16])))
                assert gpu_pairs(e, text)[0] == want, (tile, it, variant, e.plan())


def test_long_patterns_beyond_halo(mag, ref):
    rng = np.random.default_rng(9)
    text = (rng.integers(0, 4, 50000) + 65).astype(np.uint8)
    pats = [text[s:s + L].tobytes() for s, L in ((100, 2000), (9000, 1500), (30000, 3000), (49000, 1000))]
    pats.append(text[8000:8050].tobytes())
    want = as_pairs(*ref.ac(text, pats))
    for variant in ("mag", "shiftor_og"):
        assert gpu_pairs(mag.Engine(pats, variant=variant), text)[0] == want


def test_prepared_async_and_device_text(mag, ref):
    import torch
    rng = np.random.default_rng(3)
    text, pats = rand_instance(rng, sig=4, n=300000, r=50, m=20, base=65)
    want = as_pairs(*ref.ac(text, pats))
    e = mag.Engine(pats)
    p = e.prepare(text)
    assert e.search_prepared(p).pairs() == want
    d = torch.from_numpy(text).cuda()
    pd = e.prepare_device(d.data_ptr(), d.numel(), keep=d)
    s = torch.cuda.Stream()
    ms = [e.search_prepared_async(pd, s.cuda_stream) for _ in range(3)]
    for m in ms:
        assert m.pairs() == want
    # misaligned device pointer -> internal aligned copy
    pd2 = e.prepare_device(d.data_ptr() + 3, d.numel() - 3, keep=d)
    want2 = as_pairs(*ref.ac(text[3:], pats))
    assert e.search_prepared(pd2).pairs() == want2


def test_smag_codes_equal_reference_encode_text(mag, ref):
    rng = np.random.default_rng(4)
    text, pats = rand_instance(rng, sig=4, n=10000, r=10, m=16, base=65)
    for q in (1, 3, 5, 8):
        e = mag.Engine(pats, variant="smag", q=q, k=1, mapping="balance", sigma_prime=4)
        p = e.prepare(text)
        want = ref.encode_text(2, pats, 4, 0, q, text)
        assert np.array_equal(p.codes(text.size // q), want)


@pytest.mark.parametrize("cfg,scale", [(1, 1.0), (2, 1 / 64), (3, 1 / 32), (4, 1 / 64), (5, 1 / 64)])
def test_baseline_configs_reduced(mag, ref, cfg, scale):
    from paper_1405_5483_b200 import workloads
    w = workloads.generate(cfg, scale)
    want = ref.ac(w.text, w.patterns, threads=8)
    e = mag.Engine(w.patterns)
    m = e.search(w.text)
    offs, pids = m.arrays()
    assert np.array_equal(offs, want[0]) and np.array_equal(pids, want[1]), (cfg, e.plan())
    pl, n = e.plan(), w.text.size
    want_reads = n if pl["verify_all"] else (n - pl["q"] + 1 if pl["variant"] == 2 else (n // pl["q"]) // pl["k"])
    assert m.metrics().filter_reads == want_reads


def _golden():
    import os
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def _unpack(g, key):
    b, l = g[f"{key}_pat"], g[f"{key}_len"]
    out, o = [], 0
    for n in l.tolist():
        out.append(b[o:o + n].tobytes())
        o += n
    return out


def test_golden_fixtures(mag):
    """CUDA path vs the reference's own outputs (tests/golden, generated by
    the compiled reference; no /root/reference needed on the GPU box)."""
    g = _golden()
    keys = [f"spec_{i}" for i in range(6)] + [f"inst_{i}" for i in range(int(g["inst_count"][0]))]
    for key in keys:
        text, pats = g[f"{key}_text"], _unpack(g, key)
        want = as_pairs(g[f"{key}_off"], g[f"{key}_pid"])
        for variant in ("mag", "smag", "shiftor_og"):
            e = mag.Engine(pats, variant=variant)
            assert gpu_pairs(e, text)[0] == want, (key, variant, e.plan())


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_golden_configs(mag, cfg):
    from paper_1405_5483_b200 import workloads
    g = _golden()
    w = workloads.generate(cfg, float(g[f"cfg_{cfg}_scale"][0]))
    offs, pids = mag.Engine(w.patterns).search(w.text).arrays()
    assert np.array_equal(offs, g[f"cfg_{cfg}_off"]) and np.array_equal(pids, g[f"cfg_{cfg}_pid"])


def test_sharded_spans(mag, ref):
    """shard.py over device-resident text: every rank's span searched in
    place, clipped and concatenated in rank order == the whole-text result."""
    import torch
    from paper_1405_5483_b200 import shard
    rng = np.random.default_rng(12)
    text, pats = rand_instance(rng, sig=4, n=1 << 20, r=300, m=24, base=65)
    want = ref.ac(text, pats)
    e = mag.Engine(pats)
    d = torch.from_numpy(text).cuda()
    run = shard.engine_span_search(e, d.data_ptr(), keep=d)
    maxlen = max(len(p) for p in pats)
    for world in (2, 3, 8):
        b = shard.ownership(text.size, world)
        parts = []
        for g in range(world):
            lo, hi = shard.read_span(text.size, b, g, maxlen)
            o, p = run(lo, hi) if hi > lo else (np.zeros(0, np.uint64), np.zeros(0, np.uint32))
            parts.append(shard.clip(o, p, lo, b[g + 1]))
        offs = np.concatenate([x[0] for x in parts])
        pids = np.concatenate([x[1] for x in parts])
        assert np.array_equal(offs, want[0]) and np.array_equal(pids, want[1]), world


def _full_digests():
    import json
    import os
    p = os.path.join(os.path.dirname(__file__), "golden", "full_digests.json")
    with open(p) as f:
        return json.load(f)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_full_configs(mag, cfg):
    """BASELINE.json configs at FULL size: the GPU match set's count and
    sha256 equal the reference Aho–Corasick's (tests/golden/full_digests.json,
    made by tests/golden/make_full_digests.py from oracle/_ref)."""
    import sys
    import os
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from make_full_digests import input_digest, match_digest
    from paper_1405_5483_b200 import workloads
    want = _full_digests()[str(cfg)]
    w = workloads.generate(cfg, 1.0)
    assert input_digest(w) == {k: want[k] for k in ("text_sha256", "patterns_sha256")}
    e = mag.Engine(w.patterns)
    m = e.search(w.text)
    offs, pids = m.arrays()
    assert offs.size == want["matches"], (cfg, e.plan())
    assert match_digest(offs, pids) == want["matches_sha256"], (cfg, e.plan())


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_full_configs_reference_params(mag, port, cfg):
    """The same full-size digests through the reference-default exact-code
    plan: the restated tuner's q/k (tuner.hpp:38-66), the balanced map over
    the pattern histogram (alphabet_map.cpp:90-102), m' = min(L/k, w/k)
    (filter.hpp:27-31) -- the staged Shift-Or kernel with m' = 3 (cfg2), 2
    (cfg3), 7 (cfg4).  The plan's q/k equal mag_tune's."""
    import sys
    import os
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from make_full_digests import match_digest
    from paper_1405_5483_b200 import workloads
    want = _full_digests()[str(cfg)]
    w = workloads.generate(cfg, 1.0)
    e = mag.Engine(w.patterns, gram_mode=mag.GRAM_EXACT)
    pl, info = e.plan(), e.info()
    sigma = len(set(b"".join(w.patterns)))
    tu = port.tune(sigma, len(w.patterns), w.meta["m"])
    assert (pl["gram_mode"], info.q, info.k, info.mapping) == (0, tu["q"], tu["k"], mag.MAPPING_BALANCED)
    assert pl["m_prime"] == min((w.meta["m"] - info.q + 1) // info.q // info.k, 64 // info.k)
    offs, pids = e.search(w.text).arrays()
    assert offs.size == want["matches"], (cfg, pl)
    assert match_digest(offs, pids) == want["matches_sha256"], (cfg, pl)


@pytest.mark.parametrize("cfg,q,k,mp", [(1, 5, 1, 2), (3, 3, 1, 4), (5, 6, 1, 1)])
def test_full_configs_analytic_seed_params(mag, cfg, q, k, mp):
    """SURVEY.md §8a's other reading of the (bodiless) tuner: the analytic
    seeds q = round(log_sigma'(rm)) and k without the joint grid
    (tuner.hpp:44-56), which differ from the restated joint choice on cfg1
    (q = 5, m' = 2), cfg3 (q = 3, m' = 4) and cfg5 (q = 6).  Exact codes,
    balanced map; the same full-size digests."""
    import sys
    import os
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from make_full_digests import match_digest
    from paper_1405_5483_b200 import workloads
    want = _full_digests()[str(cfg)]
    w = workloads.generate(cfg, 1.0)
    e = mag.Engine(w.patterns, gram_mode=mag.GRAM_EXACT, q=q, k=k)
    pl, info = e.plan(), e.info()
    assert (pl["gram_mode"], info.q, info.k, pl["m_prime"], info.mapping) == (0, q, k, mp, mag.MAPPING_BALANCED)
    offs, pids = e.search(w.text).arrays()
    assert offs.size == want["matches"], (cfg, pl)
    assert match_digest(offs, pids) == want["matches_sha256"], (cfg, pl)


@pytest.mark.parametrize("H", [2, 3])
def test_roll_kernel(mag, ref, H):
    """The dense rolling-hash scan (forced): every template q, unequal and
    duplicate patterns, texts of every length class around the 2 KiB step
    and 32 KiB slice, dense planted occurrences, patterns longer than the
    staged halo (global compares); candidate counter == the restated filter."""
    from pyoracle import roll_candidates
    rng = np.random.default_rng(40 + H)
    sizes = [0, 7, 8, 15, 16, 17, 2047, 2048, 2049, 2063, 32768 + 13, 100000, 300001]
    for it, n in enumerate(sizes):
        m = int(rng.choice([8, 9, 12, 15, 16, 20, 24, 32, 33, 48]))
        sig = int(rng.choice([2, 4, 20, 64]))
        text = (rng.integers(0, sig, n) + 65).astype(np.uint8)
        r = int(rng.integers(1, 300))
        pats = []
        for _ in range(r):
            L = m + int(rng.integers(0, 4))
            if n > L and rng.random() < 0.6:
                s0 = int(rng.integers(0, n - L + 1))
                pats.append(text[s0:s0 + L].tobytes())
            else:
                pats.append((rng.integers(0, sig, L) + 65).astype(np.uint8).tobytes())
        if it % 3 == 0 and n > 400:
            pats.append(text[n - 300:n].tobytes())   # longer than the halo, ends at n
            pats.append(pats[0])                     # duplicate pattern id
        text = text.copy()
        for _ in range(n // 50):                      # dense plants
            p = pats[int(rng.integers(0, len(pats)))]
            if len(p) < n:
                s0 = int(rng.integers(0, n - len(p) + 1))
                text[s0:s0 + len(p)] = np.frombuffer(p, dtype=np.uint8)
        e = mag.Engine(pats, scan_kernel="roll", probes=H)
        pl = e.plan()
        assert pl["roll"] == 1
        try:
            got, met = gpu_pairs(e, text)
        except mag.MagError as ex:
            raise AssertionError(f"n={n} m={m} sig={sig} r={len(pats)} plan={pl}: {ex}")
        assert got == as_pairs(*ref.ac(text, pats)), (n, m, sig, pl)
        assert met.candidates == roll_candidates(text, pats, pl["q"], pl["table_bytes"] // 4, H), (n, m)
        # misaligned device text takes the aligned-copy path
        if n > 64:
            import torch
            d = torch.from_numpy(text).cuda()
            pd = e.prepare_device(d.data_ptr() + 5, n - 5, keep=d)
            assert e.search_prepared(pd).pairs() == as_pairs(*ref.ac(text[5:], pats))


@pytest.mark.parametrize("m,H,warps", [(8, 1, 0), (9, 2, 0), (10, 3, 0), (12, 3, 0), (12, 3, 20), (11, 3, 24),
                                       (10, 2, 24)])  # 2-probe kernels are built for <= 16 warps: the plan clamps
def test_roll_kernel_equal_short_sets(mag, ref, m, H, warps):
    """The roll kernel's path for equal-length sets of m <= 12 bytes (cfg5's
    shape): 1 KiB steps, two-entry verification sectors, verification
    pipelined across steps.  Covers texts around the step and slice sizes,
    q < m (starts past n - m), dense steps (> 64 and > 128 candidates: the
    rank-search expansion), duplicate patterns (two matches in one sector)
    and overflowing home sectors (>= 3 identical patterns: the walk)."""
    from pyoracle import roll_candidates
    rng = np.random.default_rng(100 * m + H)
    sizes = [0, m - 1, m, 1023, 1024, 1025, 1024 + m, 32768 + 5, 70001, 250000]
    for it, n in enumerate(sizes):
        sig = [2, 4, 4, 20][it % 4]
        text = (rng.integers(0, sig, n) + 65).astype(np.uint8)
        r = int(rng.integers(1, 400))
        pats = []
        for _ in range(r):
            if n > m and rng.random() < 0.6:
                s0 = int(rng.integers(0, n - m + 1))
                pats.append(text[s0:s0 + m].tobytes())
            else:
                pats.append((rng.integers(0, sig, m) + 65).astype(np.uint8).tobytes())
        pats += [pats[0]] * 4  # five identical patterns: their home sector overflows
        if n >= m:
            pats.append(text[n - m:n].tobytes())  # ends at n
        text = text.copy()
        if it % 2 == 1 and n > 4096:  # a dense stretch: every position of 3 KiB starts a match
            text[1000:4072] = np.frombuffer(pats[0], dtype=np.uint8)[0]
            pats.append(bytes([pats[0][0]]) * m)
        e = mag.Engine(pats, scan_kernel="roll", probes=H, warps=warps)
        pl = e.plan()
        assert pl["roll"] == 1 and pl["tile_bytes"] == 1024, pl
        got, met = gpu_pairs(e, text)
        assert got == as_pairs(*ref.ac(text, pats)), (n, m, sig, pl)
        assert met.candidates == roll_candidates(text, pats, pl["q"], pl["table_bytes"] // 4, H), (n, m)


def test_concurrent_searches_one_engine(mag, ref):
    """An engine is immutable and searches on it may run concurrently
    (engine.hpp:55-56): host threads searching different texts through one
    engine (per-search pooled workspaces) all get their own exact results."""
    import threading
    rng = np.random.default_rng(31)
    base = (rng.integers(0, 4, 400000) + 65).astype(np.uint8)
    pats = [base[s:s + 24].tobytes() for s in rng.integers(0, base.size - 24, 200)]
    texts = [np.roll(base, 7919 * i).copy() for i in range(6)]
    want = [as_pairs(*ref.ac(t, pats)) for t in texts]
    for kernel in ("auto", "roll", "staged"):
        e = mag.Engine(pats, scan_kernel=kernel)
        got = [None] * len(texts)
        errs = []

        def run(i):
            try:
                for _ in range(3):
                    got[i] = e.search(texts[i]).pairs()
            except Exception as ex:  # pragma: no cover - surfaced below
                errs.append(ex)

        th = [threading.Thread(target=run, args=(i,)) for i in range(len(texts))]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errs, errs
        assert got == want, kernel


@pytest.mark.parametrize("q,probes", [(8, 1), (16, 1), (8, 3)])
def test_direct_kernel(mag, ref, port, q, probes):
    """The aligned-sample kernel (forced), both sample widths, single- and
    multi-probe tables: texts of every length class around its step (odd
    8-byte sample counts included), m = 2q-1 (the shortest admissible) up to
    patterns longer than any staged halo, duplicates, dense plants, misaligned
    device text; the candidate counter equals the restated hashed machine's."""
    rng = np.random.default_rng(50 + q)
    step = 128 * q
    sizes = [0, 5, q, 2 * q - 1, step - 8, step, step + 8, step + 24, 3 * step + 8, 2048 * q + 40, 250_000]
    for it, n in enumerate(sizes):
        m = int(rng.choice([2 * q - 1, 2 * q, 3 * q, 64]))
        sig = int(rng.choice([2, 4, 20]))
        text = (rng.integers(0, sig, n) + 65).astype(np.uint8)
        pats = []
        for _ in range(int(rng.integers(1, 200))):
            L = m + int(rng.integers(0, 3))
            if n > L and rng.random() < 0.6:
                s0 = int(rng.integers(0, n - L + 1))
                pats.append(text[s0:s0 + L].tobytes())
            else:
                pats.append((rng.integers(0, sig, L) + 65).astype(np.uint8).tobytes())
        if n > 2000 and it % 2:
            pats.append(text[n - 1500:n].tobytes())
            pats.append(pats[0])
        text = text.copy()
        for _ in range(n // 64):
            p = pats[int(rng.integers(0, len(pats)))]
            if len(p) < n:
                s0 = int(rng.integers(0, n - len(p) + 1))
                text[s0:s0 + len(p)] = np.frombuffer(p, dtype=np.uint8)
        e = mag.Engine(pats, scan_kernel="direct", q=q, gram_mode=mag.GRAM_HASHED, probes=probes)
        pl = e.plan()
        assert pl["direct"] == 1 and pl["q"] == q and pl["probes"] == probes, pl
        got, met = gpu_pairs(e, text)
        assert got == as_pairs(*ref.ac(text, pats)), (n, m, sig, pl)
        P = port.params(variant=0, gram_mode=1, q=q, k=1, table_bits=pl["table_bits"], word_bits=1,
                        probes=pl["probes"], blocks=pl["blocks"])
        _, _, reads, cands = port.search(text, pats, P)
        assert (met.filter_reads, met.candidates) == (reads, cands), (n, m, pl)
        if n > 64:
            import torch
            d = torch.from_numpy(text).cuda()
            pd = e.prepare_device(d.data_ptr() + 3, n - 3, keep=d)
            assert e.search_prepared(pd).pairs() == as_pairs(*ref.ac(text[3:], pats))


def _boundary_patterns(rng, text, bounds, lengths):
    """Patterns copied from the text so that their occurrences straddle every
    boundary in `bounds` (start = b - x for x from 1 to len - 1)."""
    pats = []
    for b in bounds:
        for L in lengths:
            for x in (1, 17, L // 2, L - 1, int(rng.integers(1, L))):
                s0 = b - x
                if 0 <= s0 and s0 + L <= text.size:
                    pats.append(text[s0:s0 + L].tobytes())
    return pats


@pytest.mark.parametrize("kernel", ["direct", "staged", "roll"])
def test_mag_search_copy_chunk_boundaries(mag, ref, kernel):
    """mag_search (pinned-copy pipeline) on a 200 MiB text (copy chunks of
    64 MiB): occurrences of 0.6-4 KiB patterns straddle every copy-chunk
    boundary, the workspace is pre-dirtied by a search of a different text,
    and the result equals the reference Aho-Corasick (oracles.cpp:78-95).
    Round 1 released a slice once its staging halo had arrived, not its
    longest pattern's reach (host_engine.cpp mag_search)."""
    rng = np.random.default_rng(77)
    n = 200 << 20
    text = (rng.integers(0, 4, n, dtype=np.uint8) + 65).astype(np.uint8)
    chunk = 64 << 20
    bounds = list(range(chunk, n, chunk))
    if kernel == "roll":
        pats = _boundary_patterns(rng, text, bounds, [600, 700])
        pats += [(rng.integers(0, 4, 12) + 65).astype(np.uint8).tobytes() for _ in range(300)]
        pats += [text[s:s + 12].tobytes() for s in rng.integers(0, n - 12, 300)]
    else:
        pats = _boundary_patterns(rng, text, bounds, [1536, 2500, 4096])
        pats += [text[s:s + 1600].tobytes() for s in rng.integers(0, n - 1600, 20)]
    e = mag.Engine(pats, scan_kernel=kernel)
    pl = e.plan()
    assert (pl["direct"], pl["roll"]) == {"direct": (1, 0), "staged": (0, 0), "roll": (0, 1)}[kernel], pl
    other = (rng.integers(0, 4, n, dtype=np.uint8) + 65).astype(np.uint8)
    e.search(other).close()  # leaves stale text in the workspace's device buffer
    got = e.search(text).arrays()
    want = ref.ac(text, pats, threads=8)
    assert got[0].size == want[0].size, (kernel, got[0].size, want[0].size, pl)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]), (kernel, pl)


@pytest.mark.parametrize("q", [8, 16])
def test_text_beyond_2p32_samples(mag, q):
    """The direct kernel past 2^32 samples (W = 8: a 32 GiB text; W = 16:
    64 GiB) in device memory: random 64-byte patterns planted before, at and
    after the 2^32-sample offset are found exactly there (the sample cursor
    and offsets are 64-bit; random 64-mers occur by chance with p ~ 4^-64)."""
    import torch
    free, _ = torch.cuda.mem_get_info()
    n = (q << 32) + (3 << 20)
    if free < n + (8 << 30):
        pytest.skip(f"needs {n >> 30} GiB of free device memory")
    rng = np.random.default_rng(64 + q)
    pats = [(rng.integers(0, 4, 64) + 65).astype(np.uint8).tobytes() for _ in range(8)]
    d = torch.randint(0, 4, (n,), dtype=torch.uint8, device="cuda")
    d.add_(65)
    edge = q << 32
    # non-overlapping plants (a later plant would overwrite an earlier one)
    offs = [5, edge - 4096, edge - 100, edge - 30, edge + 40, edge + 8 * 12345 + 3, n - 200, n - 64]
    want = []
    for i, o in enumerate(offs):
        p = i % len(pats)
        d[o:o + 64] = torch.frombuffer(bytearray(pats[p]), dtype=torch.uint8).cuda()
        want.append((o, p))
    e = mag.Engine(pats, scan_kernel="direct", q=q, gram_mode=mag.GRAM_HASHED)
    assert e.plan()["direct"] == 1 and e.plan()["q"] == q
    prep = e.prepare_device(d.data_ptr(), n, keep=d)
    got = e.search_prepared(prep).pairs()
    assert got == sorted(want), (got, sorted(want))
    del prep, d
    torch.cuda.empty_cache()


@pytest.mark.parametrize("alphabet", [b"ACGT", b"acgt", b"AT", b"xyz"])
def test_pack2_kernel(mag, ref, alphabet):
    """The dense 2-bit exact-code scan (forced): texts of every length class
    around its 2 KiB step and 32 KiB slice, pattern lengths 10..40 (level-2
    key of min(m, 16) symbols; longer ones finish in global memory),
    duplicate patterns, dense plants, text bytes outside the pattern alphabet
    (they collide in the 2-bit map), misaligned device text; the candidate
    counter equals the restated level-1 filter."""
    from pyoracle import pack2_candidates
    rng = np.random.default_rng(90 + len(alphabet))
    al = np.frombuffer(alphabet, dtype=np.uint8)
    sizes = [0, 9, 10, 11, 2047, 2048, 2049, 2063, 32768 + 13, 100000, 300001]
    for it, n in enumerate(sizes):
        m = int(rng.choice([10, 11, 12, 15, 16, 17, 24, 40]))
        text = al[rng.integers(0, al.size, n)]
        if it % 2 and n > 100:  # bytes outside the pattern alphabet
            text = text.copy()
            text[rng.integers(0, n, n // 50)] = ord("N")
        r = int(rng.integers(1, 400))
        pats = []
        for _ in range(r):
            L = m + int(rng.integers(0, 4))
            if n > L and rng.random() < 0.6:
                s0 = int(rng.integers(0, n - L + 1))
                cand = text[s0:s0 + L]
                if np.isin(cand, al).all():
                    pats.append(cand.tobytes())
                    continue
            pats.append(al[rng.integers(0, al.size, L)].tobytes())
        pats.append(pats[0])  # duplicate pattern id
        text = text.copy()
        for _ in range(n // 40):
            p = pats[int(rng.integers(0, len(pats)))]
            if len(p) < n:
                s0 = int(rng.integers(0, n - len(p) + 1))
                text[s0:s0 + len(p)] = np.frombuffer(p, dtype=np.uint8)
        e = mag.Engine(pats, scan_kernel="pack2")
        pl = e.plan()
        assert pl["pack2"] == 1, pl
        got, met = gpu_pairs(e, text)
        assert got == as_pairs(*ref.ac(text, pats)), (n, m, pl)
        shift = next(s for s in range(7) if len({(c >> s) & 3 for c in set(b"".join(pats))}) == len(set(b"".join(pats))))
        assert met.filter_reads == max(0, n - pl["q"] + 1)
        assert met.candidates == pack2_candidates(text, pats, pl["q"], shift), (n, m)
        if n > 64:
            import torch
            d = torch.from_numpy(text).cuda()
            pd = e.prepare_device(d.data_ptr() + 5, n - 5, keep=d)
            assert e.search_prepared(pd).pairs() == as_pairs(*ref.ac(text[5:], pats))
