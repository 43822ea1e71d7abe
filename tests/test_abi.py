"""CPU: the C-ABI library (libmag_b200.so) loads without a GPU, exports every
symbol include/*.h declares, and its host-side logic (validation, maps,
tuner, masks, sampling, error convention) matches the reference semantics.

No compute call is made here: engines are created with device=-2 (host
tables only), and a device engine without a GPU must fail loudly.
"""
import ctypes as C
import os
import re
import subprocess
import threading

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = []
    for h in ("mag.h", "mag_b200.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        names += re.findall(r"MAG_API\s+[^;(]*?\b(mag_\w+)\s*\(", src)
    return names


def test_every_declared_symbol_is_exported(mag):
    names = declared_symbols()
    assert len(names) == len(set(names)) and len(names) >= 33
    L = mag.lib()
    for n in names:
        assert hasattr(L, n), n
    assert sorted(names) == sorted(mag.EXPORTS)
    # default visibility, dynamic table (mag.h:16-20)
    out = subprocess.run(["nm", "-D", "--defined-only", mag.LIB_PATH], capture_output=True, text=True).stdout
    dyn = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(names) <= dyn


def test_reference_enum_values(mag):
    # mag.h:26-52
    assert mag.MAG_OK == 0
    assert [mag.status_string(s) != "" for s in range(9)] == [True] * 9
    assert mag.VARIANTS == {"mag": 0, "smag": 1, "shiftor_og": 2, "naive": 3, "ac": 4}
    assert mag.MAPPINGS["auto"] == -1 and mag.MAPPINGS["identity"] == 0 and mag.MAPPINGS["lowbits"] == 3
    assert mag.version().startswith("mag-b200")


def host_engine(mag, pats, **kw):
    return mag.Engine(pats, device=-2, **kw)


def test_validation_errors(mag):
    # core.cpp:8-12, qgram.cpp:9-19, alphabet_map.cpp:37-40, superimpose.cpp:12-20
    cases = [
        ([], {}, 3),                                   # EMPTY_PATTERN_SET
        ([b"abc", b""], {}, 4),                        # EMPTY_PATTERN
        ([b"abc"], {"variant": "naive"}, 5),           # oracles are not GPU variants
        ([b"abc"], {"variant": "ac"}, 5),
        ([b"abcd"], {"q": 9, "mapping": "identity"}, 5),  # q > kMaxQ exact grams
        ([b"abcd"], {"q": 3, "k": 0}, 5),              # m < 2q-1 for MAG
        ([b"abcdefgh"], {"q": 2, "k": 9}, 5),          # k beyond m'
        ([b"abcd"], {"mapping": "freq", "sigma_prime": 1}, 5),
        ([b"abcd"], {"mapping": "lowbits", "lowbits": 9}, 5),
    ]
    for pats, kw, status in cases:
        with pytest.raises(mag.MagError) as ei:
            host_engine(mag, pats, **kw)
        assert ei.value.status == status, (pats, kw, str(ei.value))
        assert mag.lib().mag_last_error().decode() != ""


def test_last_error_is_per_thread(mag):
    with pytest.raises(mag.MagError):
        host_engine(mag, [])
    mine = mag.lib().mag_last_error().decode()
    seen = {}

    def other():
        seen["start"] = mag.lib().mag_last_error()
        try:
            host_engine(mag, [b""])
        except mag.MagError:
            pass
        seen["end"] = mag.lib().mag_last_error().decode()

    t = threading.Thread(target=other)
    t.start()
    t.join()
    assert seen["start"] is not None and seen["start"].decode() == ""  # never NULL (mag.h:156-157)
    assert "empty" in seen["end"] and mag.lib().mag_last_error().decode() == mine


def test_info_and_alphabet_follow_reference(mag, ref):
    rng = np.random.default_rng(2)
    text = (rng.integers(0, 4, 4000) + 65).astype(np.uint8)
    pats = [text[s:s + 16].tobytes() for s in range(0, 400, 40)] + [b"ACGTACGTACGTACGTAC"]
    for mapping, strategy in (("identity", 0), ("freq", 1), ("balance", 2), ("lowbits", 3)):
        kw = {"mapping": mapping, "q": 2, "k": 1}
        if mapping in ("freq", "balance"):
            kw["sigma_prime"] = 3
        if mapping == "lowbits":
            kw["lowbits"] = 2
        e = host_engine(mag, pats, **kw)
        info = e.info()
        assert (info.r, info.m, info.q, info.k, info.mapping) == (len(pats), 16, 2, 1, strategy)
        table, sp = e.alphabet()
        assert (table, sp) == ref.alphabet_map(strategy, pats, kw.get("sigma_prime", 256 if strategy == 0 else 0),
                                               kw.get("lowbits", 0))
        assert info.sigma_prime == sp


def test_masks_equal_restated_machine(mag, port):
    """Exact-gram engines upload the reference machine's mask table
    (filter.hpp:27-31) bit for bit."""
    rng = np.random.default_rng(3)
    for it in range(24):
        sig = int(rng.choice([2, 4, 16]))
        text = (rng.integers(0, sig, 3000) + 97).astype(np.uint8)
        m = int(rng.integers(4, 30))
        pats = [text[s:s + m + int(rng.integers(0, 3))].tobytes() for s in rng.integers(0, 2900, int(rng.integers(1, 30)))]
        variant = ["mag", "smag", "shiftor_og"][it % 3]
        q = int(rng.integers(1, 4))
        if variant != "shiftor_og" and 2 * q - 1 > m:
            q = 1
        kmax = max(1, (m - q + 1) // q)
        k = 0 if variant == "shiftor_og" else int(rng.integers(1, kmax + 1))
        e = host_engine(mag, pats, variant=variant, q=q, k=k, mapping="balance", sigma_prime=sig)
        pl = e.plan()
        assert pl["gram_mode"] == 0
        table, sp = e.alphabet()
        P = port.params(variant={"mag": 0, "smag": 1, "shiftor_og": 2}[variant], gram_mode=0, q=pl["q"],
                        k=pl["k"], sigma_prime=sp, table=table)
        want, shape = port.masks(pats, P)
        assert (pl["m_prime"], pl["k"]) == (shape["m_prime"], shape["k"])
        assert np.array_equal(e.masks(shape["entries"]), want), (it, variant, q, k)


def test_hashed_masks_equal_restated_machine(mag, port):
    rng = np.random.default_rng(4)
    for it in range(12):
        text = (rng.integers(0, 4, 20000) + 65).astype(np.uint8)
        pats = [text[s:s + 32].tobytes() for s in rng.integers(0, 19000, int(rng.integers(1, 2000)))]
        e = host_engine(mag, pats, variant=["mag", "shiftor_og"][it % 2])
        pl = e.plan()
        if pl["verify_all"] or pl["gram_mode"] != 1:
            continue
        if pl["roll"]:
            from pyoracle import roll_bloom
            words = pl["table_bytes"] // 4
            bits = e.masks(32 * words) & np.uint64(1)
            got = np.packbits(bits.astype(np.uint8).reshape(-1, 32)[:, ::-1], axis=1).view(">u4").reshape(-1)
            assert np.array_equal(got.astype(np.uint32), roll_bloom(pats, pl["q"], words, pl["probes"]))
            continue
        P = port.params(variant=0 if it % 2 == 0 else 2, gram_mode=1, q=pl["q"], k=pl["k"],
                        table_bits=pl["table_bits"], word_bits=pl["k"] * pl["m_prime"], probes=pl["probes"],
                        blocks=pl["blocks"])
        want, shape = port.masks(pats, P)
        got = e.masks(shape["entries"])
        wb = pl["k"] * pl["m_prime"]
        keep = np.uint64((1 << wb) - 1) if wb < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
        assert np.array_equal(got & keep, want & keep), (it, pl)


def test_plans_fit_the_sm(mag):
    """Every automatic plan fits sm_100's 227 KB of shared memory and keeps
    q within what its gram mode supports."""
    rng = np.random.default_rng(5)
    for sig, r, m in ((4, 100, 16), (4, 10000, 32), (20, 1000, 16), (64, 100000, 32), (4, 100000, 12),
                      (2, 1, 1), (256, 7, 3), (4, 300000, 64)):
        pats = [(rng.integers(0, sig, m) + 33).astype(np.uint8).tobytes() for _ in range(r)]
        pl = host_engine(mag, pats).plan()
        assert pl["smem_bytes"] <= 232448, pl
        assert 1 <= pl["q"] <= (16 if pl["gram_mode"] == 1 else 8)
        assert pl["warps"] >= 1 and pl["tile_bytes"] > 0


def test_tune_matches_restatement(mag, port):
    for sigma, r, m, n in ((4, 100, 16, 1 << 24), (4, 10000, 32, 1 << 30), (20, 1000, 16, 1 << 28),
                           (64, 100000, 32, 1 << 29), (4, 100000, 12, 1 << 30)):
        a = mag.tune(sigma, r, m, n)
        b = port.tune(sigma, r, m, n)
        assert (a["q"], a["k"], a["sigma_prime"]) == (b["q"], b["k"], b["sigma_prime"])
        assert abs(a["predicted_p"] - b["predicted_p"]) < 1e-12


def test_sample_patterns_seeded(mag, port):
    corpus = bytes(range(256)) * 40
    got = mag.sample_patterns(corpus, 50, 12, 1234)
    offs = port.sample_offsets(len(corpus), 50, 12, 1234)
    assert got == [corpus[o:o + 12] for o in offs.tolist()]
    assert mag.sample_patterns(corpus, 50, 12, 1234) == got
    with pytest.raises(mag.MagError):
        mag.sample_patterns(b"abc", 1, 4, 0)  # length > corpus


def test_device_engine_without_gpu_fails_loudly(mag):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(mag.MagError) as ei:
        mag.Engine([b"ACGT"])
    assert ei.value.status == 8  # MAG_ERR_INTERNAL: no silent CPU fallback


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1405_5483_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".h", ".c")) or f == "Makefile":
                src = open(os.path.join(dirpath, f), errors="replace").read()
                for bad in (r"import\s+pyoracle", r"from\s+pyoracle", r"#include\s*\S*mag_oracle",
                            r"libmagref", r"libmagoracle", r"oracle/_ref"):
                    assert not re.search(bad, src), (f, bad)


def test_roll_warps_follow_the_built_kernels(mag):
    """More than 16 warps exist only for the 3-probe equal-length roll kernels
    (scan_roll.cu launch_roll_qhe); other plans clamp the request."""
    pats = [b"ACGTACGTAC", b"ACGTTTGTAC", b"TTGTACGTAC"]
    for H, w, want in ((3, 24, 24), (3, 20, 20), (2, 24, 16), (1, 20, 16), (3, 0, 16)):
        pl = mag.Engine(pats, scan_kernel="roll", probes=H, warps=w, device=-2).plan()
        assert pl["warps"] == want and pl["smem_bytes"] <= 232448, (H, w, pl)
    unequal = pats + [b"ACGTACGTACGTA"]
    assert mag.Engine(unequal, scan_kernel="roll", warps=24, device=-2).plan()["warps"] == 16


def test_roll_bloom_equals_restatement(mag):
    """Forced roll plans: the uploaded Bloom words equal the restated filter
    (oracle/pyoracle.py roll_bloom) for every template q."""
    from pyoracle import roll_bloom
    rng = np.random.default_rng(21)
    for m in (8, 12, 13, 16, 20, 24, 31, 32, 40):
        pats = [(rng.integers(0, 4, m + int(rng.integers(0, 3))) + 65).astype(np.uint8).tobytes()
                for _ in range(int(rng.integers(1, 500)))]
        for H in (2, 3):
            e = host_engine(mag, pats, scan_kernel="roll", probes=H)
            pl = e.plan()
            assert pl["roll"] == 1 and pl["variant"] == 2 and pl["probes"] == H
            assert pl["q"] == max(c for c in (8, 12, 16, 20, 24, 32) if c <= m)
            words = pl["table_bytes"] // 4
            bits = e.masks(32 * words) & np.uint64(1)
            got = np.packbits(bits.astype(np.uint8).reshape(-1, 32)[:, ::-1], axis=1).view(">u4").reshape(-1)
            assert np.array_equal(got.astype(np.uint32), roll_bloom(pats, pl["q"], words, H))
    with pytest.raises(mag.MagError):
        host_engine(mag, [b"abcdefg"], scan_kernel="roll")  # m < 8: no roll plan


def test_planner_picks_the_calibrated_kernel_per_config(mag):
    """The five BASELINE shapes (reduced text; plans depend on the pattern
    set only): aligned 16-byte samples for m = 32, 8-byte samples for m = 16,
    the dense rolling-hash scan for r = 100k, m = 12 (DESIGN.md kernels)."""
    from paper_1405_5483_b200 import workloads
    want = {1: ("direct", 8), 2: ("direct", 16), 3: ("direct", 8), 4: ("direct", 16), 5: ("roll", 12)}
    for cfg, (kernel, q) in want.items():
        w = workloads.generate(cfg, 1 / 256)
        pl = host_engine(mag, w.patterns).plan()
        assert pl[kernel] == 1 and pl["q"] == q, (cfg, pl)
        assert pl["smem_bytes"] <= 232448
