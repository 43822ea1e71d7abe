"""Random engine options against the reference AC: every engine that is
created must search correctly (a bad combination must be refused at creation
with BAD_CONFIG, never fail at launch)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import paper_1405_5483_b200 as mag
from pyoracle import Ref, as_pairs
ref = Ref()
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 7)
bad = refused = 0
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 120):
    m = int(rng.choice([8, 10, 12, 13, 16, 17, 24, 31, 32, 40]))
    sig = int(rng.choice([2, 4, 20, 64]))
    n = int(rng.choice([3000, 50000, 400000]))
    r = int(rng.choice([1, 30, 800, 6000]))
    eq = rng.random() < 0.5
    text = (rng.integers(0, sig, n) + 60).astype(np.uint8)
    pats = []
    for _ in range(r):
        L = m + (0 if eq else int(rng.integers(0, 5)))
        o = int(rng.integers(0, n - L))
        pats.append(text[o:o + L].tobytes() if rng.random() < 0.6 else (rng.integers(0, sig, L) + 60).astype(np.uint8).tobytes())
    kw = {}
    if rng.random() < 0.8: kw["scan_kernel"] = str(rng.choice(["auto", "direct", "staged", "roll", "pack2"]))
    if rng.random() < 0.5: kw["probes"] = int(rng.integers(1, 5))
    if rng.random() < 0.5: kw["warps"] = int(rng.choice([1, 4, 8, 15, 16, 20, 24, 32]))
    if rng.random() < 0.2: kw["stages"] = int(rng.integers(2, 5))
    if rng.random() < 0.2: kw["table_bits"] = int(rng.integers(10, 22))
    if rng.random() < 0.2: kw["histogram_sample"] = text[:1 << 16]
    if rng.random() < 0.15: kw["variant"] = "shiftor_og"
    try:
        e = mag.Engine(pats, **kw)
    except mag.MagError as ex:
        refused += 1
        assert ex.status == 5, (kw, ex)
        continue
    try:
        got = e.search(text).pairs()
        ok = got == as_pairs(*ref.ac(text, pats, threads=8))
    except mag.MagError as ex:
        ok = False
        print("  search error:", ex)
    bad += not ok
    kwp = {k: v for k, v in kw.items() if k != "histogram_sample"}
    if not ok:
        print(it, "FAIL", m, sig, n, r, eq, kwp, e.plan(), flush=True)
print("bad", bad, "refused", refused)
