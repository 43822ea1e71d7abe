"""Repeat a config's search and report any mismatch against the reference AC
(positions missing / extra, their slice index) — race hunting."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_1405_5483_b200 as mag
from paper_1405_5483_b200 import workloads
from pyoracle import Ref
cfg = int(sys.argv[1]); scale = float(sys.argv[2]); reps = int(sys.argv[3])
kw = {}
for kv in filter(None, (sys.argv[4] if len(sys.argv) > 4 else "").split(",")):
    k, v = kv.split("="); kw[k] = int(v) if v.lstrip("-").isdigit() else v
w = workloads.generate(cfg, scale)
want = Ref().ac(w.text, w.patterns, threads=8)
wk = set(zip(want[0].tolist(), want[1].tolist()))
for it in range(reps):
    e = mag.Engine(w.patterns, **kw)
    pl = e.plan()
    for mode in ("search", "prepared"):
        m = e.search(w.text) if mode == "search" else e.search_prepared(e.prepare(w.text))
        o, p = m.arrays()
        ok = np.array_equal(o, want[0]) and np.array_equal(p, want[1])
        if not ok:
            got = set(zip(o.tolist(), p.tolist()))
            miss = sorted(wk - got)[:20]; extra = sorted(got - wk)[:20]
            print(it, mode, "MISMATCH", len(o), len(want[0]), "missing", len(wk - got), miss[:8], "extra", len(got - wk), extra[:8], flush=True)
        else:
            print(it, mode, "ok", len(o), flush=True)
print(pl)
