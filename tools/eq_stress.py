import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import numpy as np
import paper_1405_5483_b200 as mag
from pyoracle import Ref, as_pairs, roll_candidates
ref = Ref()
rng = np.random.default_rng(2025)
bad = 0
for it in range(60):
    m = int(rng.integers(8, 13))
    sig = int(rng.choice([2, 3, 4, 20, 200]))
    n = int(rng.choice([500, 5000, 40000, 300000, 2000000]))
    r = int(rng.choice([1, 7, 200, 5000, 40000]))
    text = (rng.integers(0, sig, n) + 40).astype(np.uint8)
    src = text if rng.random() < 0.7 else (rng.integers(0, sig, 4096) + 40).astype(np.uint8)
    offs = rng.integers(0, max(1, src.size - m), size=r)
    pats = [src[o:o + m].tobytes() for o in offs if o + m <= src.size] or [bytes([41]) * m]
    if it % 5 == 0:
        text[n // 3:n // 3 + min(n // 4, 5000)] = text[0]  # a run of one symbol: dense steps
        pats.append(bytes([int(text[0])]) * m)
    H = int(rng.integers(1, 4))
    kw = dict(scan_kernel="roll", probes=H, warps=int(rng.choice([0, 0, 12, 16, 20, 24])))
    e = mag.Engine(pats, **kw)
    pl = e.plan()
    assert pl["roll"] and pl["tile_bytes"] == 1024, pl
    mm = e.search(text)
    got = mm.pairs()
    want = as_pairs(*ref.ac(text, pats, threads=8))
    ok = got == want and mm.metrics().candidates == roll_candidates(text, pats, pl["q"], pl["table_bytes"] // 4, H)
    bad += not ok
    print(it, 'ok' if ok else 'MISMATCH', m, sig, n, len(pats), H, kw['warps'], len(want), flush=True)
print('bad', bad)
