"""Full-size golden digests of the five BASELINE.json workloads.

Run in the build container (needs oracle/_ref/libmagref.so, i.e. the
reference's own oracles.cpp compiled by `make -C oracle`):

    python tests/golden/make_full_digests.py [cfg ...]

For each config at scale 1.0 (workloads.generate, seeded) this runs the
reference's Aho–Corasick (ac_search, chunk-parallel over all host cores)
and records the match count plus sha256 digests of the text, the pattern
set and the sorted (offset u64 LE, pattern_index u32 LE) arrays into
tests/golden/full_digests.json.  The match sets themselves (up to ~16M
pairs) are too large to commit; the GPU test recomputes the digest of its
own output and compares (tests/test_gpu_parity.py::test_full_configs).
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from pyoracle import Ref  # noqa: E402

from paper_1405_5483_b200 import workloads  # noqa: E402

OUT = os.path.join(HERE, "full_digests.json")


def match_digest(offs: np.ndarray, pids: np.ndarray) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(offs, dtype="<u8").tobytes())
    h.update(np.ascontiguousarray(pids, dtype="<u4").tobytes())
    return h.hexdigest()


def input_digest(w) -> dict:
    ph = hashlib.sha256()
    for p in w.patterns:
        ph.update(len(p).to_bytes(4, "little"))
        ph.update(p)
    return {"text_sha256": hashlib.sha256(w.text.tobytes()).hexdigest(), "patterns_sha256": ph.hexdigest()}


def main(cfgs):
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            data = json.load(f)
    ref = Ref()
    for cfg in cfgs:
        t0 = time.time()
        w = workloads.generate(cfg, 1.0)
        t1 = time.time()
        offs, pids = ref.ac(w.text, w.patterns, threads=os.cpu_count())
        t2 = time.time()
        rec = {"workload": w.name, "n": int(w.text.size), "r": len(w.patterns), "matches": int(offs.size),
               "matches_sha256": match_digest(offs, pids), **input_digest(w),
               "ac_seconds": round(t2 - t1, 1), "ac_threads": os.cpu_count(),
               "source": "oracle/_ref ac_search (proj/src/oracles.cpp)"}
        data[str(cfg)] = rec
        print(cfg, rec, f"gen {t1 - t0:.1f}s", flush=True)
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main([int(x) for x in sys.argv[1:]] or [1, 2, 3, 4, 5])
