"""Minimal driver for ncu: a few device-resident searches of one config."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1405_5483_b200 as mag  # noqa: E402
from paper_1405_5483_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--opts", default="", help="engine kwargs, e.g. tile_bytes=16384,warps=8")
ap.add_argument("--r", type=int, default=0, help="replace the pattern set by r iid patterns (length m)")
a = ap.parse_args()
kw = {}
for kv in filter(None, a.opts.split(",")):
    k, v = kv.split("=")
    kw[k] = int(v) if v.lstrip("-").isdigit() else v
w = workloads.generate(a.config, a.scale)
if a.r:
    import numpy as np
    rng = np.random.default_rng(7)
    m = w.meta["m"]
    alpha = np.unique(w.text[: 1 << 20])
    w.patterns = [alpha[rng.integers(0, alpha.size, m)].tobytes() for _ in range(a.r)]
e = mag.Engine(w.patterns, **kw)
d = torch.from_numpy(w.text).cuda()
p = e.prepare_device(d.data_ptr(), d.numel(), keep=d)
s = torch.cuda.Stream()
e.search_prepared(p).close()  # materialised once: the engine learns the staging capacity per slice
for _ in range(2):  # warm-up: lazy module load, workspace allocation
    e.search_prepared_async(p, s.cuda_stream).close()
torch.cuda.synchronize()
mag.scan_timer(True)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record(s)
for _ in range(a.iters):
    e.search_prepared_async(p, s.cuda_stream).close()
ev1.record(s)
torch.cuda.synchronize()
step_ms = ev0.elapsed_time(ev1) / a.iters
ms, n = mag.scan_timer_read()
m = e.search_prepared(p)
print(f"{w.name} plan={e.plan()} matches={len(m)} metrics={m.metrics()} kernel_ms={ms / max(n, 1):.3f} "
      f"GB/s={w.text.size / (ms / max(n, 1)) / 1e6:.1f} step_ms={step_ms:.3f} step_GB/s={w.text.size / step_ms / 1e6:.1f}")
