"""A/B of the planner's measured-rate decision: word-Zipf text,
patterns copied from it.  Times the analytic choice, the measured choice and
the forced alternatives, device-resident."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import paper_1405_5483_b200 as mag
from test_planner import copied, zipf_words_text

rng = np.random.default_rng(3)
for vocab, r, m in ((200, 5000, 24), (200, 5000, 16), (50, 20000, 16), (200, 20000, 32)):
    text = zipf_words_text(rng, 24_000_000, vocab)
    pats = copied(rng, text, r, m)
    d = torch.from_numpy(text).cuda()
    print(f"== vocab {vocab} r {r} m {m} n {text.size}")
    for label, kw in (("analytic", {}), ("measured", dict(histogram_sample=text[:1 << 20])),
                      ("direct8", dict(scan_kernel="direct", q=8, gram_mode=1)),
                      ("direct16", dict(scan_kernel="direct", q=16, gram_mode=1)),
                      ("roll", dict(scan_kernel="roll")), ("staged", dict(scan_kernel="staged"))):
        try:
            e = mag.Engine(pats, **kw)
        except Exception as ex:
            print(f"  {label}: {str(ex)[:80]}")
            continue
        p = e.prepare_device(d.data_ptr(), d.numel(), keep=d)
        first = e.search_prepared(p)
        nm, cands = len(first), first.metrics().candidates
        first.close()
        s = torch.cuda.Stream()
        for _ in range(2):
            e.search_prepared_async(p, s.cuda_stream).close()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(5):
            e.search_prepared_async(p, s.cuda_stream).close()
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        pl = e.plan()
        print(f"  {label}: direct={pl['direct']} roll={pl['roll']} q={pl['q']} probes={pl['probes']} "
              f"matches={nm} cand/B={cands / text.size:.4f} pred={pl['predicted_candidates_per_byte']:.4f} "
              f"meas={pl['measured_candidates_per_byte']:.4f} cost={pl['predicted_cost']:.1f}/{pl['measured_cost']:.1f} "
              f"{text.size / ms / 1e6:.0f} GB/s")
