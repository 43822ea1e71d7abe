#!/usr/bin/env python3
"""Headline benchmark: text GB/s searched on B200 (BASELINE.json metric).

Workload (config.workload): BASELINE.json configs[1] — DNA, sigma=4, n=1 GiB
iid uniform text, r=10,000 patterns of m=32 (50% copied from the text, 50%
iid), seeded synthetic (workloads.py).  One step = one complete search of the
text through the fused sm_100a kernel up to the sorted (offset, pattern)
match array in HBM.  The text (1 GiB) is larger than L2 (126 MB), so no L2
flush is needed between steps.

N > 1 (torchrun, one rank per GPU): weak scaling over a text of N copies of
the workload text.  Rank g owns start offsets [g*n, (g+1)*n) and searches its
1 GiB plus maxlen-1 halo bytes (shard.py); the only exchange is the gather
of the per-rank sorted match lists, which the e2e leg includes.

Arms:
  default            our library; `value` = device-resident GB/s (CUDA events,
                     max over ranks), `e2e` = the same metric through
                     mag_search() with pinned host text (H2D + search + D2H
                     of the matches inside the timed region).
  --impl reference   the reference's own CPU implementation of the path
                     (Aho–Corasick from proj/src/oracles.cpp, compiled
                     unmodified into oracle/_ref) on all host cores, over a
                     bounded sample of the same workload.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

METRIC = "text GB/s searched (1 B200) and % of HBM roofline; matches bit-exact vs CPU"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region (NVML,
    every ~2 ms; nvidia-smi when NVML is unavailable)."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []  # (sm_mhz, max_mhz, [reason flags])
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml as N
            import torch
            N.nvmlInit()
            pr = torch.cuda.get_device_properties(gpu)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            try:
                h = N.nvmlDeviceGetHandleByPciBusId_v2(bus.encode())
            except Exception:
                h = N.nvmlDeviceGetHandleByIndex(gpu)
            bits = [N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                    N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap]
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            self._nvml = (N, h, bits, mx)
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        N, h, bits, mx = self._nvml
        sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
        r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
        return (float(sm), float(mx), [bool(r & b) for b in bits])

    def _sample_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        f = [x.strip() for x in out.split(",")]
        if len(f) < 6:
            return None
        return (float(f[0]), float(f[1]), [x.lower() == "active" for x in f[2:6]])

    def _run(self):
        while not self._stop.is_set():
            try:
                x = self._sample_nvml() if self._nvml else self._sample_smi()
                if x:
                    self.samples.append(x)
            except Exception:
                pass
            self._stop.wait(0.002 if self._nvml else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(s[0] for s in self.samples)
        reasons = sorted({self.NAMES[i] for s in self.samples for i in range(4) if s[2][i]})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples), "source": "nvml" if self._nvml else "nvidia-smi"}


def plan_kernel(plan):
    for k in ("direct", "roll", "pack2"):
        if plan.get(k):
            return k
    return "scan"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference(workload, threads=None):
    """Reference Aho–Corasick (oracles.cpp:78-95, compiled unmodified into
    oracle/_ref) over the WHOLE text of the workload (the same config as the
    GPU arm), chunk-parallel on `threads` host cores with maxlen-1 bytes of
    look-ahead per chunk.  Returns (GB/s, cores, sample, kind)."""
    from pyoracle import REF_SO, Port, Ref
    threads = threads or os.cpu_count() or 1
    text, pats = workload.text, workload.patterns
    if os.path.exists(REF_SO):
        ref, kind = Ref(), "reference"
        run = lambda t: ref.ac(t, pats, threads=threads)
    else:  # the C restatement's naive scan (parity-pinned) when _ref is absent
        port, kind = Port(), "port"
        run = lambda t: port.naive(t, pats)
        threads = 1
        text = text[: 1 << 24]
    t0 = time.perf_counter()
    run(text)
    dt = time.perf_counter() - t0
    sample = (f"whole {workload.name} text ({text.size} bytes), {threads} threads, automaton build included, "
              f"host CPU {cpu_model()}")
    return text.size / dt / 1e9, threads, sample, kind


def mag_restated_baseline(workload, threads, cap_s=8.0):
    """The restated reference MAG engine (oracle/mag_oracle.c mo_search:
    engine.hpp:79-85 -> filter.hpp:51-74 -> brute-force verify_window
    verify.hpp:28-31) at REFERENCE-DEFAULT parameters: the balanced map over
    the pattern histogram (mag.h:47, alphabet_map.cpp:90-102), the restated
    tuner's q and k (tuner.hpp:38-66).  Timed on doubling text prefixes until
    a run takes cap_s/4 or the whole text ran; threads > 1 split the prefix
    into chunks with maxlen-1 look-ahead (the chunk contract).
    Returns a dict; `extrapolated` when the prefix is shorter than the text."""
    from concurrent.futures import ThreadPoolExecutor
    import numpy as np
    from pyoracle import Port
    port = Port()
    text, pats = workload.text, workload.patterns
    allb = np.frombuffer(b"".join(pats), dtype=np.uint8)
    counts = np.bincount(allb, minlength=256).astype(np.uint64)
    sigma = int((counts > 0).sum())
    sp = sigma if sigma <= 64 else 256
    table, sp = port.map_build(2 if sp < 256 else 0, counts, max(sp, 2))
    m = min(len(p) for p in pats)
    tu = port.tune(sigma, len(pats), m, n=text.size)
    P = port.params(variant=0, gram_mode=0, q=tu["q"], k=tu["k"], sigma_prime=sp, table=table)
    look = max(len(p) for p in pats) - 1

    def run(size):
        if threads <= 1:
            port.search(text[:size], pats, P)
            return
        bounds = [size * c // threads for c in range(threads + 1)]
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda c: port.search(text[bounds[c]:min(size, bounds[c + 1] + look)], pats, P),
                        range(threads)))

    size, dt = 1 << 12, 0.0
    while True:
        t0 = time.perf_counter()
        run(size)
        dt = time.perf_counter() - t0
        if dt >= cap_s / 4 or size >= text.size:
            break
        size = min(text.size, size * 4 if dt < cap_s / 64 else size * 2)
    gbs = size / dt / 1e9
    return {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "port",
            "params": {"q": tu["q"], "k": tu["k"], "sigma_prime": sp, "mapping": "balance" if sp < 256 else "identity"},
            "sample": f"first {size} bytes of the {workload.name} text ({dt:.2f} s)",
            "extrapolated": size < text.size,
            "note": "prefix-extrapolated to the whole text" if size < text.size else "whole text"}


def config_sweep(cells, local, steps=10, warmup=3):
    """BASELINE.json configs, device-resident: step and scan GB/s, fraction of
    HBM, the plan, and whether the full-size match set's count + sha256 equal
    the reference AC's (tests/golden/full_digests.json).  `cells` holds
    (config, label, engine kwargs): the planner's plan ({}) and the
    reference-default exact-code plan (gram_mode=0: the restated tuner's q/k,
    the balanced map, m' = min(L/k, w/k) -- tuner.hpp:38-66, filter.hpp:51-74)."""
    import hashlib
    import numpy as np
    import torch
    import paper_1405_5483_b200 as mag
    from paper_1405_5483_b200 import workloads
    peak, _ = peaks()
    with open(os.path.join(ROOT, "tests", "golden", "full_digests.json")) as f:
        digests = json.load(f)
    out = {}
    cache = {}
    for c, label, kw in cells:
        if c not in cache:
            cache.clear()
            torch.cuda.empty_cache()
            cache[c] = workloads.generate(c, 1.0)
        w = cache[c]
        eng = mag.Engine(w.patterns, device=local, histogram_sample=w.text[:1 << 20], **kw)
        d = torch.from_numpy(w.text).to(f"cuda:{local}")
        prep = eng.prepare_device(d.data_ptr(), w.text.size, keep=d)
        m = eng.search_prepared(prep)
        offs, pids = m.arrays()
        h = hashlib.sha256()
        h.update(np.ascontiguousarray(offs, dtype="<u8").tobytes())
        h.update(np.ascontiguousarray(pids, dtype="<u4").tobytes())
        want = digests.get(str(c), {})
        ok = int(offs.size) == want.get("matches") and h.hexdigest() == want.get("matches_sha256")
        met = m.metrics()
        m.close()
        st = torch.cuda.Stream()
        for _ in range(warmup):
            eng.search_prepared_async(prep, st.cuda_stream).close()
        # inputs below L2 size (cfg1, 16 MiB): a read-only pass over 256 MiB
        # between steps evicts them without leaving dirty lines to write back
        flush = (torch.ones(64 << 20, dtype=torch.int32, device=f"cuda:{local}")
                 if w.text.size < (256 << 20) else None)
        torch.cuda.synchronize()
        ms = 0.0
        with torch.cuda.stream(st):
            for _ in range(steps):
                if flush is not None:
                    flush.sum()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                eng.search_prepared_async(prep, st.cuda_stream).close()
                e1.record(st)
                torch.cuda.synchronize()
                ms += e0.elapsed_time(e1)
        mag.scan_timer(True)  # scan kernel + finish grid
        with torch.cuda.stream(st):
            for _ in range(steps):
                if flush is not None:
                    flush.sum()
                eng.search_prepared_async(prep, st.cuda_stream).close()
        torch.cuda.synchronize()
        kms, kl = mag.scan_timer_read()
        mag.scan_timer(True, scan_only=True)  # the scan kernel alone
        with torch.cuda.stream(st):
            for _ in range(steps):
                if flush is not None:
                    flush.sum()
                eng.search_prepared_async(prep, st.cuda_stream).close()
        torch.cuda.synchronize()
        sms, sl = mag.scan_timer_read()
        mag.scan_timer(False)
        n = int(w.text.size)
        step_gbs = n / (ms / steps * 1e-3) / 1e9
        kern_gbs = n / (kms / max(kl, 1) * 1e-3) / 1e9
        scan_gbs = n / (sms / max(sl, 1) * 1e-3) / 1e9
        pl = eng.plan()
        out[f"cfg{c}{label}"] = {
            "workload": w.name, "n": n, "r": len(w.patterns), "GB/s": step_gbs, "kernel_GB/s": scan_gbs,
            "scan_kernel_GB/s": scan_gbs, "scan_frac_of_hbm": scan_gbs / peak,
            "frac_of_hbm": scan_gbs / peak, "step_frac_of_hbm": step_gbs / peak,
            "search_kernels_serialized_GB/s": kern_gbs, "matches": int(offs.size),
            "filter_reads": met.filter_reads, "candidates": met.candidates, "bit_exact_vs_reference": bool(ok),
            "l2": "read-only 256 MiB pass between steps" if flush is not None else "input larger than L2",
            "plan": {k: pl[k] for k in ("variant", "gram_mode", "q", "k", "m_prime", "sigma_prime", "table_bits",
                                        "probes", "direct", "roll", "pack2", "warps",
                                        "predicted_candidates_per_byte", "measured_candidates_per_byte")},
            "params": ("GPU planner" if not kw else
                       "reference-default exact codes (analytic-seed q/k of SURVEY 8a, balanced map)" if "q" in kw
                       else "reference-default exact codes (restated tuner's joint q/k, balanced map)")}
        del d, prep, eng, flush
        torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, help="BASELINE.json config (1-5); headline is 2")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--check", action="store_true", help="also verify the match set against oracle/_ref AC")
    ap.add_argument("--headline-only", action="store_true",
                    help="skip the per-config sweep of the other BASELINE.json configs")
    args = ap.parse_args()
    rank, world, local = dist_env()
    from paper_1405_5483_b200 import workloads

    if args.impl == "reference":
        if rank != 0:
            return
        w = workloads.generate(args.config, args.scale)
        vals = []
        for _ in range(max(args.warmup, 0)):
            cpu_reference(w)
        info = None
        for _ in range(max(args.steps, 1)):
            gbs, cores, sample, kind = cpu_reference(w)
            vals.append(gbs)
            info = (cores, sample, kind)
        v = sorted(vals)[len(vals) // 2]
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": w.text.size / (v * 1e9) * 1e3,
                "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
                "config": {"workload": w.name, "n": int(w.text.size), "r": len(w.patterns),
                           "m": w.meta["m"], "parallelism": "cpu threads"},
                "cpu_baseline": {"value": v, "unit": "GB/s", "cores": info[0], "kind": info[2],
                                 "sample": info[1], "cpu_model": cpu_model(), "same_config": True},
                "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1405_5483_b200 as mag

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    from paper_1405_5483_b200 import shard
    w = workloads.generate(args.config, args.scale)
    n = int(w.text.size)
    maxlen = max(len(p) for p in w.patterns)
    # this rank's read span of the N-copy text: its own copy + the next copy's first maxlen-1 bytes
    span = w.text if rank == world - 1 else np.concatenate([w.text, w.text[:maxlen - 1]])
    # the planner prices its finalist plans by candidate rates measured on a text sample
    eng = mag.Engine(w.patterns, device=local, histogram_sample=w.text[:1 << 20])
    plan = eng.plan()
    d_text = torch.from_numpy(span).to(f"cuda:{local}")
    prep = eng.prepare_device(d_text.data_ptr(), span.size, keep=d_text)
    stream = torch.cuda.Stream()

    # correctness anchor for this very text: one full materialised search
    first = eng.search_prepared(prep)
    n_matches = len(first)
    metrics = first.metrics()
    checked = None
    digest_ok = None
    if world == 1 and args.scale == 1.0:
        import hashlib
        with open(os.path.join(ROOT, "tests", "golden", "full_digests.json")) as f:
            want = json.load(f).get(str(args.config), {})
        offs, pids = first.arrays()
        h = hashlib.sha256()
        h.update(np.ascontiguousarray(offs, dtype="<u8").tobytes())
        h.update(np.ascontiguousarray(pids, dtype="<u4").tobytes())
        digest_ok = int(offs.size) == want.get("matches") and h.hexdigest() == want.get("matches_sha256")
    if args.check:
        from pyoracle import Ref
        want = Ref().ac(w.text, w.patterns, threads=os.cpu_count())
        offs, pids = first.arrays()
        checked = bool(np.array_equal(offs, want[0]) and np.array_equal(pids, want[1]))
    first.close()

    # ---- device-resident timing (value)
    for _ in range(max(args.warmup, 3)):
        eng.search_prepared_async(prep, stream.cuda_stream).close()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches0 = mag.kernel_launches()
    # the value region runs the product path as a caller gets it: no timing
    # events inside a search (events between the scan kernel and the finish
    # grid, or between searches, cost 5 us per step on B200)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        start.record(stream)
        for _ in range(args.steps):
            eng.search_prepared_async(prep, stream.cuda_stream).close()
        end.record(stream)
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms = start.elapsed_time(end) / args.steps
    launches = mag.kernel_launches() - launches0
    # the same searches again with CUDA events around each search's two
    # kernels (scan + finish) ...
    mag.scan_timer(True)
    for _ in range(args.steps):
        eng.search_prepared_async(prep, stream.cuda_stream).close()
    torch.cuda.synchronize()
    kernel_ms_total, kernel_launches = mag.scan_timer_read()
    # ... and around the dominant kernel alone (roofline): the end event sits
    # between the scan kernel and the finish grid
    mag.scan_timer(True, scan_only=True)
    for _ in range(args.steps):
        eng.search_prepared_async(prep, stream.cuda_stream).close()
    torch.cuda.synchronize()
    scan_ms_total, scan_launches = mag.scan_timer_read()
    mag.scan_timer(False)
    t = torch.tensor([ms], device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * n / (ms_max * 1e-3) / 1e9

    # ---- end to end through mag_search (pinned host text in, host matches out)
    pinned = torch.empty(span.size, dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = span
    host = pinned.numpy()
    m = eng.search(host)  # warm the host-text workspace
    m.close()
    torch.cuda.synchronize()
    barrier()
    e2e_t = []
    d2h = 0
    total_matches = None
    for _ in range(max(args.e2e_steps, 1)):
        barrier()
        t0 = time.perf_counter()
        m = eng.search(host)
        offs, pids = m.arrays()
        offs, pids = shard.clip(offs, pids, 0, n)
        got = shard.gather(offs + np.uint64(rank * n), pids, world, rank)
        e2e_t.append(time.perf_counter() - t0)
        d2h = len(m) * 8 + 4 * 8  # sorted 8-byte match keys + the mapped counter words
        if got is not None:
            total_matches = int(got[0].size)
        m.close()
    # the same pinned buffer copied to the device and nothing else: the PCIe
    # ceiling the end-to-end number sits under
    d_tmp = torch.empty(span.size, dtype=torch.uint8, device=f"cuda:{local}")
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d_tmp.copy_(pinned, non_blocking=True)
    torch.cuda.synchronize()
    c0.record()
    for _ in range(3):
        d_tmp.copy_(pinned, non_blocking=True)
    c1.record()
    torch.cuda.synchronize()
    h2d_only = span.size / (c0.elapsed_time(c1) / 3 * 1e-3) / 1e9
    del d_tmp
    e2e_s = sorted(e2e_t)[len(e2e_t) // 2]
    te = torch.tensor([e2e_s], device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * n / float(te.item()) / 1e9

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src = peaks()
    search_ms = kernel_ms_total / max(kernel_launches, 1)  # scan kernel + finish grid
    kernel_ms = scan_ms_total / max(scan_launches, 1)       # scan kernel alone
    achieved = n / (kernel_ms * 1e-3) / 1e9
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                tj = json.load(f)
            traffic = tj.get(f"cfg{args.config}")
            traffic_src = "static, not measured in this run: " + tj.get("source", "")
        except Exception:
            traffic = None
    sweep = None
    if not args.headline_only and world == 1:
        cells = []
        for c in (1, 2, 3, 4, 5):
            if c != args.config:
                cells.append((c, "", {}))
            cells.append((c, "_reference_params", {"gram_mode": 0}))
        # SURVEY 8a's other reading of the bodiless tuner (analytic seeds, no joint grid)
        for c, q, k in ((1, 5, 1), (3, 3, 1), (5, 6, 1)):
            cells.append((c, "_analytic_seed_params", {"gram_mode": 0, "q": q, "k": k}))
        cells.sort(key=lambda x: x[0])
        sweep = config_sweep(cells, local)
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        gbs, cores, sample, kind = cpu_reference(w)
        cpu = {"value": gbs, "unit": "GB/s", "cores": cores, "kind": kind, "sample": sample,
               "cpu_model": cpu_model(), "same_config": args.scale == 1.0,
               "mag_restated": [mag_restated_baseline(w, 1), mag_restated_baseline(w, os.cpu_count() or 1)]}
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": w.name, "n": n, "r": len(w.patterns), "m": w.meta["m"],
                   "parallelism": f"text shards x{world} (N copies, halo maxlen-1)" if world > 1 else "single GPU",
                   "l2": "input (1 GiB) larger than L2; no flush needed" if n > (126 << 20)
                   else "input smaller than L2 (not flushed)",
                   "plan": {k: plan[k] for k in ("variant", "gram_mode", "q", "k", "m_prime", "table_bits",
                                                 "entry_bits", "verify_all", "prefilter_bits", "tile_bytes",
                                                 "warps", "stages", "smem_bytes", "direct", "roll", "probes",
                                                 "predicted_candidates_per_byte",
                                                 "measured_candidates_per_byte", "measured_sample_bytes",
                                                 "predicted_cost", "measured_cost", "measured_plans")},
                   "matches": n_matches, "job_matches": total_matches, "filter_reads": metrics.filter_reads,
                   "candidates": metrics.candidates, "checked_vs_reference_ac": checked,
                   "bit_exact_vs_reference_digest": digest_ok},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": peak_src, "kernel_ms": kernel_ms, "algorithmic_bytes_per_launch": n,
                     "kernel": f"mag_{plan_kernel(plan)}_kernel (CUDA events around it on the launch stream, "
                               f"{scan_launches} launches after the value region)",
                     "search_kernels_serialized_ms": search_ms,
                     "search_kernels_serialized_frac": n / (search_ms * 1e-3) / 1e9 / peak,
                     "search_kernels_serialized": "scan kernel + mag_finish_kernel (one search = these two launches), "
                                       "CUDA events around each search in a pass after the value region "
                                       "(the events themselves keep consecutive searches from overlapping, "
                                       "so this can exceed ms_per_step)",
                     "step_frac": value / world / peak},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "GB/s", "h2d_bytes_per_step": int(span.size), "d2h_bytes_per_step": d2h,
                "api": "mag_search (pinned host text) + clip + rank-ordered gather",
                "h2d_copy_only_gbs": h2d_only,
                "note": "bounded by the host-to-device copy of the text (h2d_copy_only_gbs: the same pinned "
                        "buffer copied and nothing else)"},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "configs": sweep,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
