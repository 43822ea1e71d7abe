"""Attribute an ncu SASS source page to CUDA source lines.

usage: ncu_lines.py <sass.csv> <cubin> <kernel-substring> [metric] [top]

<sass.csv> is `ncu -i rep --page source --csv --print-source sass`; the
cubin comes from `cuobjdump -xelf all libmag_b200.so` of the SAME build.
Offsets are matched function-relative; line info needs -lineinfo.
"""
import csv
import re
import subprocess
import sys
from collections import defaultdict


def line_map(cubin, kern):
    out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    funcs = {}
    cur = None
    loc = None
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur = m.group(1)
            funcs[cur] = {}
            loc = None
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            loc = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m and cur is not None:
            funcs[cur][int(m.group(1), 16)] = loc
    cands = [f for f in funcs if kern in f]
    return cands, funcs


def main():
    sass, cubin, kern = sys.argv[1:4]
    metric = sys.argv[4] if len(sys.argv) > 4 else "Warp Stall Sampling (All Samples)"
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    rows = list(csv.reader(open(sass)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    base = min(int(r[ix["Address"]], 16) for r in data)
    cands, funcs = line_map(cubin, kern)
    # pick the function whose size matches the profiled one
    n = len(data)
    best = min(cands, key=lambda f: abs(len(funcs[f]) - n))
    fmap = funcs[best]
    agg = defaultdict(float)
    tot = 0.0
    for r in data:
        off = int(r[ix["Address"]], 16) - base
        try:
            v = float(r[ix[metric]].replace(",", ""))
        except ValueError:
            v = 0.0
        tot += v
        agg[fmap.get(off)] += v
    print(f"function {best[:100]} ({n} sass rows, {len(fmap)} mapped); total {metric} {tot:.4g}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        print(f"{v / max(tot, 1) * 100:6.2f}% {v:12.4g}  {k}")


if __name__ == "__main__":
    main()
