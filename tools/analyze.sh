#!/bin/bash
# usage: tools/analyze.sh <rep>   — summary of a scan-kernel ncu capture (run from repo root;
# the in-tree libmag_b200.so must be the build that was profiled)
rep=$1
mkdir -p /tmp/cubin && (cd /tmp/cubin && rm -f *.cubin && cuobjdump -xelf all "$OLDPWD/paper_1405_5483_b200/libmag_b200.so" >/dev/null 2>&1)
ncu -i $rep --page details --csv 2>/dev/null | grep -E '"Executed Instructions"|"Executed Ipc Active"|"Issue Slots Busy"|"Achieved Occupancy"|"Registers Per Thread"|"DRAM Throughput"|"Duration"' | awk -F'","' '{print $(NF-2), $NF}'
ncu -i $rep --page source --csv --print-source sass 2>/dev/null > /tmp/sass.csv
K=$(head -1 /tmp/sass.csv | grep -o "mag_scan_kernel<[^>]*>" | sed -E 's/mag_scan_kernel<\(int\)([0-9]), unsigned int, \(bool\)([01]), \(int\)([0-9]), \(int\)([0-9]), \(int\)([0-9]), \(bool\)([01])>/ILi\1EjLb\2ELi\3ELi\4ELi\5ELb\6E/')
echo "kernel $K"
python tools/ncu_lines.py /tmp/sass.csv /tmp/cubin/scan_kernels.sm_100a.cubin $K "Instructions Executed" 600 | python -c "
import re,sys,bisect
src=open('paper_1405_5483_b200/csrc/scan_kernels.cu').read().split('\n')
starts=[(i+1,l.strip()[:50]) for i,l in enumerate(src) if re.match(r'\s*(__device__|template|__global__)', l) and '(' in l]
keys=[s for s,_ in starts]
tot={}; all_=0
for ln in sys.stdin:
    m=re.search(r\"^\s*([\d.]+)%\s+([\d.e+]+)\s+\('([^']+)', (\d+)\)\",ln)
    if not m: continue
    v=float(m.group(2)); f=m.group(3); l=int(m.group(4)); all_+=v
    if f!='scan_kernels.cu': tot[f]=tot.get(f,0)+v; continue
    i=bisect.bisect_right(keys,l)-1
    name=starts[i][1] if i>=0 else '?'
    tot[name]=tot.get(name,0)+v
for n,v in sorted(tot.items(),key=lambda x:-x[1])[:16]: print(f'{v/all_*100:5.1f}% {v:10.3g}  {n}')
print('total', all_)
"
ncu -i $rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for i,k in enumerate(h):
    if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued'):
        try:
            if float(v[i])>1000: print(k.replace('smsp__pcsamp_warps_issue_stalled_',''), v[i])
        except: pass
"
