#!/bin/bash
# usage: tools/prof_summary.sh <rep> <kernel-substring>  (run from the repo root, after
# extracting the matching build's cubins into /tmp/cubin)
rep=$1; kern=$2
ncu -i $rep --page source --csv --print-source sass 2>/dev/null > /tmp/sass.csv
for metric in "Warp Stall Sampling (All Samples)" "Instructions Executed"; do
python tools/ncu_lines.py /tmp/sass.csv /tmp/cubin/scan_kernels.sm_100a.cubin "$kern" "$metric" 28 | python -c "
import re,sys
src={'scan_kernels.cu':open('paper_1405_5483_b200/csrc/scan_kernels.cu').read().split('\n'),'mag_common.h':open('paper_1405_5483_b200/csrc/mag_common.h').read().split('\n')}
for ln in sys.stdin:
    m=re.search(r\"\('([^']+)', (\d+)\)\",ln)
    extra=''
    if m and m.group(1) in src: extra=src[m.group(1)][int(m.group(2))-1].strip()[:80]
    print(ln.rstrip()[:60], '|', extra)
"
done
ncu -i $rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for i,k in enumerate(h):
    if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued'):
        try:
            if float(v[i])>2000: print(k, v[i])
        except: pass
    if k in ('gpu__time_duration.sum','sm__inst_executed.sum','smsp__inst_executed.avg.per_cycle_active','dram__bytes_read.sum','dram__bytes_write.sum','sm__warps_active.avg.pct_of_peak_sustained_active','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','lts__t_bytes.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed'): print(k,v[i])
"
