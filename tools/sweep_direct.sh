# usage: bash tools/sweep_direct.sh "<opts1>" "<opts2>" ...   (cfg2, kernel + step GB/s per option set)
for o in "$@"; do echo "== $o"; timeout 120 python tools/profile_run.py --config 2 --iters 10 --opts "$o" 2>&1 | grep -o "candidates=[0-9]*\|kernel_ms.*\|'probes': [0-9]*\|'table_bits': [0-9]*\|'warps': [0-9]*\|Error.*" | tr '\n' ' '; echo; done
