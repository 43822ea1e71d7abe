"""Top SASS instructions by warp-stall samples from an ncu source page
(ncu -i X.ncu-rep --page source --csv --print-source sass | gzip)."""
import csv, gzip, io, sys

fn = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
rows = list(csv.reader(io.StringIO(gzip.open(fn, 'rt').read())))
hi = next(i for i, r in enumerate(rows) if 'Address' in r)
hdr = rows[hi]
body = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
A, S, N, E = hdr.index('Address'), hdr.index('Source'), hdr.index('Warp Stall Sampling (All Samples)'), hdr.index('Instructions Executed')
tot = sum(float(r[N] or 0) for r in body)
print(f'{len(body)} instructions, {tot:.0f} samples')
order = sorted(range(len(body)), key=lambda i: -float(body[i][N] or 0))
for i in order[:top]:
    r = body[i]
    print(f'{r[A]:>8} {float(r[N] or 0):7.0f} {100*float(r[N] or 0)/tot:5.1f}%  exec={r[E]:>10}  {r[S][:90]}')
