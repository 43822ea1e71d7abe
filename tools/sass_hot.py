"""Summarise an ncu source page (--print-source sass --csv): hottest
instructions by executed count and by stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
key = sys.argv[2] if len(sys.argv) > 2 else "Instructions Executed"
def num(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except Exception:
        return 0.0
tot = sum(num(r, key) for r in data)
print(f"total {key}: {tot:.4g}")
for r in sorted(data, key=lambda r: -num(r, key))[: int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print(f"{num(r, key):12.4g} {num(r,'Warp Stall Sampling (All Samples)'):8.0f} {r[ix['Address']]:>6s} {r[ix['Source']][:90]}")
