"""Per-SASS-instruction hot list from `ncu -i R --page source --csv --print-source sass`.

usage: python tools/sass_hot.py SASS.csv [top]
Prints total instructions executed, the opcode mix, and the top instructions by
stall samples."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr) and r[ix["Instructions Executed"]].isdigit()]
tot = 0
mix = collections.Counter()
samp = collections.Counter()
for r in data:
    n = int(r[ix["Instructions Executed"]] or 0)
    tot += n
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    mix[op.split(".")[0]] += n
    samp[op.split(".")[0]] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
print("total warp-instructions", tot)
for op, n in mix.most_common(30):
    print(f"  {op:10s} {n:14d} {100*n/tot:5.1f}%  samples {samp[op]}")
print("--- top by samples")
data.sort(key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
for r in data[:top]:
    print(f"{r[ix['Address']][-5:]} {r[ix['Warp Stall Sampling (All Samples)']]:>6s} {r[ix['Instructions Executed']]:>11s} {r[ix['Avg. Threads Executed']]:>6s}  {r[ix['Source']].strip()}")
