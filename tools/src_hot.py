"""Per-source-line totals from `ncu -i R --page source --csv --print-source cuda,sass`.

usage: python tools/src_hot.py MIXED.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, line, src = "?", "?", ""
inst = collections.Counter()
samp = collections.Counter()
text = {}
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0] != "":
        line, src = r[0], r[1]
        text[(fname, line)] = src.strip()
        continue
    try:
        n = int(r[7])
        s = int(r[4])
    except ValueError:
        continue
    inst[(fname, line)] += n
    samp[(fname, line)] += s
tot_i = sum(inst.values())
tot_s = sum(samp.values())
print("total inst", tot_i, "samples", tot_s)
for k, s in samp.most_common(top):
    print(f"{k[0][:18]:18s}:{k[1]:>4s} samp {100*s/tot_s:5.1f}% inst {100*inst[k]/tot_i:5.1f}%  {text.get(k, '')[:90]}")
