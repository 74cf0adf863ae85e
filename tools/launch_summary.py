"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
start = next(i for i, r in enumerate(rows) if r[0] == "ID")
rows = rows[start:]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot = collections.Counter()
cnt = collections.Counter()
seen = set()
for r in rows[1:]:
    if len(r) != len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    lid = int(r[ix["ID"]])
    if lid < skip:
        continue
    name = r[ix["Kernel Name"]].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("odgs_b200::", "").split("(")[0].split("<")[0]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    v = v / 1000.0 if unit in ("nsecond", "ns") else (v if unit in ("usecond", "us") else v * 1000.0)
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"total {T/1000:.3f} ms over {sum(cnt.values())} launches")
for k, v in tot.most_common():
    print(f"  {k:40s} {v/1000:8.3f} ms  {100*v/T:5.1f}%  x{cnt[k]}")
