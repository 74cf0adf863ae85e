"""Markdown table of an ncu launch-list CSV (gpu__time_duration.sum [+ dram bytes]).

usage: python tools/launch_table.py LAUNCHES.csv > table.md
Excludes the FP32-peak microbenchmark and torch's own kernels (L2 flush, fills)."""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[i]
    ix = {h: j for j, h in enumerate(hdr)}
    tot, cnt, byts = collections.Counter(), collections.Counter(), collections.Counter()
    for r in rows[i + 1:]:
        name = r[ix["Kernel Name"]]
        if "fp32_peak" in name or "at::" in name:
            continue
        short = name.split("(")[0].replace("odgs_b200::", "").replace("<unnamed>::", "").replace("void ", "")
        v = float(r[ix["Metric Value"]].replace(",", ""))
        if r[ix["Metric Name"]] == "gpu__time_duration.sum":
            tot[short] += v
            cnt[short] += 1
        else:
            byts[short] += v
    total = sum(tot.values())
    print("| kernel | launches | total (ns) | share | DRAM r+w per launch (MB) |")
    print("|---|---|---|---|---|")
    for k, v in tot.most_common():
        print(f"| `{k}` | {cnt[k]} | {int(v)} | {100 * v / total:.1f}% | {byts[k] / cnt[k] / 1e6:.1f} |")


if __name__ == "__main__":
    main()
