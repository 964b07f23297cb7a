"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel counts, mean durations and shares of the total.

    python tools/launch_summary.py gpurun_out/launches.csv "<command line>" > profiles/rNN_bench_launches_summary.txt
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
acc = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0][:72]
    v = float(d["Metric Value"].replace(",", ""))
    if d.get("Metric Unit", "") in ("msecond", "ms"):
        v *= 1e3
    elif d.get("Metric Unit", "") in ("nsecond", "ns"):
        v *= 1e-3
    acc.setdefault(name, []).append(v)
total = sum(sum(v) for v in acc.values())
print(sys.argv[2] if len(sys.argv) > 2 else "")
print("(cold-cache, serialised launches; shares of the whole run)\n")
print(f"{'kernel':<74}{'n':>4}{'mean_us':>10}{'share':>8}")
for k, v in acc.items():
    print(f"{k:<74}{len(v):>4}{sum(v) / len(v):>10.2f}{sum(v) / total:>8.1%}")
