"""Summaries for profiles/ from raw ncu outputs.

    python tools/ncu_summaries.py launches <launches.csv> <title>   > profiles/rNN_bench_launches_summary.txt
    python tools/ncu_summaries.py full <report.ncu-rep>             > profiles/rNN_ncu_full_summary.json

`launches`: a `--metrics gpu__time_duration.sum --csv` launch list -> per-kernel
launches / mean / total / share.  `full`: key metrics per kernel of a
`--set full` capture (time, DRAM bytes, hit rates, occupancy, issue, SIMT).
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
]


def _short(name):
    name = re.sub(r"\(.*\)$", "", name) if name.count("(") > 1 else name
    return name[:60]


def launches(path, title):
    rows = list(csv.reader(open(path)))
    hdr = None
    for i, r in enumerate(rows):
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            body = rows[i + 1:]
            break
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(list)
    for r in body:
        if len(r) <= iv:
            continue
        v = float(r[iv].replace(",", ""))
        unit = r[iu]
        us = v / 1e3 if unit in ("ns", "nsecond") else v * 1e3 if unit in ("ms", "msecond") else v
        agg[r[ik]].append(us)
    tot = sum(sum(v) for v in agg.values())
    print(f"# ncu launch list of `{title}` (gpu__time_duration.sum, --clock-control none)")
    print("# cold-cache, serialised per-launch times: compare SHARES, not absolutes\n")
    print(f"{'kernel':60s} {'launches':>9s} {'mean_us':>10s} {'total_us':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{_short(k):60s} {len(v):9d} {sum(v) / len(v):10.1f} {sum(v):10.1f} {sum(v) / tot:7.3f}")


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(FULL_METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        key = d.get("Kernel Name", "?")
        out[key] = {m: f"{d[m]} {units[hdr.index(m)]}".strip() for m in FULL_METRICS if m in d}
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else sys.argv[2])
    else:
        full(sys.argv[2])
