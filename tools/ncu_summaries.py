"""Summarise ncu --set full reports into the JSON files bench.py and the
profiles/ directory carry (dram bytes per launch = the roofline `traffic`).

    python tools/ncu_summaries.py gpurun_out/r02_ncu_cfg2.ncu-rep profiles/r02_ncu_cfg2.json [...]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "smsp__inst_executed.sum": "warp_instructions",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "simt_threads_per_inst",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__cycles_active.avg": "sm_cycles_active_avg",
    "gpc__cycles_elapsed.max": "cycles_elapsed",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__occupancy_limit_registers": "occupancy_limit_registers",
    "sm__maximum_warps_per_active_cycle_pct": "theoretical_occupancy_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3,
        "nsecond": 1e-3, "ns": 1e-3}


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for d in data:
        r = {"kernel": d[hdr.index("Kernel Name")][:120]}
        for m, k in METRICS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            v = d[i].replace(",", "")
            try:
                v = float(v) * UNIT.get(units[i], 1.0)
            except ValueError:
                pass
            r[k] = v
        if "dram_read" in r and "dram_write" in r:
            r["dram_bytes_per_launch"] = r["dram_read"] + r["dram_write"]
        res.append(r)
    return res[0] if len(res) == 1 else res


if __name__ == "__main__":
    args = sys.argv[1:]
    for rep, dst in zip(args[::2], args[1::2]):
        s = summarise(rep)
        s["source"] = rep.split("/")[-1]
        with open(dst, "w") as f:
            json.dump(s, f, indent=1)
        print(dst, json.dumps({k: s[k] for k in ("kernel", "duration_us", "dram_bytes_per_launch", "issue_active_pct",
                                                 "warps_active_pct", "warp_instructions") if k in s}))
