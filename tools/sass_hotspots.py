"""Attribute ncu per-instruction warp-stall samples to source lines.

    python tools/sass_hotspots.py <report.ncu-rep> <demangled-regex> <mangled-regex> <lib.so> [top]

Uses `ncu --page source --print-source sass` (samples per SASS address) and
`nvdisasm -g` on the cubin inside the shared library (address -> file:line).
"""
import csv
import io
import re
import subprocess
import sys
import tempfile
from collections import defaultdict
from pathlib import Path

rep, dre, kre, so = sys.argv[1], sys.argv[2], sys.argv[3], str(Path(sys.argv[4]).resolve())
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
allrows = list(csv.reader(io.StringIO(raw)))
# the CSV holds one section per profiled kernel: pick the one matching kre
sections, cur = [], None
for r in allrows:
    if r and r[0] == "Kernel Name":
        cur = [r]
        sections.append(cur)
    elif cur is not None:
        cur.append(r)
rows = None
for sec in sections:
    if re.search(dre, sec[0][1]):
        rows = sec
        break
rows = rows or sections[0]
kname = rows[0][1]
hdr = rows[1]
ia, isrc, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
iexec = hdr.index("Instructions Executed")
ithr = hdr.index("Thread Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
recs = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    recs.append(r)
base = int(recs[0][ia], 16)
# map mangled name via nvdisasm function list
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=td, capture_output=True)
    dis = ""
    for cub in Path(td).glob("*.cubin"):
        d = subprocess.run(["nvdisasm", "-gi", "-c", str(cub)], capture_output=True, text=True).stdout
        if re.search(kre, d):
            dis = d
            break
# find function block matching kernel regex on demangled-ish name
funcs = re.split(r"\n\s*\.text\.", dis)
target = None
for f in funcs:
    head = f.split("\n", 1)[0]
    if re.search(kre, head):
        target = f
        break
if target is None:
    sys.exit(f"kernel {kre} not found in cubin")
HELPER_MAX_LINE = int(__import__("os").environ.get("HELPER_MAX_LINE", "100"))


def _is_helper(fname, line):
    return fname.endswith(".hpp") or fname.endswith(".h") or (fname == "vv_device.cuh" and line < HELPER_MAX_LINE)


line_of = {}
cur = None
in_chain = False
for ln in target.split("\n"):
    m = re.search(r"//## File \"([^\"]+)\", line (\d+)(?: inlined at \"([^\"]+)\", line (\d+))?", ln)
    if m:
        # nvdisasm -gi prints the inline chain innermost -> outermost: keep the first
        if in_chain:
            continue
        in_chain = True
        cur = f"{Path(m.group(1)).name}:{m.group(2)}"
        # tiny helpers (fp64 wrappers, intrinsics headers) -> their call site
        if m.group(3) and (_is_helper(Path(m.group(1)).name, int(m.group(2)))):
            cur = f"{Path(m.group(3)).name}:{m.group(4)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m:
        in_chain = False
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
agg = defaultdict(lambda: [0, 0, 0, defaultdict(int)])
total = 0
for r in recs:
    off = int(r[ia], 16) - base
    s = int(r[isamp] or 0)
    total += s
    key = line_of.get(off, "?")
    a = agg[key]
    a[0] += s
    a[1] += int(r[iexec] or 0)
    a[2] += int(r[ithr] or 0)
    for i in stall_cols:
        a[3][hdr[i]] += int(r[i] or 0)
print(kname[:120], "total samples", total)
REGIONS = __import__("os").environ.get("REGIONS")  # "name:lo-hi,name:lo-hi" over vv_device.cuh lines
if REGIONS:
    buckets = defaultdict(lambda: [0, 0])
    tot_wait = sum(a[3].get("stall_wait", 0) for a in agg.values())
    for key, (s_, ex, th, st) in agg.items():
        f, _, ln = key.partition(":")
        name = "other:" + f
        if f == "vv_device.cuh" and ln.isdigit():
            for spec in REGIONS.split(","):
                nm, rng = spec.split(":")
                lo_, hi_ = (int(x) for x in rng.split("-"))
                if lo_ <= int(ln) <= hi_:
                    name = nm
                    break
        buckets[name][0] += ex
        buckets[name][1] += s_
        buckets[name].append(st.get("stall_wait", 0))
    tot_ex = sum(v[0] for v in buckets.values())
    for nm, vals in sorted(buckets.items(), key=lambda kv: -kv[1][0]):
        ex, s_, w = vals[0], vals[1], sum(vals[2:])
        print(f"  region {nm:24s} inst={ex:>11d} ({ex / tot_ex * 100:5.1f}%)  samples {s_ / total * 100:5.1f}%"
              f"  wait {w:6d} ({w / max(tot_wait, 1) * 100:4.1f}% of wait)")
SORT_IDX = int(__import__("os").environ.get("SORT", "0"))
for key, (s, ex, th, st) in sorted(agg.items(), key=lambda kv: -kv[1][SORT_IDX])[:int(sys.argv[5]) if len(sys.argv) > 5 else 40]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    eff = th / ex if ex else 0
    print(f"{s / total * 100:5.1f}%  {key:28s} inst={ex:>10d} thr/inst={eff:5.1f}  " +
          " ".join(f"{k[6:]}={v}" for k, v in top))
