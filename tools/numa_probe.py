"""Host topology of the GPU box and device->host bandwidth into pinned
memory allocated with the process bound to each NUMA node in turn (the
e2e number is PCIe/host-memory bound)."""
import json
import os
import subprocess
import sys
import time

import torch

out = {"cpu_count": os.cpu_count(), "affinity": sorted(os.sched_getaffinity(0))}
try:
    out["smi_topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[-1500:]
except Exception as e:  # noqa: BLE001
    out["smi_topo"] = str(e)
bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
out["pci_bus_id"] = bus
nodes = {}
base = "/sys/devices/system/node"
if os.path.isdir(base):
    for d in sorted(os.listdir(base)):
        if d.startswith("node") and d[4:].isdigit():
            with open(f"{base}/{d}/cpulist") as f:
                nodes[int(d[4:])] = f.read().strip()
out["nodes"] = nodes
try:
    busid = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader"], capture_output=True,
                           text=True).stdout.strip().lower()
    dom = busid[4:] if len(busid) > 12 else busid
    for cand in (busid, "0000" + busid[8:] if busid.startswith("00000000") else busid):
        p = f"/sys/bus/pci/devices/{cand.lower()}/numa_node"
        if os.path.exists(p):
            out["gpu_numa_node"] = open(p).read().strip()
            out["gpu_sysfs"] = p
except Exception as e:  # noqa: BLE001
    out["gpu_numa_err"] = str(e)


def parse(lst):
    cpus = set()
    for part in lst.split(","):
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        elif part:
            cpus.add(int(part))
    return cpus


n = 5 * 1920 * 1080
dev = torch.empty(n, device="cuda")
res = {}
orig = os.sched_getaffinity(0)
for node, lst in (nodes or {-1: ""}).items():
    if node >= 0:
        cpus = parse(lst) & orig
        if not cpus:
            continue
        os.sched_setaffinity(0, cpus)
    host = torch.empty(n, pin_memory=True)
    for _ in range(3):
        host.copy_(dev, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(20):
        host.copy_(dev, non_blocking=True)
    torch.cuda.synchronize()
    res[node] = round(20 * 4 * n / (time.perf_counter() - t) / 1e9, 2)
    del host
    os.sched_setaffinity(0, orig)
out["d2h_gbs_by_node"] = res
print(json.dumps(out, indent=1))
