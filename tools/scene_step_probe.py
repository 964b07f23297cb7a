import sys, time, json
sys.path.insert(0, "/root/repo")
import torch
import bench
import paper_2202_06088_b200 as vv
from paper_2202_06088_b200.device import replica
wl = bench.Workload(4)
dev = torch.device("cuda", 0)
reps = [replica(t, dev) for t in wl.trees]
st = bench.Stepper(wl, dev)
frames = list(range(30))
st.prepare(set(frames))
stream = torch.cuda.current_stream(dev)
flush = torch.empty(4 * bench.L2_BYTES // 4, dtype=torch.float32, device=dev)
for f in frames[:3]:
    st(f)
torch.cuda.synchronize()
res = {}
for name, fl in (("noflush", False), ("flush", True)):
    hs = []
    for f in frames:
        if fl: flush.zero_()
        t = time.perf_counter(); st(f, None, stream); hs.append((time.perf_counter() - t) * 1e3)
    t = time.perf_counter(); torch.cuda.synchronize(); tail = (time.perf_counter() - t) * 1e3
    hs.sort(); res[name] = {"host_med_ms": round(hs[15], 3), "host_max_ms": round(hs[-1], 3), "host_sum": round(sum(hs), 2), "tail_sync_ms": round(tail, 2)}
    print(name, res[name], flush=True)
