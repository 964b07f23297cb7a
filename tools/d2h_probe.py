"""D2H bandwidth into pinned host memory: one copy stream vs two concurrent
streams (each moving half of every 41.5 MB frame)."""
import torch

n = 5 * 1920 * 1080
dev = torch.device("cuda", 0)
src = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(4)]
dst = [torch.empty(n, dtype=torch.float32, pin_memory=True) for _ in range(4)]
streams = [torch.cuda.Stream(dev) for _ in range(2)]


def run(k, frames=40):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for st in streams:
        st.wait_stream(torch.cuda.current_stream())
    for f in range(frames):
        for j in range(k):
            lo, hi = n * j // k, n * (j + 1) // k
            with torch.cuda.stream(streams[j]):
                dst[f % 4][lo:hi].copy_(src[f % 4][lo:hi], non_blocking=True)
    for st in streams[:k]:
        torch.cuda.current_stream().wait_stream(st)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    return frames * n * 4 / ms / 1e6


for _ in range(2):
    print({k: round(run(k), 1) for k in (1, 2)}, "GB/s")
