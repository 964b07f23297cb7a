"""cfg2 slice pass alone: complete slice (build_frame_cache) vs the
render-internal one render() runs (build_frame_caches(render_only=True)),
L2 flushed before each pass."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2202_06088_b200 as vv  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402

tree = synthetic.shell_tree()
flush = torch.empty(64 * 2**20, dtype=torch.float32, device="cuda")


def ev(fn, n=15):
    for i in range(3):
        fn(i)
    tot = 0.0
    for i in range(n):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        c = fn(i)
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
        del c
    return round(tot / n, 4)


print(json.dumps({"complete_ms": ev(lambda i: vv.build_frame_cache(tree, (7 * i) % 30)),
                  "render_only_ms": ev(lambda i: vv.build_frame_caches(tree, [(7 * i) % 30], render_only=True))}))
