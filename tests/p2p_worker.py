"""One rank of test_tiles_gpu.test_p2p_renderer_two_processes_ipc (run as a
script: RANK / WORLD_SIZE / MASTER_* from the environment, gloo, cuda:0;
argv[1]: TileRenderer mode, "p2p" (interleaved tiles) or "regions" (row bands))."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

import paper_2202_06088_b200 as vv
from paper_2202_06088_b200 import synthetic
from paper_2202_06088_b200.distributed import TileRenderer

W, H, TILE = 208, 144, 64


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    tree, cam = synthetic.shell_tree(depth=7, n_max=1, frames=8, seed=3), synthetic.bench_camera(W, H)
    mode = sys.argv[1] if len(sys.argv) > 1 else "p2p"
    tr = TileRenderer(W, H, TILE, rank=rank, world=world, device=dev, mode=mode)
    ok = True
    for f in (1, 4, 6):
        out = tr.render_frame(tree, cam, f)
        if rank == 0:
            torch.cuda.synchronize()
            ref = vv.render(tree, cam, f)
            for name in ("rgb", "alpha", "depth"):
                a = getattr(out, name).cpu().numpy()
                b = getattr(ref, name)
                b = b.cpu().numpy() if hasattr(b, "cpu") else np.asarray(b)
                if not np.array_equal(a, b):
                    print(f"frame {f} {name}: {np.count_nonzero(a != b)} mismatches", flush=True)
                    ok = False
        dist.barrier()  # rank 0 has read slot f before anyone renders f + 2 into it
    dist.barrier()
    tr.close()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0 and ok:
        print("P2P_OK", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
