"""Multi-rank tile sharding protocol on CPU: gloo backend, world_size 2.

Checks the host half of the multi-GPU path (paper_2202_06088_b200/distributed.py):
interleaved tile ownership is a partition of the tile grid, equal-size rank
slabs all-gather into the shard-major layout vv_unpack_tiles expects, and
unpacking reproduces the full image exactly.
"""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2202_06088_b200.distributed import pack_tiles_host, slab_tiles, tile_grid, tiles_of, unpack_tiles_host

W, H, TILE = 200, 150, 64


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        img = np.random.default_rng(7).random((H, W, 5)).astype(np.float32)
        slab = torch.from_numpy(pack_tiles_host(img, rank, world, TILE))
        parts = [torch.empty_like(slab) for _ in range(world)]
        dist.all_gather(parts, slab)
        full = unpack_tiles_host(torch.stack(parts).numpy(), W, H, TILE, world)
        t = torch.tensor([float(np.array_equal(full, img))])
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if rank == 0:
            q.put(float(t.item()))
    finally:
        dist.destroy_process_group()


def test_tile_partition():
    for world in (1, 2, 3, 8):
        _, _, total = tile_grid(W, H, TILE)
        owned = [t for r in range(world) for t in tiles_of(r, world, W, H, TILE)]
        assert sorted(owned) == list(range(total))
        assert max(len(tiles_of(r, world, W, H, TILE)) for r in range(world)) == slab_tiles(world, W, H, TILE)


def test_gather_unpack_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) == 1.0


def test_band_plan_balances_and_aligns():
    from paper_2202_06088_b200.distributed import band_plan

    rng = np.random.default_rng(1)
    costs = np.concatenate([np.full(200, 0.1), rng.uniform(5, 50, 680), np.full(200, 0.1)])
    for n in (1, 2, 3, 8):
        e = band_plan(costs, n)
        assert len(e) == n + 1 and e[0] == 0 and e[-1] == len(costs)
        assert all(a <= b for a, b in zip(e, e[1:]))
        assert all(x % 8 == 0 for x in e[1:-1])
        per = [costs[a:b].sum() for a, b in zip(e, e[1:])]
        assert max(per) <= costs.sum() / n + 8 * costs.max() + 1e-9
    assert band_plan(np.ones(5), 4)[-1] == 5  # fewer rows than bands
