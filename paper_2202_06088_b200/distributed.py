"""Image-tile sharding across GPUs (one process per GPU, torch.distributed/NCCL).

Each rank holds a full replica of the tree and renders the square tiles
whose row-major tile index i satisfies i % world == rank (interleaved, so
the ~33% of hit rays, which cluster on the performer, spread evenly).  A
rank writes its tiles packed as (n_my_tiles, tile*tile, 5) float32
[r, g, b, alpha, depth] (vv_render_camera_tiles); one all-gather (NCCL over
NVLink/NVSwitch) of equal-size slabs brings every rank's slab to the
output rank, where vv_unpack_tiles scatters them into full images.  This is
the only exchange step per frame.

The host-side layout helpers here are also restated in numpy
(``unpack_tiles_host``) so the CPU test-suite can check the protocol with
the gloo backend and world_size 2 without a GPU.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native

__all__ = ["tile_grid", "tiles_of", "slab_tiles", "unpack_tiles_host", "pack_tiles_host", "TileRenderer"]


def tile_grid(width: int, height: int, tile: int):
    tx = (width + tile - 1) // tile
    ty = (height + tile - 1) // tile
    return tx, ty, tx * ty


def tiles_of(rank: int, world: int, width: int, height: int, tile: int) -> list:
    """Row-major tile ids owned by `rank` (interleaved assignment)."""
    _, _, total = tile_grid(width, height, tile)
    return list(range(rank, total, world))


def slab_tiles(world: int, width: int, height: int, tile: int) -> int:
    """Tiles per rank slab (equal-size slabs for all-gather; short ranks pad)."""
    _, _, total = tile_grid(width, height, tile)
    return (total + world - 1) // world


def pack_tiles_host(img5: np.ndarray, rank: int, world: int, tile: int) -> np.ndarray:
    """Numpy restatement of vv_render_camera_tiles' output layout from a full
    (H, W, 5) image (test helper)."""
    h, w, _ = img5.shape
    tx, _, _ = tile_grid(w, h, tile)
    per = slab_tiles(world, w, h, tile)
    out = np.zeros((per, tile * tile, 5), dtype=np.float32)
    for k, tid in enumerate(tiles_of(rank, world, w, h, tile)):
        x0, y0 = (tid % tx) * tile, (tid // tx) * tile
        blk = np.zeros((tile, tile, 5), dtype=np.float32)
        blk[..., 4] = 1e9
        sub = img5[y0:y0 + tile, x0:x0 + tile]
        blk[: sub.shape[0], : sub.shape[1]] = sub
        out[k] = blk.reshape(-1, 5)
    return out


def unpack_tiles_host(packed_all: np.ndarray, width: int, height: int, tile: int, world: int) -> np.ndarray:
    """Numpy restatement of vv_unpack_tiles: (world, per, tile*tile, 5) -> (H, W, 5)."""
    tx, _, total = tile_grid(width, height, tile)
    per = slab_tiles(world, width, height, tile)
    packed_all = packed_all.reshape(world, per, tile, tile, 5)
    out = np.zeros((height, width, 5), dtype=np.float32)
    for tid in range(total):
        shard, k = tid % world, tid // world
        x0, y0 = (tid % tx) * tile, (tid // tx) * tile
        blk = packed_all[shard, k]
        out[y0:y0 + tile, x0:x0 + tile] = blk[: min(tile, height - y0), : min(tile, width - x0)]
    return out


class TileRenderer:
    """Per-rank tile renderer + NCCL gather for one camera size."""

    def __init__(self, width: int, height: int, tile: int = 64, rank: int = 0, world: int = 1, device=None,
                 group=None):
        import torch

        from .device import torch_device

        if tile % 16:
            raise ValueError("tile must be a multiple of 16")
        self.width, self.height, self.tile = int(width), int(height), int(tile)
        self.rank, self.world, self.group = int(rank), int(world), group
        self.device = torch_device(device)
        self.per = slab_tiles(world, width, height, tile)
        self.slab = torch.zeros((self.per, tile * tile, 5), dtype=torch.float32, device=self.device)
        self.all = torch.empty((world, self.per, tile * tile, 5), dtype=torch.float32, device=self.device)

    def render_slab(self, tree, cam, frame, opts=None, cache=None):
        """Render this rank's tiles into self.slab (async on the current stream)."""
        from .device import replica, stream_ptr
        from .render import RenderOptions, _check_cache

        opts = opts or RenderOptions()
        rep = replica(tree, self.device)
        ch = _check_cache(cache, int(frame), rep)
        oc = opts.c_struct()
        cd = cam.desc()
        _native.check(_native.lib().vv_render_camera_tiles(
            rep.handle, int(frame), ch, ctypes.byref(oc), ctypes.byref(cd), self.tile, self.rank, self.world,
            self.slab.data_ptr(), stream_ptr(self.device)))
        return self.slab

    def gather(self):
        """All-gather every rank's slab (one collective per frame)."""
        import torch.distributed as dist

        if self.world == 1:
            self.all[0].copy_(self.slab)
        elif dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(self.all.view(-1), self.slab.view(-1), group=self.group)
        else:  # gloo (functional runs): list form
            dist.all_gather(list(self.all.unbind(0)), self.slab, group=self.group)
        return self.all

    def unpack(self, rgb, alpha, depth):
        from .device import stream_ptr

        _native.check(_native.lib().vv_unpack_tiles(
            self.all.data_ptr(), self.width, self.height, self.tile, self.world,
            rgb.data_ptr() if rgb is not None else None, alpha.data_ptr() if alpha is not None else None,
            depth.data_ptr() if depth is not None else None, stream_ptr(self.device)))
