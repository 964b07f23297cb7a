"""Image-tile sharding across GPUs (one process per GPU, torch.distributed/NCCL).

Each rank holds a full replica of the tree and renders the square tiles
whose row-major tile index i satisfies i % world == rank (interleaved, so
the ~33% of hit rays, which cluster on the performer, spread evenly).  A
rank writes its tiles packed as (n_my_tiles, tile*tile, 5) float32
[r, g, b, alpha, depth] (vv_render_camera_tiles); one all-gather (NCCL over
NVLink/NVSwitch) of equal-size slabs brings every rank's slab to the
output rank, where vv_unpack_tiles scatters them into full images.  This is
the only exchange step per frame.

``mode="p2p"`` fuses the render and the gather instead: the output rank
allocates the frame's image planes (two slots) with CUDA IPC
(vv_ipc_alloc), every rank maps them (vv_ipc_open) and its tile kernel
(vv_render_camera_tiles_direct) stores each finished pixel straight into
the output rank's planes over NVLink/NVSwitch -- no slab, no all-gather,
no unpack kernel.  One stream-ordered barrier per frame (a one-element
NCCL all-reduce, queued after the kernel on every rank) publishes it.

``mode="regions"`` splits the frame into contiguous row bands instead,
balanced by each row's measured walk cost (``row_costs``: the leaf samples
of a counting render; ``band_plan``): a rank renders its band with
vv_render_camera_region straight into the output rank's planes, and --
the point of contiguous regions -- slices only the leaf chunks whose cells
can project into its band (k_chunk_cull), so the per-frame decode is
sharded across the ranks along with the walk.  Interleaved tiles make
every rank decode the whole tree.

The host-side layout helpers here are also restated in numpy
(``unpack_tiles_host``) so the CPU test-suite can check the protocol with
the gloo backend and world_size 2 without a GPU.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native

__all__ = ["tile_grid", "tiles_of", "slab_tiles", "unpack_tiles_host", "pack_tiles_host", "tile_mask_host",
           "band_plan", "pixel_costs", "row_costs", "block_shape", "block_order", "render_region", "TileRenderer"]

BAND_ALIGN = 8  # band edges on camera-block rows (vv_kernels.cuh kTH)


def band_plan(costs, n: int, align: int = BAND_ALIGN) -> list:
    """Split rows into n contiguous bands of near-equal total cost.

    ``costs``: per-row cost (len = image height).  Edges sit on multiples of
    ``align`` (whole camera blocks) except the last; returns n + 1 edges
    [0, e1, ..., H] (a band may be empty when rows are scarce)."""
    costs = np.asarray(costs, dtype=np.float64)
    h = len(costs)
    cum = np.concatenate([[0.0], np.cumsum(costs)])
    edges = [0]
    for k in range(1, n):
        target = cum[-1] * k / n
        r = int(np.searchsorted(cum, target))
        r = int(round(r / align)) * align
        edges.append(min(max(r, edges[-1]), h))
    edges.append(h)
    return edges


def pixel_costs(tree, cam, frame: int = 0, opts=None, device=None, miss_cost: float = 1.0):
    """(H, W) float64 CUDA tensor: each pixel's walk cost -- the leaf samples
    its ray consumes (one counting render, vv_render_camera_counts) plus
    ``miss_cost`` for ray generation and setup (a ray that misses costs
    about as much as one sample).  Deterministic: every rank computes the
    same plan from it."""
    import torch

    from .device import torch_device
    from .render import RenderOptions, render_into

    dev = torch_device(device)
    h, w = int(cam.height), int(cam.width)
    used = torch.empty((h, w), dtype=torch.int32, device=dev)
    alpha = torch.empty((h, w), dtype=torch.float32, device=dev)
    render_into(tree, cam, frame, None, alpha, None, opts or RenderOptions(), sample_count=used)
    return used.to(torch.float64) + miss_cost


def row_costs(tree, cam, frame: int = 0, opts=None, device=None, miss_cost: float = 1.0):
    """Per-row sums of ``pixel_costs`` (numpy)."""
    return pixel_costs(tree, cam, frame, opts, device, miss_cost).sum(dim=1).cpu().numpy()


def block_shape():
    """Pixel footprint (width, height) of one camera-kernel block."""
    w, h = ctypes.c_int32(), ctypes.c_int32()
    _native.check(_native.lib().vv_camera_block_shape(ctypes.byref(w), ctypes.byref(h)))
    return int(w.value), int(h.value)


def block_order(costs, rect):
    """Launch order of the camera blocks of ``rect`` = (x0, y0, x1, y1),
    costliest first (int32 CUDA tensor for vv_render_camera_region), from
    per-pixel ``costs`` (H, W tensor): the expensive blocks start first and
    the cheap ones fill the tail of the kernel."""
    import torch

    x0, y0, x1, y1 = (int(v) for v in rect)
    bw, bh = block_shape()
    nbx, nby = -(-(x1 - x0) // bw), -(-(y1 - y0) // bh)
    sub = torch.zeros((nby * bh, nbx * bw), dtype=torch.float64, device=costs.device)
    sub[: y1 - y0, : x1 - x0] = costs[y0:y1, x0:x1]
    per = sub.reshape(nby, bh, nbx, bw).sum(dim=(1, 3)).reshape(-1)
    return torch.argsort(per, descending=True, stable=True).to(torch.int32).contiguous()


def render_region(tree, cam, frame, rect, rgb, alpha, depth, opts=None, cache=None, *, peer: bool = False,
                  device=None, order=None, plan=None):
    """Render the pixel rectangle rect = (x0, y0, x1, y1) of ``cam`` into
    full-size planes (device pointers or tensors; may be a peer's IPC
    mapping), its blocks launched in ``order`` (block_order) if given, or
    scheduled by a CameraPlan (``plan``: the rank's own cost order and cached
    coverage).  Async on the device's current stream."""
    from .device import replica, stream_ptr, torch_device
    from .render import RenderOptions, _check_cache

    dev = torch_device(device)
    opts = opts or RenderOptions()
    rep = replica(tree, dev)
    ch = _check_cache(cache, int(frame), rep)
    ptr = (lambda x: x if isinstance(x, int) or x is None else x.data_ptr())
    r = (ctypes.c_int32 * 4)(*[int(v) for v in rect])
    if plan is not None:
        _native.check(_native.lib().vv_render_camera_planned(
            rep.handle, int(frame), ch, ctypes.byref(opts.c_struct()), ctypes.byref(cam.desc()), r, plan._handle,
            ptr(rgb), ptr(alpha), ptr(depth), int(bool(peer)), stream_ptr(dev)))
        return
    _native.check(_native.lib().vv_render_camera_region(
        rep.handle, int(frame), ch, ctypes.byref(opts.c_struct()), ctypes.byref(cam.desc()), r, ptr(order), ptr(rgb),
        ptr(alpha), ptr(depth), int(bool(peer)), stream_ptr(dev)))


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


def tile_mask_host(rank: int, world: int, width: int, height: int, tile: int) -> np.ndarray:
    """(H, W) bool: the pixels `rank`'s tiles cover (what the direct tile
    kernel writes; the ranks' masks partition the image)."""
    tx, _, _ = tile_grid(width, height, tile)
    m = np.zeros((height, width), dtype=bool)
    for tid in tiles_of(rank, world, width, height, tile):
        x0, y0 = (tid % tx) * tile, (tid // tx) * tile
        m[y0:y0 + tile, x0:x0 + tile] = True
    return m


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


class _Planes:
    """A raw device allocation seen by torch (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3,
                                         "strides": None}


class TileRenderer:
    """Per-rank tile renderer for one camera size.

    mode="gather": render_slab + gather (NCCL all-gather) + unpack.
    mode="p2p": render_frame stores this rank's tiles straight into the
    output rank's image planes (CUDA IPC over NVLink), then one
    stream-ordered barrier; see the module docstring.
    """

    def __init__(self, width: int, height: int, tile: int = 64, rank: int = 0, world: int = 1, device=None,
                 group=None, mode: str = "gather", out_rank: int = 0):
        import torch

        from .device import torch_device

        if tile % 16:
            raise ValueError("tile must be a multiple of 16")
        if mode not in ("gather", "p2p", "regions"):
            raise ValueError(f"mode must be 'gather', 'p2p' or 'regions', not {mode!r}")
        self.width, self.height, self.tile = int(width), int(height), int(tile)
        self.rank, self.world, self.group = int(rank), int(world), group
        self.mode, self.out_rank = mode, int(out_rank)
        self.device = torch_device(device)
        self.per = slab_tiles(world, width, height, tile)
        self.bands = None
        if mode == "gather":
            self.slab = torch.zeros((self.per, tile * tile, 5), dtype=torch.float32, device=self.device)
            self.all = torch.empty((world, self.per, tile * tile, 5), dtype=torch.float32, device=self.device)
        else:
            self._init_p2p(torch)

    # ------------------------------------------------------------ regions mode
    def plan(self, tree, cam, frame: int = 0, opts=None, costs=None):
        """Row bands for mode="regions", balanced on ``costs`` (per-pixel
        (H, W) CUDA tensor; default: the measured pixel_costs of ``frame``),
        and this rank's block launch order.  Call with the same arguments on
        every rank (the plan is deterministic)."""
        if costs is None:
            costs = pixel_costs(tree, cam, frame, opts, self.device)
        from .render import CameraPlan

        self.bands = band_plan(costs.sum(dim=1).cpu().numpy(), self.world)
        self.cam_plan = CameraPlan(self.device)  # launch order learned from this rank's own frames
        return self.bands

    def region(self, rank=None):
        r = self.rank if rank is None else rank
        return (0, self.bands[r], self.width, self.bands[r + 1])

    # ------------------------------------------------------------ p2p mode
    def _init_p2p(self, torch):
        import torch.distributed as dist

        lib, dev = _native.lib(), self.device.index
        n = 2 * 5 * self.width * self.height  # two frame slots of [rgb | alpha | depth]
        self._slot = 0
        self._owned = self._mapped = None
        handle = (ctypes.c_ubyte * 64)()
        base = None
        if self.rank == self.out_rank:
            ptr = ctypes.c_void_p()
            _native.check(lib.vv_ipc_alloc(dev, 4 * n, ctypes.byref(ptr), handle))
            self._owned = base = ptr.value
        if self.world > 1:
            obj = [bytes(handle) if self.rank == self.out_rank else None]
            dist.broadcast_object_list(obj, src=self.out_rank, group=self.group)
            if self.rank != self.out_rank:
                ctypes.memmove(handle, obj[0], 64)
                ptr = ctypes.c_void_p()
                _native.check(lib.vv_ipc_open(dev, handle, ctypes.byref(ptr)))
                self._mapped = base = ptr.value
            self._flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._base = base
        self.planes = None
        if self.rank == self.out_rank:
            self.planes = torch.as_tensor(_Planes(base, n), device=self.device).view(2, -1)

    def _slot_ptrs(self, slot):
        hw = self.width * self.height
        base = self._base + slot * 5 * hw * 4
        return base, base + 3 * hw * 4, base + 4 * hw * 4

    def _views(self, slot):
        from .render import LayerImages

        h, w = self.height, self.width
        b = self.planes[slot]
        return LayerImages(b[: 3 * h * w].view(h, w, 3), b[3 * h * w: 4 * h * w].view(h, w), b[4 * h * w:].view(h, w))

    def barrier(self):
        """Stream-ordered on NCCL (a one-element all-reduce queued after the
        tile kernel); host-synchronous on gloo (functional runs)."""
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return
        torch.cuda.nvtx.range_push("vv:gather_barrier")
        try:
            self._barrier(torch, dist)
        finally:
            torch.cuda.nvtx.range_pop()

    def _barrier(self, torch, dist):
        if dist.get_backend(self.group) == "nccl":
            dist.all_reduce(self._flag, group=self.group)
        else:
            torch.cuda.current_stream(self.device).synchronize()
            dist.barrier(group=self.group)

    def render_frame(self, tree, cam, frame, opts=None, cache=None):
        """p2p mode: render this rank's tiles of `frame` into the output
        rank's planes and publish them.  On the output rank returns device
        LayerImages views of the frame's slot (valid until the render_frame
        call after next: two slots); None elsewhere."""
        from .device import replica, stream_ptr
        from .render import RenderOptions, _check_cache

        if self.mode == "gather":
            raise RuntimeError("render_frame needs mode='p2p' or 'regions' (gather mode: render_slab/gather/unpack)")
        if (int(cam.width), int(cam.height)) != (self.width, self.height):
            raise ValueError(f"camera is {cam.width}x{cam.height}, renderer {self.width}x{self.height}")
        opts = opts or RenderOptions()
        rep = replica(tree, self.device)
        ch = _check_cache(cache, int(frame), rep)
        oc = opts.c_struct()
        cd = cam.desc()
        slot = self._slot
        self._slot ^= 1
        rgb, alpha, depth = self._slot_ptrs(slot)
        if self.mode == "regions":
            if self.bands is None:
                self.plan(tree, cam, frame, opts)
            r = (ctypes.c_int32 * 4)(*self.region())
            _native.check(_native.lib().vv_render_camera_planned(
                rep.handle, int(frame), ch, ctypes.byref(oc), ctypes.byref(cd), r, self.cam_plan._handle, rgb, alpha,
                depth, int(self.rank != self.out_rank), stream_ptr(self.device)))
        else:
            _native.check(_native.lib().vv_render_camera_tiles_direct(
                rep.handle, int(frame), ch, ctypes.byref(oc), ctypes.byref(cd), self.tile, self.rank, self.world,
                rgb, alpha, depth, int(self.rank != self.out_rank), stream_ptr(self.device)))
        self.barrier()
        return self._views(slot) if self.rank == self.out_rank else None

    def close(self):
        """Unmap / free the IPC planes (p2p mode).  Call on every rank once
        no rank will render into them again."""
        if self.mode == "gather":
            return
        import torch

        torch.cuda.synchronize(self.device)
        lib, dev = _native.lib(), self.device.index
        self.planes = None
        if self._mapped:
            _native.check(lib.vv_ipc_close(dev, self._mapped))
            self._mapped = None
        if self._owned:
            _native.check(lib.vv_ipc_free(dev, self._owned))
            self._owned = None

    # --------------------------------------------------------- gather mode

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

        import torch

        torch.cuda.nvtx.range_push("vv:gather")
        try:
            self._gather(dist)
        finally:
            torch.cuda.nvtx.range_pop()
        return self.all

    def _gather(self, dist):
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
