"""Device replicas of VOctrees and the torch plumbing around the C ABI.

A replica (``DeviceTree``) is one ``vv_tree`` handle: node table, payload
re-laid out as a padded w_sigma plane (128 B per leaf at C=31, one cache
line) and a padded [w_gamma | w_hh] plane, basis matrices and edit
channels, resident in HBM on one device.  Replicas are cached on the tree
object and rebuilt when any of its arrays is replaced; call
``tree.invalidate_device()`` (or ``invalidate(tree)``) after editing host
arrays in place.  Any object with the reference VOctree's attributes
(depth, n_max, node_child, leaf_data, bases.a/.b, bbox_lo, side, edit_rgb,
edit_t) is accepted, so trees built by the reference package upload too.

PyTorch provides device memory, streams and torch.distributed; it is not
on the compute path.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _native

__all__ = ["DeviceTree", "load_device", "replica", "invalidate", "sync_edits", "torch_device", "stream_ptr",
           "require_cuda"]

_lock = threading.Lock()


def _torch():
    import torch

    return torch


def require_cuda():
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("voxvid_b200 renders on a CUDA device; no GPU is visible (there is no CPU fallback)")
    return torch


def torch_device(device=None):
    torch = require_cuda()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device) if not isinstance(device, int) else torch.device("cuda", device)
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def stream_ptr(device) -> int:
    torch = _torch()
    return int(torch.cuda.current_stream(device).cuda_stream)


def _key(tree):
    ed_rgb = getattr(tree, "edit_rgb", None)
    ed_t = getattr(tree, "edit_t", None)
    return (
        id(tree.node_child), id(tree.leaf_data), id(tree.bases.a), id(tree.bases.b), id(ed_rgb), id(ed_t),
        int(tree.depth), float(tree.side), tuple(np.asarray(tree.bbox_lo, dtype=np.float64).reshape(3)),
    )


class DeviceTree:
    """An uploaded VOctree on one CUDA device (owns a ``vv_tree`` handle)."""

    def __init__(self, tree, device=None):
        torch = require_cuda()
        self.device = torch_device(device)
        lib = _native.lib()
        nc = np.ascontiguousarray(tree.node_child, dtype=np.int32)
        ld = np.ascontiguousarray(tree.leaf_data, dtype=np.float32)
        a = np.ascontiguousarray(tree.bases.a, dtype=np.float32)
        b = np.ascontiguousarray(tree.bases.b, dtype=np.float32)
        n_leaves = ld.shape[0]
        if nc.ndim != 2 or nc.shape[1] != 8:
            raise ValueError(f"node_child must be (n, 8), got {nc.shape}")
        limit = max(nc.shape[0], n_leaves)
        if nc.size and int(nc.max()) >= limit:
            raise ValueError("node table references rows beyond the tree")
        desc = _native.TreeDesc()
        desc.depth = int(tree.depth)
        desc.n_max = int(tree.n_max)
        desc.frames = int(a.shape[0])
        desc.coeff_count = int(a.shape[1])
        desc.n_internal = int(nc.shape[0])
        desc.n_leaves = int(n_leaves)
        lo = np.asarray(tree.bbox_lo, dtype=np.float64).reshape(3)
        for i in range(3):
            desc.bbox_lo[i] = float(lo[i])
        desc.side = float(tree.side)
        desc.node_child = nc.ctypes.data
        desc.leaf_data = ld.ctypes.data if n_leaves else None
        desc.basis_a = a.ctypes.data
        desc.basis_b = b.ctypes.data
        keep = [nc, ld, a, b]
        er = getattr(tree, "edit_rgb", None)
        et = getattr(tree, "edit_t", None)
        if er is not None and n_leaves:
            er = np.ascontiguousarray(er, dtype=np.float32)
            et = np.ascontiguousarray(et, dtype=np.int32)
            desc.edit_rgb = er.ctypes.data
            desc.edit_t = et.ctypes.data
            keep += [er, et]
        handle = ctypes.c_void_p()
        _native.check(lib.vv_tree_upload(ctypes.byref(desc), self.device.index, ctypes.byref(handle)))
        del keep
        self.handle = handle
        self.n_leaves = int(n_leaves)
        self.n_internal = int(nc.shape[0])
        self.depth = int(tree.depth)
        self.frames = int(a.shape[0])
        self.coeff_count = int(a.shape[1])
        self.n_max = int(tree.n_max)
        self.s = (self.n_max + 1) ** 2
        nb = ctypes.c_int64()
        _native.check(lib.vv_tree_info(handle, None, None, None, None, ctypes.byref(nb)))
        self.device_bytes = int(nb.value)

    @classmethod
    def from_voct(cls, data, device=None) -> "DeviceTree":
        """A .voct stream straight to the device (vv_voct_upload): the same
        checks and exception classes as VOctree.from_bytes (octree.py:
        413-501), no host VOctree arrays.  ``data``: bytes-like or path."""
        from . import octree as _oct

        torch = require_cuda()
        if not isinstance(data, (bytes, bytearray, memoryview, np.ndarray)):
            data = np.fromfile(str(data), dtype=np.uint8)
        buf = np.frombuffer(data, dtype=np.uint8) if not isinstance(data, np.ndarray) else data
        buf = np.ascontiguousarray(buf, dtype=np.uint8)
        self = cls.__new__(cls)
        self.device = torch_device(device)
        lib = _native.lib()
        handle = ctypes.c_void_p()
        info = _native.VoctInfo()
        rc = lib.vv_voct_upload(buf.ctypes.data if buf.size else None, buf.size, self.device.index,
                                ctypes.byref(handle), ctypes.byref(info))
        if rc != _native.VV_OK:
            exc = {_native.VV_E_TRUNCATED: _oct.TruncatedStreamError, _native.VV_E_MAGIC: _oct.BadMagicError,
                   _native.VV_E_VERSION: _oct.UnsupportedVersionError, _native.VV_E_CHECKSUM: _oct.ChecksumError,
                   _native.VV_E_FORMAT: _oct.VoctError}.get(rc)
            if exc is not None:
                raise exc(_native.last_error())
            _native.check(rc)
        self.handle = handle
        self.n_leaves = int(info.n_leaves)
        self.n_internal = int(max(info.n_internal, 1))
        self.depth = int(info.depth)
        self.frames = int(info.frames)
        self.coeff_count = int(info.coeff_count)
        self.n_max = int(info.n_max)
        self.s = (self.n_max + 1) ** 2
        self.bbox_lo = np.array(info.bbox_lo[:], dtype=np.float64)
        self.side = float(info.side)
        self.has_edits = bool(info.flags & 1)
        nb = ctypes.c_int64()
        _native.check(lib.vv_tree_info(handle, None, None, None, None, ctypes.byref(nb)))
        self.device_bytes = int(nb.value)
        return self

    @property
    def leaf_order(self) -> np.ndarray:
        """Reference row id of every device leaf row (the walk-order layout)."""
        out = np.empty(self.n_leaves, dtype=np.int32)
        _native.check(_native.lib().vv_tree_leaf_order(self.handle, out.ctypes.data))
        return out

    @property
    def dark_fraction(self) -> float:
        """Share of leaves with sigma 0 over frames 0, T/2, T-1 (measured at
        upload; above 0.5 the sliced kernels walk with the long segment queue)."""
        v = ctypes.c_float()
        _native.check(_native.lib().vv_tree_dark_fraction(self.handle, ctypes.byref(v)))
        return float(v.value)

    def visible_count(self) -> tuple:
        """(leaves, 64-leaf chunks) in the tree's visible set -- what a
        render-internal slice decodes colour for (synchronises the device)."""
        import torch

        n, c = ctypes.c_int64(), ctypes.c_int64()
        _native.check(_native.lib().vv_tree_visible_count(
            self.handle, ctypes.byref(n), ctypes.byref(c), ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)))
        return int(n.value), int(c.value)

    def visible_mask(self) -> np.ndarray:
        """Per device leaf row: whether it is in the tree's visible set."""
        import torch

        words = ((self.n_leaves + 63) // 64) * 2
        out = np.zeros(max(words, 1), dtype=np.uint32)
        _native.check(_native.lib().vv_tree_visible_bits(
            self.handle, out.ctypes.data, words, ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)))
        bits = np.unpackbits(out.view(np.uint8), bitorder="little").astype(bool)
        return bits[: self.n_leaves]

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _native.lib().vv_tree_free(h)
            except Exception:
                pass
            self.handle = None


def replica(tree, device=None) -> DeviceTree:
    """The cached device replica of ``tree`` on ``device`` (uploads on first use)."""
    if isinstance(tree, DeviceTree):
        return tree
    dev = torch_device(device)
    key = _key(tree)
    with _lock:
        cache = getattr(tree, "_vv_replicas", None)
        if cache is None:
            cache = {}
            try:
                setattr(tree, "_vv_replicas", cache)
            except AttributeError:
                pass
        hit = cache.get(dev.index)
        if hit is not None and hit[0] == key:
            return hit[1]
        rep = DeviceTree(tree, dev)
        cache[dev.index] = (key, rep)
        return rep


def invalidate(tree) -> None:
    cache = getattr(tree, "_vv_replicas", None)
    if cache:
        cache.clear()


def sync_edits(tree) -> None:
    """Push ``tree``'s host edit channels (edit_rgb / edit_t) to its cached
    replicas in place (vv_tree_set_edits) -- after paint -- instead of
    re-uploading the payload."""
    cache = getattr(tree, "_vv_replicas", None)
    if not cache:
        return
    er = getattr(tree, "edit_rgb", None)
    et = getattr(tree, "edit_t", None)
    lib = _native.lib()
    with _lock:
        for dev, (_, rep) in list(cache.items()):
            if er is None or et is None:
                _native.check(lib.vv_tree_set_edits(rep.handle, None, None))
            else:
                rgb = np.ascontiguousarray(er, dtype=np.float32)
                t = np.ascontiguousarray(et, dtype=np.int32)
                if rgb.shape != (rep.n_leaves, 4) or t.shape != (rep.n_leaves, 2):
                    raise ValueError(f"edit arrays must be ({rep.n_leaves}, 4) / ({rep.n_leaves}, 2)")
                _native.check(lib.vv_tree_set_edits(rep.handle, rgb.ctypes.data, t.ctypes.data))
            cache[dev] = (_key(tree), rep)


def load_device(path, device=None) -> DeviceTree:
    """``VOctree.load`` straight to a device replica (vv_voct_upload)."""
    return DeviceTree.from_voct(path, device)
