"""Volume rendering of one VOctree at a camera and frame index -- B200 path.

Drop-in for the reference's ``voxvid.render`` (pkg/src/voxvid/render.py):
``Camera``, ``LayerImages``, ``RenderOptions``, ``FrameSlice``,
``render``, ``render_rays``, ``finalize_layer``, ``composite_background``
and ``build_frame_cache`` keep their names, arguments, defaults and error
behaviour (ValueError for a frame outside [0, T) or a cache built for
another frame).  Every render runs the hand-written sm_100a kernels of
libvoxvid_b200.so; there is no CPU fallback.

Return types: ``render`` returns float32 numpy images by default
(``out="torch"`` keeps them as CUDA tensors); ``render_rays`` returns
float64 arrays like the reference -- numpy for numpy inputs, CUDA tensors
for CUDA tensor inputs.  ``render`` fuses Camera.rays, the render kernel
and finalize_layer into one launch; camera rays are generated on the GPU
in float64 (they agree with the host's BLAS-built rays to <= 1 ulp; use
``render_rays`` with host rays when bit-exact visit lists are required).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .device import replica, require_cuda, stream_ptr, torch_device

__all__ = [
    "Camera",
    "LayerImages",
    "RenderOptions",
    "FrameSlice",
    "CameraPlan",
    "render",
    "render_into",
    "render_frames_into",
    "render_sequence",
    "render_rays",
    "render_ray_visits",
    "finalize_layer",
    "composite_background",
    "build_frame_cache",
    "build_frame_caches",
    "count_segments",
    "collect_segments",
]


@dataclass(frozen=True)
class Camera:
    """Pinhole camera (render.py:42-125): pixel centres, +z forward, +y down."""

    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    c2w: np.ndarray

    def __post_init__(self):
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError("focal lengths must be positive")
        c2w = np.asarray(self.c2w, dtype=np.float64).reshape(4, 4)
        object.__setattr__(self, "c2w", c2w)
        r = c2w[:3, :3]
        err = float(np.abs(r @ r.T - np.eye(3)).max())
        if err > 1e-9:
            raise ValueError(f"camera rotation not orthonormal: max deviation {err:.3e}")
        if not np.allclose(c2w[3], [0, 0, 0, 1], atol=1e-12):
            raise ValueError("camera pose must be a rigid transform (last row 0 0 0 1)")

    @property
    def origin(self) -> np.ndarray:
        return self.c2w[:3, 3]

    def rays(self):
        """All pixel rays on the host, row-major, unit directions (render.py:74-83)."""
        ix, iy = np.meshgrid(np.arange(self.width), np.arange(self.height), indexing="xy")
        x = (ix + 0.5 - self.cx) / self.fx
        y = (iy + 0.5 - self.cy) / self.fy
        d_cam = np.stack([x, y, np.ones_like(x)], axis=-1).reshape(-1, 3)
        d_world = d_cam @ self.c2w[:3, :3].T
        d_world /= np.linalg.norm(d_world, axis=1, keepdims=True)
        origins = np.broadcast_to(self.origin, d_world.shape).copy()
        return origins, np.ascontiguousarray(d_world)

    def pixel_rays(self, ix, iy):
        ix = np.asarray(ix, dtype=np.float64)
        iy = np.asarray(iy, dtype=np.float64)
        x = (ix + 0.5 - self.cx) / self.fx
        y = (iy + 0.5 - self.cy) / self.fy
        d_cam = np.stack([x, y, np.ones_like(x)], axis=-1)
        d_world = d_cam @ self.c2w[:3, :3].T
        d_world /= np.linalg.norm(d_world, axis=-1, keepdims=True)
        origins = np.broadcast_to(self.origin, d_world.shape).copy()
        return origins.reshape(-1, 3), np.ascontiguousarray(d_world.reshape(-1, 3))

    @staticmethod
    def look_at(eye, target, up=(0.0, 0.0, 1.0), width=128, height=128, focal=None, cx=None, cy=None) -> "Camera":
        eye = np.asarray(eye, dtype=np.float64)
        target = np.asarray(target, dtype=np.float64)
        fwd = target - eye
        fwd /= np.linalg.norm(fwd)
        upv = np.asarray(up, dtype=np.float64)
        right = np.cross(fwd, upv)
        if np.linalg.norm(right) < 1e-12:
            upv = np.array([0.0, 1.0, 0.0])
            right = np.cross(fwd, upv)
        right /= np.linalg.norm(right)
        down = np.cross(fwd, right)
        c2w = np.eye(4)
        c2w[:3, 0] = right
        c2w[:3, 1] = down
        c2w[:3, 2] = fwd
        c2w[:3, 3] = eye
        focal = float(focal) if focal is not None else 1.2 * max(width, height)
        return Camera(width=width, height=height, fx=focal, fy=focal,
                      cx=width / 2.0 if cx is None else cx, cy=height / 2.0 if cy is None else cy, c2w=c2w)

    def desc(self) -> _native.CameraDesc:
        d = _native.CameraDesc()
        d.width = int(self.width)
        d.height = int(self.height)
        d.fx, d.fy, d.cx, d.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        flat = np.ascontiguousarray(self.c2w, dtype=np.float64).reshape(16)
        for i in range(16):
            d.c2w[i] = float(flat[i])
        return d


@dataclass
class LayerImages:
    """One rendered layer: unpremultiplied rgb, alpha matte, expected depth (render.py:128-145)."""

    rgb: object
    alpha: object
    depth: object

    def __post_init__(self):
        if tuple(self.rgb.shape[:2]) != tuple(self.alpha.shape) or tuple(self.alpha.shape) != tuple(self.depth.shape):
            raise ValueError("layer channel shapes disagree")

    @property
    def shape(self):
        return tuple(self.alpha.shape)

    def copy(self) -> "LayerImages":
        c = (lambda x: x.clone()) if hasattr(self.rgb, "clone") else (lambda x: x.copy())
        return LayerImages(c(self.rgb), c(self.alpha), c(self.depth))


_SLICE_MODES = {"auto": 0, "per_sample": 1, "per_frame": 2}


@dataclass(frozen=True)
class RenderOptions:
    """render.py:148-153, plus ``frame_slice``: how leaves are decoded when no
    FrameSlice is passed -- "per_sample" (inside the render kernel, like the
    reference's uncached branch), "per_frame" (one coalesced pass over all
    leaves into a transient device slice, then render from it) or "auto".
    All are bitwise identical."""

    early_stop: float = 1e-4
    far_plane: float = 1e9
    alpha_floor: float = 1e-3
    edit_weight: float = 1.0
    frame_slice: str = "auto"

    def __post_init__(self):
        if self.frame_slice not in _SLICE_MODES:
            raise ValueError(f"frame_slice must be one of {sorted(_SLICE_MODES)}, got {self.frame_slice!r}")

    def c_struct(self, tmin: float = 0.0, tmax: float = 1e30) -> _native.RenderOpts:
        o = _native.RenderOpts()
        o.early_stop = float(self.early_stop)
        o.far_plane = float(self.far_plane)
        o.alpha_floor = float(self.alpha_floor)
        o.edit_weight = float(self.edit_weight)
        o.tmin = float(tmin)
        o.tmax = float(tmax)
        o.frame_slice = _SLICE_MODES[self.frame_slice]
        return o


class FrameSlice:
    """Per-frame device cache: sigma (f64) and sliced SH coefficients (fp32) per leaf.

    Built by build_frame_cache (render.py:170-179); renders with and
    without it are bitwise equal.  ``sigma`` (n_leaves,) float64 and ``q``
    (n_leaves, 3S) float32 are exported lazily as CUDA tensors.
    """

    def __init__(self, frame: int, handle, rep, device, plan=None):
        self.frame = int(frame)
        self._handle = handle
        self._rep = rep
        self._device = device
        self._plan = plan  # a plan-backed visible slice reads the plan's walk table: keep the plan alive
        self._sigma = None
        self._q = None

    @property
    def sigma(self):
        if self._sigma is None:
            torch = require_cuda()
            sigma = torch.empty(self._rep.n_leaves, dtype=torch.float64, device=self._device)
            _native.check(_native.lib().vv_slice_export(self._handle, sigma.data_ptr(), None,
                                                        stream_ptr(self._device)))
            self._sigma = sigma
        return self._sigma

    @property
    def q(self):
        if self._q is None:
            torch = require_cuda()
            q = torch.empty((self._rep.n_leaves, 3 * self._rep.s), dtype=torch.float32, device=self._device)
            _native.check(_native.lib().vv_slice_export(self._handle, None, q.data_ptr(), stream_ptr(self._device)))
            self._q = q
        return self._q

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                _native.lib().vv_slice_free(h)
            except Exception:
                pass
            self._handle = None


class CameraPlan:
    """Launch plan of one camera stream (vv_camera_plan).

    Renders through a plan run the camera kernel as persistent warps taking
    the frame's warp chunks in the previous render's measured cost order
    (costliest first), and record this render's costs for the next -- for
    playback, a fixed view or one rank's region, where consecutive frames
    cost alike.  Scheduling only: the pixels are bitwise those of a plain
    render.  Use a plan from one CUDA stream at a time.
    """

    def __init__(self, device=None):
        dev = torch_device(device)
        self.device = dev
        h = ctypes.c_void_p()
        _native.check(_native.lib().vv_camera_plan_create(dev.index if dev.index is not None else 0,
                                                          ctypes.byref(h)))
        self._handle = h

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                _native.lib().vv_camera_plan_free(h)
            except Exception:
                pass
            self._handle = None


_PLANS = {}


def _stream_plan(dev, stream_handle: int, kind: str = "camera") -> CameraPlan:
    """The plan render() (kind "camera") or render_scene() ("scene") keeps per
    (device, stream): renders on one stream are ordered, so its plan is never
    used concurrently."""
    key = (dev.index, stream_handle, kind)
    p = _PLANS.get(key)
    if p is None:
        if len(_PLANS) > 16:
            _PLANS.clear()
        p = _PLANS[key] = CameraPlan(dev)
    return p


class _PinnedPool:
    """Reusable pinned host buffers for device->host results.

    A buffer is handed out again only after every numpy array viewing it has
    been garbage-collected (tracked with a weakref to the base array), so
    results never alias while avoiding a cudaHostAlloc per call.
    """

    def __init__(self):
        self._free = {}  # nbytes -> list of (tensor, weakref or None)
        self._lock = __import__("threading").Lock()

    def get(self, n_floats: int):
        import weakref

        torch = require_cuda()
        with self._lock:
            lst = self._free.setdefault(n_floats, [])
            for i, (t, ref) in enumerate(lst):
                if ref is None or ref() is None:
                    arr = t.numpy()
                    lst[i] = (t, weakref.ref(arr))
                    return t, arr
            t = torch.empty(n_floats, dtype=torch.float32, pin_memory=True)
            arr = t.numpy()
            lst.append((t, weakref.ref(arr)))
            if len(lst) > 8:  # drop the oldest idle buffers beyond a small cap
                lst[:] = [e for e in lst if e[1] is not None and e[1]() is not None] + \
                    [e for e in lst if e[1] is None or e[1]() is None][:4]
            return t, arr


_PINNED = _PinnedPool()


def _frame_index(frame, tree=None) -> int:
    """Frame index of ``frame``.  A non-integer float is a continuous time:
    clamped to [0, T-1] and rounded to the nearest frame, as the reference's
    track_value does (temporal.py:229-235); integers keep the
    reference's range check (ValueError in _check_frame)."""
    if isinstance(frame, (float, np.floating)) and not float(frame).is_integer():
        t = float(frame)
        if tree is not None:
            frames = tree.bases.frames if hasattr(tree, "bases") else tree.frames
            t = min(max(t, 0.0), frames - 1.0)
        return int(round(t))
    return int(frame)


def _check_frame(tree, frame: int):
    frames = tree.bases.frames if hasattr(tree, "bases") else tree.frames
    if not (0 <= frame < frames):
        raise ValueError(f"frame {frame} out of range [0, {frames})")


def _check_cache(cache, frame, rep):
    if cache is None:
        return None
    if not isinstance(cache, FrameSlice):
        raise TypeError("cache must be a FrameSlice from build_frame_cache")
    if cache.frame != frame:
        raise ValueError(f"cache built for frame {cache.frame}, not {frame}")
    if cache._rep is not rep:
        raise ValueError("cache was built for a different tree or device")
    return cache._handle


def build_frame_cache(tree, frame: int, device=None) -> FrameSlice:
    frame = _frame_index(frame, tree)
    _check_frame(tree, frame)
    dev = torch_device(device)
    rep = replica(tree, dev)
    handle = ctypes.c_void_p()
    _native.check(_native.lib().vv_slice_build(rep.handle, frame, stream_ptr(dev), ctypes.byref(handle)))
    return FrameSlice(frame, handle, rep, dev)


def build_frame_caches(tree, frames, device=None, *, render_only: bool = False, visible: bool = False,
                       plan=None) -> list:
    """Slices of 1..4 frames from ONE pass over the payload (vv_slice_build_multi):
    each leaf row is read once and sliced per frame; ``[build_frame_cache(tree, f) for f in frames]``
    with a quarter to a half of the HBM traffic.  ``render_only``: the
    colour of leaves dark (sigma 0) in every frame is omitted
    (VV_SLICE_RENDER_ONLY) -- rendering is bitwise the same, ``q`` cannot be
    read.  ``visible`` (one frame, implies ``render_only``): colour only for
    the tree's visible set -- the leaves its camera renders have shaded
    lately; the walk decodes any other lit leaf it meets from the payload
    (VV_SLICE_VISIBLE; what render() slices internally).  Single-frame
    renders only: ``render_frames_into`` rejects such a slice.  ``plan``
    (with ``visible``): a CameraPlan keeping the slice's walk table across
    frames (rebuilt only when the set changes); render each such slice
    before building the plan's next one."""
    frames = [_frame_index(f, tree) for f in frames]
    for f in frames:
        _check_frame(tree, f)
    if not 1 <= len(frames) <= 4:
        raise ValueError("1..4 frames per slice pass")
    if visible and len(frames) != 1:
        raise ValueError("a visible-set slice holds one frame")
    flags = (_native.VV_SLICE_RENDER_ONLY if render_only or visible else 0) | \
        (_native.VV_SLICE_VISIBLE if visible else 0)
    dev = torch_device(device)
    rep = replica(tree, dev)
    n = len(frames)
    handles = (ctypes.c_void_p * n)()
    if visible and plan is not None:
        _native.check(_native.lib().vv_slice_build_visible(rep.handle, frames[0], plan._handle, stream_ptr(dev),
                                                           handles))
        return [FrameSlice(frames[0], ctypes.c_void_p(handles[0]), rep, dev, plan)]
    _native.check(_native.lib().vv_slice_build_frames(rep.handle, n, (ctypes.c_int32 * n)(*frames), flags,
                                                      stream_ptr(dev), handles))
    return [FrameSlice(f, ctypes.c_void_p(h), rep, dev) for f, h in zip(frames, handles)]


def _as_device_rays(x, dev):
    torch = require_cuda()
    if isinstance(x, torch.Tensor):
        t = x.to(device=dev, dtype=torch.float64)
        return t.reshape(-1, 3).contiguous(), True
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1, 3))
    return torch.from_numpy(a).to(dev, non_blocking=False), False


def render_rays(tree, origins, dirs, frame: int, opts: RenderOptions = RenderOptions(), cache=None, *,
                device=None, stats: bool = False):
    """Raw per-ray accumulators (premult, alpha, tbar), float64 (render.py:182-215).

    With ``stats=True`` also returns a dict of per-ray int32 counters:
    ``sample_count`` (leaf segments consumed up to and including the
    early-stop one), ``node_pops`` and ``shaded``.
    """
    torch = require_cuda()
    frame = _frame_index(frame, tree)
    _check_frame(tree, frame)
    if cache is not None and getattr(cache, "frame", frame) != frame:
        raise ValueError(f"cache built for frame {cache.frame}, not {frame}")
    dev = torch_device(device if device is not None else (origins.device if isinstance(origins, torch.Tensor) else None))
    rep = replica(tree, dev)
    ch = _check_cache(cache, frame, rep)
    o, on_dev = _as_device_rays(origins, dev)
    d, _ = _as_device_rays(dirs, dev)
    n = o.shape[0]
    premult = torch.empty((n, 3), dtype=torch.float64, device=dev)
    alpha = torch.empty(n, dtype=torch.float64, device=dev)
    tbar = torch.empty(n, dtype=torch.float64, device=dev)
    counters = None
    if stats:
        counters = {k: torch.empty(n, dtype=torch.int32, device=dev) for k in ("sample_count", "node_pops", "shaded")}
    oc = opts.c_struct()
    _native.check(_native.lib().vv_render_rays(
        rep.handle, frame, ch, ctypes.byref(oc), o.data_ptr(), d.data_ptr(), n,
        premult.data_ptr(), alpha.data_ptr(), tbar.data_ptr(),
        counters["sample_count"].data_ptr() if stats else None,
        counters["node_pops"].data_ptr() if stats else None,
        counters["shaded"].data_ptr() if stats else None,
        stream_ptr(dev)))
    if on_dev:
        out = (premult, alpha, tbar)
        return out + (counters,) if stats else out
    out = (premult.cpu().numpy(), alpha.cpu().numpy(), tbar.cpu().numpy())
    if stats:
        return out + ({k: v.cpu().numpy() for k, v in counters.items()},)
    return out


def render_ray_visits(tree, origins, dirs, frame: int, opts: RenderOptions = RenderOptions(), cache=None, *,
                      device=None):
    """Visited-leaf lists (reference row ids) for each ray, as CSR.

    Returns (sample_count (n,) int32, visit_start (n+1,) int64, visit_leaf
    (sum,) int64) as numpy arrays; visit_leaf[visit_start[r]:visit_start[r+1]]
    are the leaves ray r consumed, near to far, up to and including the
    early-stop one (the reference's seg_leaf[start:start+used],
    train.py:269-296).
    """
    torch = require_cuda()
    frame = _frame_index(frame, tree)
    _check_frame(tree, frame)
    dev = torch_device(device)
    rep = replica(tree, dev)
    ch = _check_cache(cache, frame, rep)
    o, _ = _as_device_rays(origins, dev)
    d, _ = _as_device_rays(dirs, dev)
    n = o.shape[0]
    _, _, _, st = render_rays(tree, o, d, frame, opts, cache, device=dev, stats=True)
    used = st["sample_count"]
    start = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    if n:
        start[1:] = torch.cumsum(used.to(torch.int64), 0)
    total = int(start[-1].item()) if n else 0
    leaf = torch.empty(max(total, 1), dtype=torch.int64, device=dev)
    oc = opts.c_struct()
    if n:
        _native.check(_native.lib().vv_render_rays_visits(
            rep.handle, frame, ch, ctypes.byref(oc), o.data_ptr(), d.data_ptr(), n, start.data_ptr(),
            leaf.data_ptr(), stream_ptr(dev)))
    return used.cpu().numpy(), start.cpu().numpy(), leaf[:total].cpu().numpy()


def finalize_layer(premult, alpha, tbar, shape, opts: RenderOptions, depth_scale=None) -> LayerImages:
    """LayerImages from raw accumulators (render.py:218-233), float64 numpy."""
    h, w = shape
    premult = np.asarray(premult, dtype=np.float64)
    alpha = np.asarray(alpha, dtype=np.float64)
    tbar = np.asarray(tbar, dtype=np.float64)
    alpha_img = alpha.reshape(h, w)
    safe = np.maximum(alpha, 1e-300)[:, None]
    rgb = np.where(alpha[:, None] > 0.0, premult / safe, 0.0).reshape(h, w, 3)
    t = tbar / np.maximum(alpha, 1e-300)
    if depth_scale is not None:
        t = t * depth_scale
    depth = np.where(alpha >= opts.alpha_floor, t, opts.far_plane).reshape(h, w)
    return LayerImages(rgb=rgb, alpha=alpha_img, depth=depth)


def render_into(tree, cam: Camera, frame: int, rgb, alpha, depth, opts: RenderOptions = RenderOptions(),
                cache=None, *, stream=None, sample_count=None, plan=None):
    """Render into caller-owned CUDA float32 tensors (rgb (H,W,3), alpha/depth (H,W); any may be None).

    The allocation-free device path used by the benchmark; asynchronous on
    the current (or given) stream.  ``sample_count``: optional CUDA int32
    (H, W) tensor receiving each pixel's consumed leaf samples (the
    reference's per-ray ``used`` count), from the same kernel.  ``plan``:
    a CameraPlan scheduling the kernel from the previous frames' costs
    (bitwise the same pixels).
    """
    frame = _frame_index(frame, tree)
    _check_frame(tree, frame)
    ref = next(x for x in (rgb, alpha, depth) if x is not None)
    dev = ref.device
    rep = replica(tree, dev)
    ch = _check_cache(cache, frame, rep)
    oc = opts.c_struct()
    cd = cam.desc()
    s = int(stream.cuda_stream) if stream is not None else stream_ptr(dev)
    planes = (rgb.data_ptr() if rgb is not None else None, alpha.data_ptr() if alpha is not None else None,
              depth.data_ptr() if depth is not None else None)
    if sample_count is not None:
        _native.check(_native.lib().vv_render_camera_counts(
            rep.handle, frame, ch, ctypes.byref(oc), ctypes.byref(cd), *planes, sample_count.data_ptr(), s))
        return
    if plan is not None:
        _native.check(_native.lib().vv_render_camera_planned(rep.handle, frame, ch, ctypes.byref(oc),
                                                             ctypes.byref(cd), None, plan._handle, *planes, 0, s))
        return
    _native.check(_native.lib().vv_render_camera(rep.handle, frame, ch, ctypes.byref(oc), ctypes.byref(cd),
                                                 *planes, s))


def render(tree, cam: Camera, frame: int, opts: RenderOptions = RenderOptions(), cache=None, *,
           out: str = "numpy", device=None) -> LayerImages:
    """Render one VOctree (render.py:236-240): rays + render + finalize in one kernel."""
    torch = require_cuda()
    frame = _frame_index(frame, tree)
    _check_frame(tree, frame)
    if cache is not None and getattr(cache, "frame", frame) != frame:
        raise ValueError(f"cache built for frame {cache.frame}, not {frame}")
    dev = torch_device(device)
    h, w = int(cam.height), int(cam.width)
    buf = torch.empty(5 * h * w, dtype=torch.float32, device=dev)
    rgb = buf[: 3 * h * w].view(h, w, 3)
    alpha = buf[3 * h * w: 4 * h * w].view(h, w)
    depth = buf[4 * h * w:].view(h, w)
    stream = torch.cuda.current_stream(dev)
    if out == "torch":
        render_into(tree, cam, frame, rgb, alpha, depth, opts, cache, plan=_stream_plan(dev, stream.cuda_stream))
        return LayerImages(rgb, alpha, depth)
    # to the host: each 64-row band copied (pinned, copy engine) as soon as
    # the kernel has stored it, overlapping the rest of the render
    rep = replica(tree, dev)
    ch = _check_cache(cache, frame, rep)
    host, a = _PINNED.get(5 * h * w)
    _native.check(_native.lib().vv_render_camera_to_host(rep.handle, frame, ch, ctypes.byref(opts.c_struct()),
                                                          ctypes.byref(cam.desc()), buf.data_ptr(), host.data_ptr(),
                                                          _stream_plan(dev, stream.cuda_stream)._handle,
                                                          stream.cuda_stream))
    stream.synchronize()
    return LayerImages(a[: 3 * h * w].reshape(h, w, 3), a[3 * h * w: 4 * h * w].reshape(h, w),
                       a[4 * h * w:].reshape(h, w))


def render_frames_into(tree, cam: Camera, frames, outs, opts: RenderOptions = RenderOptions(), *, stream=None):
    """Render 1..4 frames of ONE camera into caller-owned CUDA float32
    tensors ``outs[k] = (rgb, alpha, depth)`` (any may be None).

    The rays -- and so the octree walk and every ray's segment list -- do not
    depend on the frame, so the frames share one walk
    (vv_render_camera_multi); each frame has its own slice pass,
    accumulators and early termination, and its images are bitwise
    identical to ``render_into`` of that frame.  When the decode policy
    would decode per sample (a tree small on screen) the frames render one
    by one instead.  Asynchronous on the current (or given) stream.
    """
    torch = require_cuda()
    frames = [_frame_index(f, tree) for f in frames]
    if len(frames) != len(outs):
        raise ValueError(f"{len(frames)} frames but {len(outs)} outputs")
    if not 1 <= len(frames) <= 4:
        raise ValueError("1..4 frames per walk")
    for f in frames:
        _check_frame(tree, f)
    ref = next(x for o in outs for x in o if x is not None)
    dev = ref.device
    rep = replica(tree, dev)
    oc = opts.c_struct()
    cd = cam.desc()
    mode = ctypes.c_int32(0)
    _native.check(_native.lib().vv_camera_decode_mode(rep.handle, ctypes.byref(cd), ctypes.byref(oc),
                                                      ctypes.byref(mode)))
    if len(frames) == 1 or mode.value == 0:
        for f, o in zip(frames, outs):
            render_into(tree, cam, f, *o, opts, stream=stream)
        return
    ctx = torch.cuda.stream(stream) if stream is not None else torch.cuda.stream(torch.cuda.current_stream(dev))
    with ctx:
        # one payload pass (colour skipped where every frame is dark); freed
        # stream-ordered after the walk
        caches = build_frame_caches(tree, frames, device=dev, render_only=True)
        n = len(frames)
        P = ctypes.c_void_p

        def ptrs(j):
            return (P * n)(*[o[j].data_ptr() if o[j] is not None else None for o in outs])

        s = stream_ptr(dev)
        _native.check(_native.lib().vv_render_camera_multi_planned(
            rep.handle, n, (ctypes.c_int32 * n)(*frames), (P * n)(*[c._handle for c in caches]),
            ctypes.byref(oc), ctypes.byref(cd), ptrs(0), ptrs(1), ptrs(2), _stream_plan(dev, s, "multi")._handle, s))
        del caches


# frames per shared walk in playback (measured per-frame render-kernel cost
# at cfg2 for 1/2/3/4 frames: 0.76 / 0.49 / 0.39 / 0.38 ms; cfg3 2.03 / 1.13 /
# 0.87 / 0.78 ms); at n_max 3 the 4-frame kernel spills, so 3 there
PLAYBACK_GROUP = 4


def playback_group(tree) -> int:
    return PLAYBACK_GROUP if int(tree.n_max) <= 2 else 3


# render_sequence delivers every frame to the host: PCIe (41.5 MB per 1080p
# frame at ~56 GB/s) bounds it, and smaller groups pipeline the copies
# better (measured e2e 2,600 Mrays/s with 3 vs 2,260 with 4)
SEQUENCE_GROUP = 3

_PLAYBACK = {}
_PLAYBACK_MAX = 4  # cached playback states per device (concurrent sequences)


def _playback_state(torch, dev, n: int):
    """Per-device playback streams and double-buffered frame groups, kept across calls.

    Dedicated streams (the legacy default stream would serialise render and
    copy), and the SAME streams every call: the frame slices are allocated
    stream-ordered (cudaMallocAsync) on the render stream, and the pool only
    recycles a block on the stream that freed it -- a fresh stream per call
    re-maps ~1.9 GB of slice memory on its first frame (tens of ms).
    Several playbacks live at once (e.g. the two eyes of a stereo sequence,
    zipped) each get a cached state of their own (up to _PLAYBACK_MAX).
    """
    key = (dev.index if dev.index is not None else torch.cuda.current_device(), n)
    states = _PLAYBACK.get(key)
    if states is None:
        for k in [k for k in _PLAYBACK if k[0] == key[0]]:
            del _PLAYBACK[k]  # one resolution per device at a time
        states = _PLAYBACK[key] = []
    st = next((s for s in states if not s[3][0]), None)
    if st is None:
        comp, copy = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        with torch.cuda.stream(comp):
            bufs = [[torch.empty(n, dtype=torch.float32, device=dev) for _ in range(PLAYBACK_GROUP)]
                    for _ in range(2)]
        for grp in bufs:
            for b in grp:
                b.record_stream(copy)
        st = (comp, copy, bufs, [False])
        if len(states) < _PLAYBACK_MAX:
            states.append(st)  # else a private state, not cached
    st[0].wait_stream(st[1])  # an abandoned playback may still be copying out of the buffers
    return st


def render_sequence(tree, cam: Camera, frames, opts: RenderOptions = RenderOptions(), *, device=None):
    """Playback: render `frames` in order, yielding numpy LayerImages (fp32).

    Frames render in groups of SEQUENCE_GROUP (3) sharing one octree walk
    (render_frames_into: one camera, so the walk is frame-independent; each
    frame's images are bitwise identical to ``render``).  Double-buffered:
    group g renders on a per-device render stream (ordered after the
    caller's current stream) while group g-1's 20 B/pixel results are copied
    device->host on a side stream into pinned memory.  Each yielded frame is
    complete on the host.
    """
    torch = require_cuda()
    dev = torch_device(device)
    h, w = int(cam.height), int(cam.width)
    n = 5 * h * w
    caller = torch.cuda.current_stream(dev)
    comp, copy, bufs, busy = _playback_state(torch, dev, n)
    comp.wait_stream(caller)
    busy[0] = True
    try:
        yield from _playback(torch, tree, cam, frames, opts, comp, copy, bufs, h, w, n)
    finally:
        busy[0] = False


def _playback(torch, tree, cam, frames, opts, comp, copy, bufs, h, w, n):
    # warm the pinned pool for the frames in flight (two groups pending + the
    # caller's current and previous frame): a 41 MB cudaHostAlloc costs
    # 25-100 ms, so grow the pool once up front instead of stalling mid-sequence
    warm = [_PINNED.get(n) for _ in range(2 * PLAYBACK_GROUP + 2)]
    del warm
    copied = [None, None]
    pending = []

    def views(a):
        return LayerImages(a[: 3 * h * w].reshape(h, w, 3), a[3 * h * w: 4 * h * w].reshape(h, w),
                           a[4 * h * w:].reshape(h, w))

    def split(b):
        return (b[: 3 * h * w].view(h, w, 3), b[3 * h * w: 4 * h * w].view(h, w), b[4 * h * w:].view(h, w))

    frames = list(frames)
    G = min(SEQUENCE_GROUP, playback_group(tree))
    try:
        yield from _playback_groups(torch, tree, cam, frames, opts, comp, copy, bufs, n, G, copied, pending, views,
                                    split)
    finally:
        # a consumer that stops early (generator closed) drops the pinned
        # arrays of the groups still in flight: wait for their copies first,
        # or the pool could hand a buffer to another call while the DMA into
        # it is still running
        for ev, _ in pending:
            ev.synchronize()
        pending.clear()


def _sequence_groups(n_frames: int, G: int, first: int):
    """Frame groups of a playback: a short first group (the copy engine,
    which bounds delivery, starts sooner), then groups of G."""
    out, i = [], 0
    if first and n_frames:
        out.append((0, min(first, n_frames)))
        i = out[-1][1]
    while i < n_frames:
        out.append((i, min(i + G, n_frames)))
        i += G
    return out


# first playback group: 2 frames.  Steady state is PCIe-bound (0.73 ms per
# 1080p frame = the 41.5 MB copy alone); a short first group starts the
# copies sooner: 20-frame sequences 0.813 / 0.834 / 0.824 ms per frame with
# a first group of 2 / 1 / 3 (tools/seq_probe.py).  VV_SEQ_FIRST overrides.
SEQUENCE_FIRST = 2


def _playback_groups(torch, tree, cam, frames, opts, comp, copy, bufs, n, G, copied, pending, views, split):
    import os

    first = int(os.environ.get("VV_SEQ_FIRST", SEQUENCE_FIRST))
    for gi, (g0, g1) in enumerate(_sequence_groups(len(frames), G, first)):
        group = frames[g0:g1]
        b = gi % 2
        if copied[b] is not None:
            comp.wait_event(copied[b])  # group b's previous frames have left the device
        grp = bufs[b][:len(group)]
        with torch.cuda.stream(comp):
            render_frames_into(tree, cam, group, [split(x) for x in grp], opts)
        rendered = torch.cuda.Event()
        rendered.record(comp)
        copy.wait_event(rendered)
        arrs = []
        for x in grp:
            host, arr = _PINNED.get(n)
            with torch.cuda.stream(copy):
                host.copy_(x, non_blocking=True)
            arrs.append(arr)
        done = torch.cuda.Event()
        done.record(copy)
        copied[b] = done
        pending.append((done, arrs))
        if len(pending) > 1:
            ev, a = pending.pop(0)
            ev.synchronize()
            while a:  # hand frames over without keeping them (their pinned buffers recycle)
                yield views(a.pop(0))
    while pending:
        ev, a = pending.pop(0)
        ev.synchronize()
        while a:
            yield views(a.pop(0))


def composite_background(layer: LayerImages, bg) -> np.ndarray:
    """alpha * rgb + (1 - alpha) * bg (render.py:243-251)."""
    rgb = layer.rgb
    if hasattr(rgb, "cpu"):
        rgb = rgb.cpu().numpy()
    alpha = layer.alpha.cpu().numpy() if hasattr(layer.alpha, "cpu") else layer.alpha
    bg = np.asarray(bg, dtype=np.float64)
    if bg.ndim == 1:
        bg = np.broadcast_to(bg, rgb.shape)
    if bg.shape != rgb.shape:
        raise ValueError(f"background shape {bg.shape} != layer shape {rgb.shape}")
    a = np.asarray(alpha)[..., None]
    return a * rgb + (1.0 - a) * bg


def _seg_rays(tree, origins, dirs, dev):
    o, _ = _as_device_rays(origins, dev)
    d, _ = _as_device_rays(dirs, dev)
    return o, d


def count_segments(tree, origins, dirs, tmin: float = 0.0, tmax: float = 1e30, *, device=None) -> np.ndarray:
    """Leaf segments per ray without early stop (count_segments_kernel, kernels.py:313-335)."""
    torch = require_cuda()
    dev = torch_device(device)
    rep = replica(tree, dev)
    o, d = _seg_rays(tree, origins, dirs, dev)
    n = o.shape[0]
    cnt = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    _native.check(_native.lib().vv_count_segments(rep.handle, o.data_ptr(), d.data_ptr(), n, float(tmin),
                                                  float(tmax), cnt.data_ptr(), stream_ptr(dev)))
    return cnt[:n].cpu().numpy()


def collect_segments(tree, origins, dirs, tmin: float = 0.0, tmax: float = 1e30, *, device=None):
    """CSR of all leaf segments per ray (collect_segments_kernel, kernels.py:338-367).

    Returns (ray_start (n+1,), seg_leaf, seg_t0, seg_t1) numpy arrays.
    """
    torch = require_cuda()
    dev = torch_device(device)
    rep = replica(tree, dev)
    o, d = _seg_rays(tree, origins, dirs, dev)
    n = o.shape[0]
    cnt = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    lib = _native.lib()
    s = stream_ptr(dev)
    _native.check(lib.vv_count_segments(rep.handle, o.data_ptr(), d.data_ptr(), n, float(tmin), float(tmax),
                                        cnt.data_ptr(), s))
    start = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    if n:
        start[1:] = torch.cumsum(cnt[:n], 0)
    total = int(start[-1].item()) if n else 0
    leaf = torch.empty(max(total, 1), dtype=torch.int64, device=dev)
    t0 = torch.empty(max(total, 1), dtype=torch.float64, device=dev)
    t1 = torch.empty(max(total, 1), dtype=torch.float64, device=dev)
    if n:
        _native.check(lib.vv_collect_segments(rep.handle, o.data_ptr(), d.data_ptr(), n, float(tmin), float(tmax),
                                              start.data_ptr(), leaf.data_ptr(), t0.data_ptr(), t1.data_ptr(), s))
    return (start.cpu().numpy(), leaf[:total].cpu().numpy(), t0[:total].cpu().numpy(), t1[:total].cpu().numpy())
