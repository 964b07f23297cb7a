"""ctypes binding of libvoxvid_b200.so (the C ABI in include/voxvid_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_2202_06088_b200/csrc``).  There is no fallback: if the shared library
is missing, or a compute call is made without a CUDA device, the call fails
loudly.  Loading the library itself works on a CPU-only host (the CUDA
runtime is statically linked), which the CPU test-suite uses to check the
exported symbols and the host-only entry points.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

__all__ = [
    "LIB_PATH",
    "lib",
    "check",
    "VVError",
    "TreeDesc",
    "VoctInfo",
    "RenderOpts",
    "CameraDesc",
    "InstanceDesc",
    "LightDesc",
    "EXPORTED_SYMBOLS",
]

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libvoxvid_b200.so"
if os.environ.get("VV_LIB_PATH"):  # A/B experiments with alternative in-tree builds (tools/build_variants.sh)
    LIB_PATH = Path(os.environ["VV_LIB_PATH"]).resolve()

VV_OK = 0
VV_E_INVALID = -1
VV_E_CUDA = -2
VV_E_NOMEM = -3
VV_E_UNSUPPORTED = -4
VV_E_FORMAT = -5
VV_E_MAGIC = -6
VV_E_VERSION = -7
VV_E_TRUNCATED = -8
VV_E_CHECKSUM = -9

# every entry point declared in include/voxvid_b200.h
EXPORTED_SYMBOLS = (
    "vv_abi_version",
    "vv_last_error",
    "vv_device_count",
    "vv_debug_checks",
    "vv_basis_tables",
    "vv_tree_upload",
    "vv_tree_bind",
    "vv_tree_free",
    "vv_tree_info",
    "vv_tree_dark_fraction",
    "vv_tree_visible_count",
    "vv_profile_split_event",
    "vv_tree_visible_bits",
    "vv_tree_leaf_order",
    "vv_slice_build",
    "vv_slice_free",
    "vv_slice_export",
    "vv_slice_frame",
    "vv_render_rays",
    "vv_render_rays_visits",
    "vv_render_camera",
    "vv_render_camera_counts",
    "vv_render_camera_region",
    "vv_camera_block_shape",
    "vv_render_camera_to_host",
    "vv_camera_plan_create",
    "vv_camera_plan_free",
    "vv_render_camera_planned",
    "vv_render_camera_tiles",
    "vv_unpack_tiles",
    "vv_render_camera_tiles_direct",
    "vv_ipc_alloc",
    "vv_ipc_open",
    "vv_ipc_close",
    "vv_ipc_free",
    "vv_render_scene",
    "vv_scene_decode_modes",
    "vv_render_scene_joint",
    "vv_render_scene_planned",
    "vv_render_camera_multi",
    "vv_render_camera_multi_planned",
    "vv_slice_build_multi",
    "vv_slice_build_frames",
    "vv_slice_build_visible",
    "vv_camera_decode_mode",
    "vv_shadow_blur",
    "vv_scene_lighting",
    "vv_scene_lighting_ex",
    "vv_count_segments",
    "vv_collect_segments",
    "vv_termination_leaves",
    "vv_tree_set_edits",
    "vv_voct_parse_nodes",
    "vv_voct_encode_nodes",
    "vv_crc32",
    "vv_voct_upload",
)


class VVError(RuntimeError):
    """A failure reported by the native library (CUDA or unsupported input)."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


class TreeDesc(ctypes.Structure):
    _fields_ = [
        ("depth", ctypes.c_int32),
        ("n_max", ctypes.c_int32),
        ("frames", ctypes.c_int32),
        ("coeff_count", ctypes.c_int32),
        ("n_internal", ctypes.c_int64),
        ("n_leaves", ctypes.c_int64),
        ("bbox_lo", ctypes.c_double * 3),
        ("side", ctypes.c_double),
        ("node_child", ctypes.c_void_p),
        ("leaf_data", ctypes.c_void_p),
        ("basis_a", ctypes.c_void_p),
        ("basis_b", ctypes.c_void_p),
        ("edit_rgb", ctypes.c_void_p),
        ("edit_t", ctypes.c_void_p),
    ]


class VoctInfo(ctypes.Structure):
    """vv_voct_info: header of an uploaded .voct stream."""

    _fields_ = [
        ("version", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("depth", ctypes.c_int32),
        ("frames", ctypes.c_int32),
        ("coeff_count", ctypes.c_int32),
        ("basis_count", ctypes.c_int32),
        ("n_max", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("n_internal", ctypes.c_int64),
        ("n_leaves", ctypes.c_int64),
        ("bbox_lo", ctypes.c_double * 3),
        ("side", ctypes.c_double),
    ]


class RenderOpts(ctypes.Structure):
    _fields_ = [
        ("early_stop", ctypes.c_double),
        ("far_plane", ctypes.c_double),
        ("alpha_floor", ctypes.c_double),
        ("edit_weight", ctypes.c_double),
        ("tmin", ctypes.c_double),
        ("tmax", ctypes.c_double),
        ("frame_slice", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class CameraDesc(ctypes.Structure):
    _fields_ = [
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
        ("fx", ctypes.c_double),
        ("fy", ctypes.c_double),
        ("cx", ctypes.c_double),
        ("cy", ctypes.c_double),
        ("c2w", ctypes.c_double * 16),
    ]


class LightDesc(ctypes.Structure):
    """vv_light (include/voxvid_b200.h)."""

    _fields_ = [
        ("position", ctypes.c_double * 3),
        ("ground_plane", ctypes.c_double * 4),
        ("shadow_strength", ctypes.c_double),
        ("falloff_r0", ctypes.c_double),
        ("falloff_min_scale", ctypes.c_double),
        ("cast_shadows", ctypes.c_int32),
        ("falloff_enabled", ctypes.c_int32),
        ("shadow_map", ctypes.c_void_p),
        ("shadow_res", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("w2c", ctypes.c_double * 12),
        ("fx", ctypes.c_double),
        ("fy", ctypes.c_double),
        ("cx", ctypes.c_double),
        ("cy", ctypes.c_double),
    ]


class InstanceDesc(ctypes.Structure):
    _fields_ = [
        ("tree", ctypes.c_void_p),
        ("frame", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("pose", ctypes.c_double * 16),
        ("inv", ctypes.c_double * 16),
    ]


VV_SLICE_RENDER_ONLY = 1
VV_SLICE_VISIBLE = 2
_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_D = ctypes.c_double

_SIGNATURES = {
    "vv_abi_version": (ctypes.c_int, []),
    "vv_last_error": (ctypes.c_char_p, []),
    "vv_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "vv_debug_checks": (ctypes.c_int, [_I32, _P, _P, _P, _P, _I32]),
    "vv_basis_tables": (ctypes.c_int, [ctypes.c_int, _P, _P, _P, _P, _P, _P, _P]),
    "vv_tree_upload": (ctypes.c_int, [ctypes.POINTER(TreeDesc), ctypes.c_int, ctypes.POINTER(_P)]),
    "vv_tree_bind": (ctypes.c_int, [ctypes.POINTER(TreeDesc), ctypes.c_int, ctypes.POINTER(_P)]),
    "vv_tree_free": (ctypes.c_int, [_P]),
    "vv_tree_info": (ctypes.c_int, [_P, _P, _P, _P, _P, _P]),
    "vv_tree_dark_fraction": (ctypes.c_int, [_P, _P]),
    "vv_tree_visible_count": (ctypes.c_int, [_P, _P, _P, _P]),
    "vv_profile_split_event": (ctypes.c_int, [_P]),
    "vv_tree_visible_bits": (ctypes.c_int, [_P, _P, ctypes.c_int64, _P]),
    "vv_tree_leaf_order": (ctypes.c_int, [_P, _P]),
    "vv_slice_build": (ctypes.c_int, [_P, _I32, _P, ctypes.POINTER(_P)]),
    "vv_slice_free": (ctypes.c_int, [_P]),
    "vv_slice_export": (ctypes.c_int, [_P, _P, _P, _P]),
    "vv_slice_frame": (ctypes.c_int, [_P, _P]),
    "vv_render_rays": (
        ctypes.c_int,
        [_P, _I32, _P, ctypes.POINTER(RenderOpts), _P, _P, _I64, _P, _P, _P, _P, _P, _P, _P],
    ),
    "vv_render_rays_visits": (
        ctypes.c_int,
        [_P, _I32, _P, ctypes.POINTER(RenderOpts), _P, _P, _I64, _P, _P, _P],
    ),
    "vv_render_camera": (
        ctypes.c_int,
        [_P, _I32, _P, ctypes.POINTER(RenderOpts), ctypes.POINTER(CameraDesc), _P, _P, _P, _P],
    ),
    "vv_render_camera_counts": (
        ctypes.c_int,
        [_P, _I32, _P, ctypes.POINTER(RenderOpts), ctypes.POINTER(CameraDesc), _P, _P, _P, _P, _P],
    ),
    "vv_render_camera_region": (
        ctypes.c_int,
        [_P, _I32, _P, ctypes.POINTER(RenderOpts), ctypes.POINTER(CameraDesc), _P, _P, _P, _P, _P, _I32, _P],
    ),
    "vv_camera_block_shape": (ctypes.c_int, [_P, _P]),
    "vv_render_camera_to_host": (
        ctypes.c_int, [_P, _I32, _P, ctypes.POINTER(RenderOpts), ctypes.POINTER(CameraDesc), _P, _P, _P, _P]),
    "vv_camera_plan_create": (ctypes.c_int, [_I32, ctypes.POINTER(_P)]),
    "vv_camera_plan_free": (ctypes.c_int, [_P]),
    "vv_render_camera_planned": (
        ctypes.c_int,
        [_P, _I32, _P, ctypes.POINTER(RenderOpts), ctypes.POINTER(CameraDesc), _P, _P, _P, _P, _P, _I32, _P],
    ),
    "vv_render_camera_tiles": (
        ctypes.c_int,
        [_P, _I32, _P, ctypes.POINTER(RenderOpts), ctypes.POINTER(CameraDesc), _I32, _I32, _I32, _P, _P],
    ),
    "vv_unpack_tiles": (ctypes.c_int, [_P, _I32, _I32, _I32, _I32, _P, _P, _P, _P]),
    "vv_render_camera_tiles_direct": (
        ctypes.c_int,
        [_P, _I32, _P, ctypes.POINTER(RenderOpts), ctypes.POINTER(CameraDesc), _I32, _I32, _I32, _P, _P, _P,
         _I32, _P],
    ),
    "vv_ipc_alloc": (ctypes.c_int, [_I32, ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p), _P]),
    "vv_ipc_open": (ctypes.c_int, [_I32, _P, ctypes.POINTER(ctypes.c_void_p)]),
    "vv_ipc_close": (ctypes.c_int, [_I32, _P]),
    "vv_ipc_free": (ctypes.c_int, [_I32, _P]),
    "vv_camera_decode_mode": (ctypes.c_int, [_P, _P, _P, _P]),
    "vv_slice_build_multi": (ctypes.c_int, [_P, ctypes.c_int32, _P, _P, _P]),
    "vv_slice_build_frames": (ctypes.c_int, [_P, ctypes.c_int32, _P, ctypes.c_int32, _P, _P]),
    "vv_slice_build_visible": (ctypes.c_int, [_P, ctypes.c_int32, _P, _P, _P]),
    "vv_render_camera_multi": (ctypes.c_int, [_P, ctypes.c_int32, _P, _P, _P, _P, _P, _P, _P, _P]),
    "vv_render_camera_multi_planned": (ctypes.c_int, [_P, ctypes.c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "vv_shadow_blur": (ctypes.c_int, [_P, ctypes.c_int32, _P, ctypes.c_int32, _P, _P, _P]),
    "vv_scene_lighting": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, ctypes.c_int32, _P, _P]),
    "vv_scene_lighting_ex": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, ctypes.c_int32, _P, _P, _P]),
    "vv_render_scene": (
        ctypes.c_int,
        [ctypes.POINTER(InstanceDesc), _I32, ctypes.POINTER(RenderOpts), ctypes.POINTER(CameraDesc),
         _P, _P, _P, _P, _P],
    ),
    "vv_render_scene_joint": (
        ctypes.c_int,
        [ctypes.POINTER(InstanceDesc), _I32, ctypes.POINTER(RenderOpts), ctypes.POINTER(CameraDesc),
         _P, _P, _P, _P, _P],
    ),
    "vv_render_scene_planned": (
        ctypes.c_int,
        [ctypes.POINTER(InstanceDesc), _I32, ctypes.POINTER(RenderOpts), ctypes.POINTER(CameraDesc),
         _P, _P, _P, _P, _P, _P],
    ),
    "vv_scene_decode_modes": (
        ctypes.c_int, [ctypes.POINTER(InstanceDesc), _I32, _P, ctypes.POINTER(CameraDesc), _P]),
    "vv_count_segments": (ctypes.c_int, [_P, _P, _P, _I64, _D, _D, _P, _P]),
    "vv_collect_segments": (ctypes.c_int, [_P, _P, _P, _I64, _D, _D, _P, _P, _P, _P, _P]),
    "vv_termination_leaves": (ctypes.c_int, [_P, ctypes.c_int32, _P, _P, _P, _I64, _D, _P, _P]),
    "vv_tree_set_edits": (ctypes.c_int, [_P, _P, _P]),
    "vv_voct_parse_nodes": (ctypes.c_int, [_P, ctypes.c_size_t, _I64, _P, ctypes.POINTER(ctypes.c_size_t)]),
    "vv_voct_encode_nodes": (ctypes.c_int, [_P, _I64, _P, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    "vv_crc32": (ctypes.c_uint32, [ctypes.c_uint32, _P, ctypes.c_size_t]),
    "vv_voct_upload": (ctypes.c_int, [_P, ctypes.c_size_t, ctypes.c_int, _P, _P]),
}

_lib = None
_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """The loaded native library; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"native library {LIB_PATH} is missing: run __graft_entry__.build() "
                    "(there is no CPU fallback)"
                )
            handle = ctypes.CDLL(os.fspath(LIB_PATH))
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(handle, name, None)
                if fn is None:
                    if os.environ.get("VV_LIB_PATH"):  # an older A/B build: entry points it predates stay unbound
                        continue
                    raise ImportError(f"{LIB_PATH} does not export {name}")
                fn.restype = res
                fn.argtypes = args
            if handle.vv_abi_version() != 1:
                raise ImportError("libvoxvid_b200 ABI version mismatch")
            _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().vv_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int) -> None:
    """Raise the reference's exception type for a failed native call.

    Invalid arguments (frame out of range, cache/frame mismatch, ...) raise
    ValueError with the reference's message, as render.py does
    (render.py:165-167, 188-190); everything else raises VVError.
    """
    if rc == VV_OK:
        return
    msg = last_error()
    if rc == VV_E_INVALID:
        raise ValueError(msg)
    raise VVError(rc, msg)
