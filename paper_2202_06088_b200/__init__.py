"""voxvid_b200 -- B200-native VOctree renderer (NeuVV, arXiv 2202.06088).

Drop-in for the render path of the reference package ``voxvid``: the same
module-level names (VOctree.load, render, render_rays, build_frame_cache,
Camera, RenderOptions, LayerImages, Scene, SceneInstance, render_scene, ...)
backed by hand-written sm_100a CUDA kernels in libvoxvid_b200.so.
"""

from .compose import (
    Light,
    Scene,
    SceneInstance,
    ShadowMap,
    TimeMap,
    blend_layers,
    duplicate,
    falloff_pass,
    paint,
    render_instance,
    render_scene,
    render_scene_sequence,
    shadow_pass,
    termination_leaves,
)
from .device import DeviceTree, load_device
from .octree import (
    BadMagicError,
    ChecksumError,
    RaySegment,
    TruncatedStreamError,
    UnsupportedVersionError,
    VOctree,
    VoctError,
)
from .render import (
    Camera,
    CameraPlan,
    FrameSlice,
    LayerImages,
    RenderOptions,
    build_frame_cache,
    build_frame_caches,
    collect_segments,
    composite_background,
    count_segments,
    finalize_layer,
    render,
    render_frames_into,
    render_into,
    render_sequence,
    render_ray_visits,
    render_rays,
)
from .temporal import TemporalBases, make_bump_bases

__all__ = [
    "VOctree", "DeviceTree", "load_device", "RaySegment", "VoctError", "BadMagicError", "UnsupportedVersionError", "TruncatedStreamError",
    "ChecksumError", "Camera", "LayerImages", "RenderOptions", "FrameSlice", "CameraPlan", "render", "render_into", "render_frames_into", "render_sequence",
    "render_rays", "render_ray_visits", "finalize_layer", "composite_background", "build_frame_cache", "build_frame_caches",
    "count_segments", "collect_segments", "TimeMap", "SceneInstance", "Scene", "Light", "blend_layers",
    "render_instance", "render_scene", "render_scene_sequence", "duplicate", "paint", "termination_leaves", "ShadowMap", "shadow_pass",
    "falloff_pass", "TemporalBases",
    "make_bump_bases",
]
