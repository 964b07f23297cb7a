"""CPU tests: the C-ABI library's exported surface and host-only entry points,
the .voct codec, the BFS node-table builder, and the host halves of the
render/compose API (ports of the reference's own tests where they apply)."""

import math
import re
from pathlib import Path

import numpy as np
import pytest

from golden_util import load, tree_from
from paper_2202_06088_b200 import _native
from paper_2202_06088_b200.compose import Scene, SceneInstance, TimeMap, blend_layers, duplicate
from paper_2202_06088_b200.octree import (
    BadMagicError,
    ChecksumError,
    TruncatedStreamError,
    UnsupportedVersionError,
    VOctree,
)
from paper_2202_06088_b200.render import Camera, LayerImages, RenderOptions, composite_background, finalize_layer
from paper_2202_06088_b200.temporal import make_bump_bases

ROOT = Path(__file__).resolve().parent.parent


# ---------------------------------------------------------------- C ABI surface
def test_header_symbols_exported():
    header = (ROOT / "include" / "voxvid_b200.h").read_text()
    declared = set(re.findall(r"\b(vv_[a-z0-9_]+)\s*\(", header))
    assert declared == set(_native.EXPORTED_SYMBOLS)
    lib = _native.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.vv_abi_version() == 1


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_native_tables_bit_exact():
    g = load("tables")
    import ctypes

    for n_max in range(4):
        pn = np.zeros(64, np.int64)
        pl = np.zeros(64, np.int64)
        pnorm = np.zeros(64)
        k2p = np.zeros(256, np.int64)
        k2s = np.zeros(256, np.int64)
        shp = np.zeros(128)
        sizes = np.zeros(3, np.int32)
        _native.check(_native.lib().vv_basis_tables(n_max, pn.ctypes.data, pl.ctypes.data, pnorm.ctypes.data,
                                                    k2p.ctypes.data, k2s.ctypes.data, shp.ctypes.data,
                                                    sizes.ctypes.data))
        k, s, npairs = (int(v) for v in sizes)
        assert np.array_equal(pnorm[:npairs], g[f"n{n_max}_pair_norm"])
        assert np.array_equal(shp[:s], g[f"n{n_max}_sh_pref"])
        assert np.array_equal(k2p[:k], g[f"n{n_max}_k2pair"])
        assert np.array_equal(k2s[:k], g[f"n{n_max}_k2sh"])
    assert ctypes is not None


def test_native_crc32_matches_zlib():
    import zlib

    rng = np.random.default_rng(0)
    buf = rng.integers(0, 256, 100_003, dtype=np.uint8)
    assert _native.lib().vv_crc32(0, buf.ctypes.data, buf.size) == zlib.crc32(buf.tobytes())


# ---------------------------------------------------------------- .voct codec
def test_voct_bytes_bit_exact_with_reference():
    g = load("voct")
    tree = tree_from(g)
    assert tree.to_bytes() == g["voct"].tobytes()
    back = VOctree.from_bytes(g["voct"].tobytes())
    assert np.array_equal(back.node_child, tree.node_child)
    assert np.array_equal(back.leaf_coords, tree.leaf_coords)
    assert np.array_equal(back.leaf_data, tree.leaf_data)
    tree.ensure_edit_arrays()
    tree.edit_rgb[:] = g["edit_rgb"]
    tree.edit_t[:] = g["edit_t"]
    assert tree.to_bytes() == g["voct_edits"].tobytes()
    back = VOctree.from_bytes(g["voct_edits"].tobytes())
    assert np.array_equal(back.edit_rgb, g["edit_rgb"]) and np.array_equal(back.edit_t, g["edit_t"])


def test_voct_errors():
    data = load("voct")["voct"].tobytes()
    with pytest.raises(BadMagicError):
        VOctree.from_bytes(b"XXXX" + data[4:])
    bad_ver = bytearray(data)
    bad_ver[4] = 9
    with pytest.raises(UnsupportedVersionError):
        VOctree.from_bytes(bytes(bad_ver))
    with pytest.raises(TruncatedStreamError):
        VOctree.from_bytes(data[:2])
    corrupt = bytearray(data)
    corrupt[200] ^= 0xFF
    with pytest.raises(ChecksumError):
        VOctree.from_bytes(bytes(corrupt))


def test_voct_save_load(tmp_path):
    g = load("voct")
    tree = tree_from(g)
    p = tmp_path / "t.voct"
    tree.save(p)
    assert VOctree.load(p).to_bytes() == tree.to_bytes()


# ---------------------------------------------------------------- from_cells
@pytest.mark.parametrize("name", ["scalar_d2", "cache_d3", "edge_d4", "edits_d3", "nmax3"])
def test_from_cells_matches_reference_tables(name):
    g = load(name)
    t = VOctree.from_cells(g["tree_leaf_coords"], g["tree_leaf_data"], tree_from(g).bases, int(g["tree_n_max"]),
                           depth=int(g["tree_depth"]))
    assert np.array_equal(t.node_child, g["tree_node_child"])


def test_from_cells_errors():
    bases = make_bump_bases(4, 3)
    data = np.zeros((2, 21), np.float32)
    with pytest.raises(ValueError, match="duplicate"):
        VOctree.from_cells([[0, 0, 0], [0, 0, 0]], data, bases, 1, depth=2)
    with pytest.raises(ValueError, match="out of range"):
        VOctree.from_cells([[0, 0, 0], [4, 0, 0]], data, bases, 1, depth=2)
    empty = VOctree.from_cells(np.zeros((0, 3)), np.zeros((0, 21), np.float32), bases, 1, depth=2)
    assert empty.node_child.shape == (1, 8) and np.all(empty.node_child == -1)


def test_query_matches_linear_scan():
    g = load("edge_d4")
    tree = tree_from(g)
    rng = np.random.default_rng(2)
    boxes = [tree.leaf_box(i) for i in range(tree.n_leaves)]
    for _ in range(200):
        p = rng.random(3)
        hit = None
        for row, (blo, h) in enumerate(boxes):
            if all(blo[a] <= p[a] < blo[a] + h for a in range(3)):
                hit = row
                break
        got = tree.query(p)
        assert (got is None) == (hit is None)
        if got is not None:
            np.testing.assert_allclose(got[1][0], boxes[hit][0])


def test_upsample_doubles_depth():
    g = load("scalar_d2")
    tree = tree_from(g)
    up = tree.upsample()
    assert up.depth == tree.depth + 1 and up.n_leaves == 8 * tree.n_leaves


# ---------------------------------------------------------------- render host API
def test_camera_rays_unit_and_centered():
    cam = Camera.look_at([3.0, 1.0, 2.0], [0.5, 0.5, 0.5], width=9, height=9)
    o, d = cam.rays()
    np.testing.assert_allclose(np.linalg.norm(d, axis=1), 1.0, atol=1e-12)
    center = d[(9 // 2) * 9 + 9 // 2]
    to_target = np.array([0.5, 0.5, 0.5]) - cam.origin
    to_target /= np.linalg.norm(to_target)
    np.testing.assert_allclose(center, to_target, atol=1e-9)


def test_camera_rejects_skewed_rotation():
    c2w = np.eye(4)
    c2w[0, 1] = 0.01
    with pytest.raises(ValueError, match="orthonormal"):
        Camera(8, 8, 10, 10, 4, 4, c2w)


def test_finalize_layer_depth_scale():
    layer = finalize_layer(np.array([[0.5, 0.5, 0.5]]), np.array([1.0]), np.array([2.0]), (1, 1), RenderOptions(),
                           depth_scale=np.array([3.0]))
    assert layer.depth[0, 0] == pytest.approx(6.0)


def test_composite_background():
    layer = LayerImages(np.full((1, 1, 3), [1.0, 0.0, 0.0]), np.full((1, 1), 0.25), np.ones((1, 1)))
    np.testing.assert_allclose(composite_background(layer, np.array([0.0, 0.0, 1.0]))[0, 0], [0.25, 0.0, 0.75])
    with pytest.raises(ValueError, match="background shape"):
        composite_background(LayerImages(np.zeros((4, 4, 3)), np.zeros((4, 4)), np.zeros((4, 4))),
                             np.zeros((5, 5, 3)))


# ---------------------------------------------------------------- compose host API
def test_timemap_round_trip_and_laws():
    for expr in ("id", "shift(5)", "shift(5)|loop(30)|reverse", "clip(2,9)|speed(0.5)", "pause(7)"):
        assert str(TimeMap.parse(expr)) == expr
    rev, clip, loop = TimeMap.parse("reverse|reverse"), TimeMap.parse("clip(5,20)"), TimeMap.parse("loop(13)")
    for g in range(64):
        assert rev.apply(g, 64) == g
        assert 5 <= clip.apply(g, 64) <= 20
        assert loop.apply(g, 64) == loop.apply(g + 13, 64)
    assert TimeMap.parse("shift(4)").apply(10, 64) == 6
    assert TimeMap.parse("shift(4)").apply(1, 64) == 0
    with pytest.raises(ValueError, match="unknown timemap"):
        TimeMap.parse("warp(3)")
    with pytest.raises(ValueError, match="loop period"):
        TimeMap.parse("loop(0)")


def _alg1_scalar(layers):
    h, w = layers[0].shape
    out_i = layers[0].rgb.astype(float).copy()
    out_d = layers[0].depth.astype(float).copy()
    out_a = layers[0].alpha.astype(float).copy()
    for layer in layers[1:]:
        for y in range(h):
            for x in range(w):
                ai, di, a = float(layer.alpha[y, x]), float(layer.depth[y, x]), float(out_a[y, x])
                if di <= out_d[y, x]:
                    out_i[y, x] = ai * layer.rgb[y, x] + (1 - ai) * a * out_i[y, x]
                    out_d[y, x] = di
                else:
                    out_i[y, x] = a * out_i[y, x] + (1 - a) * ai * layer.rgb[y, x]
                out_a[y, x] = a + ai * (1 - a)
    return out_i, out_a, out_d


def test_blend_layers_alg1():
    rng = np.random.default_rng(42)
    layers = [LayerImages(rng.random((6, 5, 3)), rng.random((6, 5)), rng.uniform(1, 5, (6, 5))) for _ in range(3)]
    out = blend_layers(layers)
    ri, ra, rd = _alg1_scalar(layers)
    np.testing.assert_allclose(out.rgb, ri, atol=1e-12)
    np.testing.assert_allclose(out.alpha, ra, atol=1e-12)
    np.testing.assert_allclose(out.depth, rd, atol=1e-12)
    prod = np.prod([1.0 - l.alpha for l in layers], axis=0)
    np.testing.assert_allclose(out.alpha, 1.0 - prod, atol=1e-12)
    with pytest.raises(ValueError, match="resolution"):
        blend_layers([layers[0], LayerImages(np.zeros((7, 5, 3)), np.zeros((7, 5)), np.zeros((7, 5)))])


def test_duplicate_shares_tree():
    g = load("scalar_d2")
    base = SceneInstance(name="a", tree=tree_from(g))
    scene = Scene(instances=[base])
    before = scene.memory_report()
    for i in range(5):
        scene.instances.append(duplicate(base, name=f"d{i}"))
    after = scene.memory_report()
    assert after["payload_bytes"] == before["payload_bytes"] and after["trees"] == 1


def test_effective_affine_yaw():
    g = load("scalar_d2")
    inst = SceneInstance(name="a", tree=tree_from(g), yaw_rate=90.0)
    m = inst.effective_affine(1)
    c = np.array([0.5, 0.5, 0.5, 1.0])
    np.testing.assert_allclose(m @ c, c, atol=1e-12)
    assert math.isclose(m[0, 1], -1.0, abs_tol=1e-12)


def test_crc32_parallel_matches_zlib():
    """vv_crc32 splits >= 64 MB buffers across threads (zlib crc32_combine)."""
    import zlib

    rng = np.random.default_rng(3)
    buf = rng.integers(0, 256, (64 << 20) + 12345, dtype=np.uint8)
    lib = _native.lib()
    assert lib.vv_crc32(0, buf.ctypes.data, buf.size) == zlib.crc32(buf.tobytes()) & 0xFFFFFFFF
    head = 1000
    c0 = lib.vv_crc32(0, buf.ctypes.data, head)
    assert lib.vv_crc32(c0, buf[head:].ctypes.data, buf.size - head) == zlib.crc32(buf.tobytes()) & 0xFFFFFFFF


def test_voct_upload_error_classes():
    """vv_voct_upload validates like VOctree.from_bytes (octree.py:413-501);
    every check runs before any CUDA call."""
    import ctypes
    import struct
    import zlib

    from golden_util import load

    good = bytes(load("voct")["voct"])
    lib = _native.lib()

    def rc_of(data):
        b = np.frombuffer(data, dtype=np.uint8).copy()
        h = ctypes.c_void_p()
        return lib.vv_voct_upload(b.ctypes.data if b.size else None, b.size, 0, ctypes.byref(h), None)

    def recrc(body):
        return body + struct.pack("<I", zlib.crc32(body) & 0xFFFFFFFF)

    assert rc_of(good[:3]) == _native.VV_E_TRUNCATED
    assert rc_of(b"XXXX" + good[4:]) == _native.VV_E_MAGIC
    assert "bad magic b'XXXX'" in _native.last_error()
    assert rc_of(good[:6]) == _native.VV_E_TRUNCATED
    assert rc_of(good[:4] + struct.pack("<I", 9) + good[8:]) == _native.VV_E_VERSION
    assert rc_of(good[:40]) == _native.VV_E_TRUNCATED
    bad = bytearray(good)
    bad[200] ^= 1
    assert rc_of(bytes(bad)) == _native.VV_E_CHECKSUM
    body = good[:-4]
    assert rc_of(recrc(body + b"\0\0\0\0")) == _native.VV_E_FORMAT
    assert "trailing bytes" in _native.last_error()
    assert rc_of(recrc(body[:-100])) == _native.VV_E_TRUNCATED
    cube = bytearray(body)
    struct.pack_into("<d", cube, 28 + 3 * 8, 2.0)  # hi.x: not a cube
    assert rc_of(recrc(bytes(cube))) == _native.VV_E_FORMAT
    assert "not a cube" in _native.last_error()
