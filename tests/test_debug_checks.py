"""The bounds-checked build (compute-sanitizer is not available on this GPU
pool): `make debug` builds _lib/debug/libvoxvid_b200.so with device-side
checks of node rows, stack slots, segment-queue fill, leaf rows and slice
chunk ids in the render kernels.  Here the parity suites run against it in
a subprocess and every test must leave zero violations (tests/conftest.py),
and the cfg1 sanitizer workload (tools/sanitize_cfg1.py) runs clean."""

import ctypes
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
DEBUG_LIB = ROOT / "paper_2202_06088_b200" / "_lib" / "debug" / "libvoxvid_b200.so"

pytestmark = pytest.mark.gpu


def _env():
    if not DEBUG_LIB.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "paper_2202_06088_b200" / "csrc"), "debug"], check=True)
    return dict(os.environ, VV_LIB_PATH=str(DEBUG_LIB), VV_DEBUG_EXPECT_CLEAN="1",
                PYTHONPATH=str(ROOT) + os.pathsep + os.environ.get("PYTHONPATH", ""))


def test_parity_suites_under_bounds_checks(cuda):
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", "-m", "gpu",
                        "tests/test_gpu_parity.py", "tests/test_node_mask.py", "tests/test_tiles_gpu.py",
                        "tests/test_joint.py", "tests/test_paint.py", "tests/test_visible_set.py",
                        "tests/test_schedule_fuzz.py", "-k", "not full_size and not cfg3"],
                       cwd=ROOT, env=_env(), capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]


def test_sanitize_workload_clean(cuda):
    code = ("import runpy, ctypes; runpy.run_path('tools/sanitize_cfg1.py'); "
            "from paper_2202_06088_b200 import _native; "
            "en, n, c = ctypes.c_int32(), ctypes.c_uint32(), ctypes.c_uint32(); "
            "_native.check(_native.lib().vv_debug_checks(0, ctypes.byref(en), ctypes.byref(n), ctypes.byref(c), None, 0)); "
            "print('DEBUG', en.value, n.value, c.value)")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=_env(), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "SANITIZE_WORKLOAD_OK" in r.stdout and "DEBUG 1 0 0" in r.stdout, r.stdout[-2000:]


STACK_PROBE = r"""
import ctypes, sys
import numpy as np
import paper_2202_06088_b200 as vv
from paper_2202_06088_b200 import _native
out = []
for depth in (3, 4, 5, 6):
    res = 1 << depth
    coords = np.argwhere(np.ones((res, res, res), bool))  # dense: every sibling is kept
    data = np.zeros((len(coords), 2 * 3 + 3 * 5), np.float32)
    tree = vv.VOctree.from_cells(coords, data, vv.make_bump_bases(2, 3), 1, depth=depth)
    # near-diagonal rays entering at a corner: at every level the three
    # mid-plane crossings are distinct, so each node pushes three siblings
    d = np.array([[1.0, 1.0 + 1e-3, 1.0 + 2e-3], [1.0 + 2e-3, 1.0, 1.0 + 1e-3], [1.0 + 1e-3, 1.0 + 2e-3, 1.0]])
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o = np.array([-0.5, -0.5, -0.5]) - 0.0 * d
    o = np.repeat(o[None], 3, axis=0)
    en, n, c, hw = ctypes.c_int32(), ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
    _native.check(_native.lib().vv_debug_checks(0, None, None, None, None, 1))
    vv.render_rays(tree, o, d, 0, vv.RenderOptions(early_stop=0.0, frame_slice="per_sample"), stats=True)
    _native.check(_native.lib().vv_debug_checks(0, ctypes.byref(en), ctypes.byref(n), ctypes.byref(c),
                                                ctypes.byref(hw), 0))
    out.append((depth, int(hw.value), int(n.value)))
print("STACK", out)
"""


def test_stack_bound_reached_and_never_exceeded(cuda):
    """The traversal stack holds at most 3 (depth - 1) slots (vv_device.cuh
    stack_cap): near-diagonal rays through dense trees fill it exactly, and
    the bounds-checked build records no overflow."""
    r = subprocess.run([sys.executable, "-c", STACK_PROBE], cwd=ROOT, env=_env(), capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("STACK")][0]
    res = eval(line[len("STACK "):])
    for depth, high, viol in res:
        assert viol == 0, (depth, viol)
        assert high == 3 * (depth - 1), (depth, high)
