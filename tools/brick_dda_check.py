"""Compare the brick-DDA traversal prototype (tools/brick_dda_check.c) with the
oracle's collect_segments bit for bit, and report per-ray work."""
import ctypes
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))
from oracle import oracle  # noqa: E402
from paper_2202_06088_b200 import synthetic  # noqa: E402
from make_golden import edge_rays  # noqa: E402

lib = ctypes.CDLL(str(ROOT / "tools" / "_build" / "libbrick_dda.so"))
lib.bdc_build.restype = ctypes.c_void_p
lib.bdc_build.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int64]
lib.bdc_free.argtypes = [ctypes.c_void_p]
_P = ctypes.c_void_p
lib.bdc_collect.argtypes = [_P, _P, _P, ctypes.c_double, _P, _P, ctypes.c_int64, ctypes.c_double, ctypes.c_double] + \
    [_P] * 7


def check(tree, o, d, tmin=0.0, tmax=1e30, label="", limit=None):
    child = np.ascontiguousarray(tree.node_child, np.int32)
    b = lib.bdc_build(child.ctypes.data, child.shape[0], int(tree.depth), int(tree.n_leaves))
    start, leaf, t0, t1 = oracle.collect_segments(tree, o, d, tmin, tmax)
    n = o.shape[0]
    lo = np.ascontiguousarray(tree.bbox_lo, np.float64)
    tot = int(start[-1])
    gl, g0, g1 = np.zeros(max(tot, 1), np.int64), np.zeros(max(tot, 1)), np.zeros(max(tot, 1))
    cnt = np.zeros(n, np.int64)
    work = np.zeros((n, 3), np.int64)
    lib.bdc_collect(child.ctypes.data, b, lo.ctypes.data, float(tree.side), o.ctypes.data, d.ctypes.data, n,
                    float(tmin), float(tmax), start.ctypes.data, gl.ctypes.data, g0.ctypes.data, g1.ctypes.data,
                    cnt.ctypes.data, work.ctypes.data, None if limit is None else limit.ctypes.data)
    lib.bdc_free(b)
    ok = np.array_equal(cnt, np.diff(start)) and np.array_equal(gl[:tot], leaf) and \
        np.array_equal(g0[:tot].view(np.int64), t0.view(np.int64)) and \
        np.array_equal(g1[:tot].view(np.int64), t1.view(np.int64))
    print(f"{label:28s} rays {n:7d} segs {tot:9d} equal={ok}  node steps {work[:, 0].mean():.2f} "
          f"bricks {work[:, 1].mean():.2f} dda steps {work[:, 2].mean():.2f}")
    return ok, work, start


if __name__ == "__main__":
    rng = np.random.default_rng(7)
    allok = True
    for depth in (1, 2, 3, 4, 5, 6):
        tree = synthetic.shell_tree(depth, 1, 4, depth)
        o, d = edge_rays(rng, 3000)
        ok, _, _ = check(tree, o, d, label=f"shell depth {depth} edge rays")
        allok &= ok
        ok, _, _ = check(tree, o, d, 0.3, 1.7, label=f"shell depth {depth} tmin/tmax")
        allok &= ok
    tree = synthetic.shell_tree(9, 2, 30, 0)
    o, d = edge_rays(rng, 20000)
    ok, _, _ = check(tree, o, d, label="cfg2 tree edge rays")
    allok &= ok
    cam = synthetic.bench_camera(1920, 1080)
    co, cd = cam.rays()
    idx = rng.choice(len(co), 200000, replace=False)
    ok, work, start = check(tree, co[idx], cd[idx], label="cfg2 camera rays")
    allok &= ok
    hit = np.diff(start) > 0
    print("hit rays: node steps %.2f bricks %.2f dda steps %.2f segs %.2f" % (
        work[hit, 0].mean(), work[hit, 1].mean(), work[hit, 2].mean(), np.diff(start)[hit].mean()))
    out = oracle.render_rays(tree, co[idx], cd[idx], 5)
    used = np.ascontiguousarray(out["used"], np.int64)
    used[used == 0] = -1
    _, work, _ = check(tree, co[idx], cd[idx], label="cfg2 camera, early stop", limit=used)
    h = out["alpha"] > 0
    print("early-stop hit rays: node steps %.2f bricks %.2f dda steps %.2f used %.2f" % (
        work[h, 0].mean(), work[h, 1].mean(), work[h, 2].mean(), out["used"][h].mean()))
    print("ALL EQUAL" if allok else "MISMATCH")
