"""The C ABI from a non-Python host: examples/render_voct.cpp loads a .voct
with vv_voct_upload and renders with vv_render_camera."""
import os
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
EXE = ROOT / "examples" / "render_voct"


def _build():
    subprocess.run(["make", "-s", "-C", str(ROOT / "examples")], check=True, capture_output=True)


def test_example_links():
    _build()
    out = subprocess.run(["ldd", str(EXE)], capture_output=True, text=True).stdout
    assert "libvoxvid_b200.so" in out and "not found" not in out


@pytest.mark.gpu
def test_example_matches_python_render(cuda, tmp_path):
    import paper_2202_06088_b200 as vv
    from paper_2202_06088_b200 import synthetic

    _build()
    tree = synthetic.shell_tree(depth=7, n_max=1, frames=16, seed=0)
    path = tmp_path / "shell.voct"
    tree.save(path)
    w, h, frame = 96, 64, 5
    res = subprocess.run([str(EXE), str(path), str(frame), str(w), str(h), str(tmp_path / "out.ppm"),
                          str(tmp_path / "out.f32")], capture_output=True, text=True, env=dict(os.environ))
    assert res.returncode == 0, res.stderr
    raw = np.fromfile(tmp_path / "out.f32", dtype=np.float32).reshape(h, w, 5)
    layer = vv.render(tree, synthetic.bench_camera(w, h), frame)
    assert np.abs(raw[..., :3] - layer.rgb).max() < 1e-4
    assert np.abs(raw[..., 3] - layer.alpha).max() < 1e-4
    hit = layer.alpha >= 1e-3
    assert hit.any() and np.abs(raw[..., 4][hit] - layer.depth[hit]).max() < 1e-4
    assert (tmp_path / "out.ppm").read_bytes().startswith(b"P6")
