"""bench.py end to end on the GPU: every BASELINE config emits one correctly
labelled JSON line (roofline, cpu_baseline, e2e), and the N > 1 path runs
under torchrun with two ranks sharing this GPU (VV_BENCH_FUNCTIONAL_GLOO=1:
gloo collectives, numbers not measurements) -- frame split into row bands
stored into rank 0's planes through CUDA IPC."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402

pytestmark = pytest.mark.gpu


def _line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-3000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("config", [3, 4, 5])
def test_bench_config_lines(cuda, config):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--config", str(config), "--steps", "3",
                        "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    assert d["metric"] == bench.METRIC and d["unit"] == bench.UNIT
    assert d["config"]["workload"] == bench.CONFIGS[config]["workload"] and d["config"]["config"] == config
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["scaling"] == "weak"
    ro = d["roofline"]
    assert ro["bound"] == "hbm" and 0 < ro["frac"] and ro["kernel"] in ("k_render_camera", "k_render_scene_lean")
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["clocks"]["samples"] >= 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_torchrun_two_ranks(cuda):
    env = dict(os.environ, VV_BENCH_FUNCTIONAL_GLOO="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--no-cpu"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["workload"] == bench.WORKLOAD
    assert "row bands" in d["config"]["parallelism"]
    assert d["frame_sharded"]["scaling"] == "weak" and d["frame_sharded"]["value"] > 0
    assert d["playback"]["value"] > 0 and d["e2e"]["value"] > 0
