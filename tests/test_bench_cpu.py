"""bench.py's reference arm on CPU: the JSON-line contract the driver reads.

The reference arm runs on host cores only (the reference's numba renderer
from baseline/_ref, or the C oracle port with ``--port``), so its contract is
checkable here: one JSON line from rank 0 with the ours-arm metric, unit,
workload and direction, the W warm-up frames rendered untimed, and nothing
printed by the other ranks.
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def _run(extra_env=None, *args):
    env = dict(os.environ, **(extra_env or {}))
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", *args],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return [ln for ln in r.stdout.splitlines() if ln.startswith("{")]


@pytest.mark.timeout(600)
def test_reference_arm_json_contract():
    lines = _run(None, "--port", "--steps", "1", "--warmup", "0")
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference"
    assert line["metric"] == bench.METRIC and line["unit"] == bench.UNIT
    assert line["higher_is_better"] is True
    assert line["config"]["workload"] == bench.WORKLOAD
    assert line["warmup"] == 3 and line["config"]["warmup_frames"] == [0, 1, 2]  # W raised to 3, run untimed
    assert line["config"]["frames"] == [3] and line["steps"] == 1
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["value"] == line["value"] and cb["cores"] >= 1


def test_reference_arm_other_ranks_silent():
    assert _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, "--port", "--steps", "1") == []
