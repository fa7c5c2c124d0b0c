"""bench.py --gpus N launches N ranks itself when started without torchrun
(CPU: the reference arm under gloo; GPU: the z-slab arm, 2 ranks sharing the
box's GPU through host barriers), and refuses a WORLD_SIZE that disagrees with
--gpus."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _last_json(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


def _env():
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    return e


def test_world_size_must_match_gpus():
    e = _env()
    e["WORLD_SIZE"] = "1"
    p = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--impl", "reference"], env=e,
                       capture_output=True, text=True, timeout=120)
    assert p.returncode == 2
    assert "WORLD_SIZE=1 but --gpus 2" in p.stdout


def test_reference_arm_spawns_ranks_and_rank0_prints():
    p = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--ref-cells", "16"], env=_env(), capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    line = _last_json(p.stdout)
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert sum(1 for ln in p.stdout.splitlines() if ln.startswith("{")) == 1  # rank 0 only


@pytest.mark.gpu
def test_bench_gpus2_runs_slab_path_on_one_box():
    p = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--cells", "64", "--steps", "2", "--warmup", "1",
                        "--solve", "0", "--mixed", "0", "--no-cpu"], env=_env(), capture_output=True, text=True,
                       timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    line = _last_json(p.stdout)
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert "z-slab x2" in line["config"]["parallelism"]
    assert [r["rank"] for r in line["ipc_ranks_attached"]] == [0, 1]
    assert line["value"] > 0
