"""bench.py host logic on CPU: the self-spawn of N ranks (the driver's `python bench.py --gpus N`
form) and the reference arm's JSON line (what it actually ran)."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def test_spawn_ranks_builds_torchrun_command(monkeypatch):
    import bench
    seen = {}

    def fake_call(cmd, env=None):
        seen["cmd"], seen["env"] = cmd, env
        return 0
    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    monkeypatch.delenv("VBD_DIST_BACKEND", raising=False)
    args = bench.parse()
    assert bench.spawn_ranks(args) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"]
    # no GPU here: fewer GPUs than ranks -> the ranks share devices over a gloo control plane
    assert seen["env"]["VBD_DIST_BACKEND"] == "gloo"
    assert seen["env"]["NCCL_DEBUG"] == "INFO"


def test_reference_arm_reports_what_it_ran():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["impl"] == "reference"
    assert line["steps"] == 2 and line["warmup"] == 1
    assert line["extrapolated"] is True
    cb = line["cpu_baseline"]
    assert cb["sample_steps"] == 2 and cb["sample_vertices"] == 4961
    assert "1_threads" in cb["threads_probe"] and cb["cpu_model"]
    # ms_per_step is the sample's own step time, consistent with value
    vit = cb["sample_vertices"] * line["config"]["n_max"]
    assert abs(vit / (line["ms_per_step"] / 1e3) / line["value"] - 1) < 1e-9
    assert line["e2e"]["h2d_bytes_per_step"] == 0
