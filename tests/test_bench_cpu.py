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


def test_layout_bytes_model_per_layout():
    """roofline.frac's numerator for the three kernels that carry a layout:
    K1T (8 B slots), K1T-X (8 B slots + 36 B of streamed rows per slot) and the global K1
    (entry_bytes per entry + CSR offset)."""
    import types
    import bench
    base = dict(num_vertices=1000, num_solved=900, num_colors=4, color_count=[250, 250, 250, 250],
                tile_slots=20000, tile_nbr_refs=5000, tiles=16, num_entries=18000, entry_bytes=48)
    other = sum(16 * (1000 - 250) for _ in range(4))
    k1t = types.SimpleNamespace(layout=1, **base)
    k1tx = types.SimpleNamespace(layout=0, **base)
    glob = types.SimpleNamespace(layout=0, **dict(base, tiles=0))
    tiles = 8 * 20000 + 4 * 5000 + 64 * 16 + 4 * 16 * 900 + other
    assert bench.layout_bytes_per_iteration(k1t, "fp32") == tiles
    assert bench.layout_bytes_per_iteration(k1tx, "fp32") == tiles + 36 * 20000
    assert bench.layout_bytes_per_iteration(glob, "fp32") == 900 * (8 + 64) + 18000 * 48 + other
    k1tx.tile_lanes, k1tx.tile_stages = 2, 2
    assert bench.layout_name(k1tx).startswith("K1T-X")
