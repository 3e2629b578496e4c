"""bench.py as the driver runs it: `python bench.py --gpus N` (no torchrun around it) spawns
its N ranks itself; on a one-GPU box they share the GPU (gloo control plane, fused cudaIpc
peer-memory halo for slabs, no data-path traffic for object shards).  The N-rank state must be
bitwise equal to the 1-rank state, and the JSON line must say n_gpus = N."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _bench(*args, timeout=900):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args, "--steps", "2", "--warmup", "3",
                        "--e2e-steps", "1", "--no-cpu-baseline", "--no-fp64-record", "--checksum"],
                       capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0]), r.stderr


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


@pytest.mark.parametrize("config,scale", [("c5", 1e-4), ("c4", 4e-4)])
def test_self_spawned_ranks_bitwise_equal_one_rank(gpu, config, scale):
    one, _ = _bench("--gpus", "1", "--config", config, "--scale", str(scale))
    two, err = _bench("--gpus", "2", "--config", config, "--scale", str(scale))
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["config"]["parallelism"].startswith("slabs" if config == "c5" else "objects")
    assert one["state_sha256"] == two["state_sha256"]
    assert two["value"] > 0 and two["roofline"]["frac"] > 0
