"""run_simulation / scene_build / the CLI on the GPU against the reference's own outputs
(tests/golden/harness.npz from make_golden.harness_fixture: pkg/src/vbdsim/harness.py:521-691
and cli.py run on the reference's native CPU path)."""

import json
from pathlib import Path

import numpy as np
import pytest
from click.testing import CliRunner

from paper_2403_06321_b200 import load_frame, parse_scene, run_simulation, scene_build
from paper_2403_06321_b200.cli import main as cli_main
from paper_2403_06321_b200.harness import surface_faces

pytestmark = pytest.mark.gpu

GOLD = np.load(Path(__file__).parent / "golden" / "harness.npz")
SCENES = ("base", "placed", "mixed", "contact")
G_RTOL = 1e-9      # per-iteration G: fp64 device reduction vs the reference's host sum
X_TOL = 1e-10      # positions, relative to the scene's bounding-box diagonal
PEN_TOL = 1e-9     # max_penetration, absolute (metres)


def _scene(name, **over):
    doc = json.loads(str(GOLD[f"{name}_scene"]))
    doc.update(over)
    return parse_scene(json.dumps(doc))


@pytest.mark.parametrize("name", SCENES)
def test_scene_build_matches_reference(name):
    system, state, params = scene_build(_scene(name))
    g = lambda f: GOLD[f"{name}_{f}"]
    for f in ("tets", "springs", "color_verts", "color_off"):
        assert np.array_equal(np.asarray(getattr(system, f)).reshape(g(f).shape), g(f)), f
    for f in ("rest_positions", "masses", "sp_l0", "sp_k", "sp_kd"):
        np.testing.assert_allclose(np.asarray(getattr(system, f)).reshape(g(f).shape), g(f),
                                   rtol=1e-14, atol=1e-15, err_msg=f)
    for f in system.cons._fields:
        np.testing.assert_allclose(np.asarray(getattr(system.cons, f), dtype=np.float64),
                                   np.asarray(g(f"cons_{f}"), dtype=np.float64),
                                   rtol=1e-14, atol=1e-15, err_msg=f)
    np.testing.assert_allclose(state.x, g("x0"), rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(state.v_t, g("v0"), rtol=1e-14, atol=1e-15)
    assert np.array_equal(surface_faces(system), g("faces"))


def _metrics(path):
    lines = (path / "metrics.csv").read_text().splitlines()
    assert lines[0] == "step,iteration,G,relative_loss,contact_count,max_penetration,wall_ms"
    return np.array([[float(c) for c in ln.split(",")[:-1]] for ln in lines[1:]])


@pytest.mark.parametrize("name", SCENES)
def test_run_simulation_matches_reference(name, tmp_path):
    """harness.py:637-691: the same frame files, the same per-iteration metric rows (step,
    iteration, G, relative_loss, contact_count, max_penetration) and the same last frame."""
    summary = run_simulation(_scene(name), tmp_path)
    want = GOLD[f"{name}_metrics"]
    got = _metrics(tmp_path)
    assert got.shape == want.shape
    assert np.array_equal(got[:, :2], want[:, :2])                       # step, iteration
    np.testing.assert_allclose(got[:, 2], want[:, 2], rtol=G_RTOL)         # G
    assert np.array_equal(got[:, 4], want[:, 4])                         # contact_count
    np.testing.assert_allclose(got[:, 5], want[:, 5], rtol=0, atol=PEN_TOL)
    # relative_loss = (G_n - G_last)/(G_1 - G_last): a ratio of G differences
    span = np.abs(want[:, 2]).max() * G_RTOL
    np.testing.assert_allclose(got[:, 3], want[:, 3], rtol=0, atol=max(1e-6, 1e3 * span))
    files = sorted(p.name for p in tmp_path.glob("frame_*"))
    assert files == list(GOLD[f"{name}_frame_files"])
    assert summary["frame_files"] == len(files) and summary["backend"] == "b200"
    pos, fac = load_frame(tmp_path / files[-1])
    rest = GOLD[f"{name}_rest_positions"]
    diag = np.linalg.norm(rest.max(0) - rest.min(0))
    np.testing.assert_allclose(pos, GOLD[f"{name}_last_x"], rtol=0, atol=X_TOL * diag)
    assert np.array_equal(fac, GOLD[f"{name}_last_faces"])


def test_simulation_deterministic(tmp_path):
    for tag in ("a", "b"):
        run_simulation(_scene("contact"), tmp_path / tag)
    for f in ("frame_00000.bin", "frame_00003.bin"):
        assert (tmp_path / "a" / f).read_bytes() == (tmp_path / "b" / f).read_bytes()
    assert np.array_equal(_metrics(tmp_path / "a"), _metrics(tmp_path / "b"))


@pytest.mark.parametrize("name", ("base", "mixed"))
def test_metrics_off_same_trajectory(name, tmp_path):
    """metrics_mode='off' (one CUDA graph per step) reaches the same frames bit for bit."""
    run_simulation(_scene(name), tmp_path / "it")
    run_simulation(_scene(name), tmp_path / "off", metrics_mode="off")
    assert len(_metrics(tmp_path / "off")) == 0
    for p in sorted((tmp_path / "it").glob("frame_*")):
        assert p.read_bytes() == (tmp_path / "off" / p.name).read_bytes(), p.name


def test_frames_override_and_every(tmp_path):
    cfg = _scene("base", frames=4, output={"format": "bin", "every": 2})
    s = run_simulation(cfg, tmp_path, frames=5)
    assert s["frames"] == 5 and s["steps"] == 5
    assert sorted(p.name for p in tmp_path.glob("frame_*")) == [
        "frame_00000.bin", "frame_00002.bin", "frame_00004.bin", "frame_00005.bin"]


def test_cli_simulate_and_divergence(tmp_path):
    scene = tmp_path / "s.json"
    scene.write_text(str(GOLD["base_scene"]))
    res = CliRunner().invoke(cli_main, ["simulate", "--scene", str(scene), "--out", str(tmp_path / "o")])
    assert res.exit_code == 0, res.output
    assert json.loads(res.output)["frames"] == 2
    doc = json.loads(str(GOLD["base_scene"]))
    doc.update(frames=1, gravity=[0.0, 0.0, -1e308])  # t_harness:333-343
    doc["solver"]["n_max"] = 2
    scene.write_text(json.dumps(doc))
    res = CliRunner().invoke(cli_main, ["simulate", "--scene", str(scene), "--out", str(tmp_path / "d")])
    assert res.exit_code == 3, res.output
    assert "diverged" in res.output


def test_cli_color_matches_reference(tmp_path):
    (tmp_path / "m.node").write_text(str(GOLD["mesh_node"]))
    (tmp_path / "m.ele").write_text(str(GOLD["mesh_ele"]))
    res = CliRunner().invoke(cli_main, ["color", "--nodes", str(tmp_path / "m.node"),
                                        "--eles", str(tmp_path / "m.ele")])
    assert res.exit_code == 0, res.output
    assert json.dumps(json.loads(res.output), sort_keys=True) == str(GOLD["color_json"])


@pytest.mark.parametrize("name", ("base", "mixed"))
def test_run_simulation_fp32_within_tolerance(name, tmp_path):
    """solver.precision = "fp32" (the performance build): same frames within 1e-5 x bbox
    diagonal of the reference's fp64 run (BASELINE north_star tolerance)."""
    doc = json.loads(str(GOLD[f"{name}_scene"]))
    doc.setdefault("solver", {})["precision"] = "fp32"
    run_simulation(parse_scene(json.dumps(doc)), tmp_path)
    files = sorted(p.name for p in tmp_path.glob("frame_*"))
    assert files == list(GOLD[f"{name}_frame_files"])
    pos, _ = load_frame(tmp_path / files[-1])
    rest = GOLD[f"{name}_rest_positions"]
    diag = np.linalg.norm(rest.max(0) - rest.min(0))
    assert np.abs(pos - GOLD[f"{name}_last_x"]).max() <= 1e-5 * diag
    got = _metrics(tmp_path)
    np.testing.assert_allclose(got[:, 2], GOLD[f"{name}_metrics"][:, 2], rtol=1e-4)


def test_chain_only_scene_obj_frames(tmp_path):
    """A spring-net-only scene has no collision surface: frames carry vertices and no faces."""
    doc = {"objects": [{"generator": {"kind": "chain", "count": 8, "spacing": 0.05, "stiffness": 500.0}}],
           "gravity": [0.0, 0.0, -9.8],
           "constraints": [{"kind": "fixed", "object": 0, "vertices": [0]}],
           "solver": {"h": 0.01, "n_max": 5}, "frames": 3, "output": {"format": "obj", "every": 1}}
    s = run_simulation(parse_scene(json.dumps(doc)), tmp_path)
    assert s["frame_files"] == 4 and s["steps"] == 3
    pos, fac = load_frame(tmp_path / "frame_00003.obj")
    assert pos.shape == (8, 3) and fac.shape == (0, 3) and np.isfinite(pos).all()
    assert np.array_equal(pos[0], [0.0, 0.0, 0.0])      # the fixed end stays put
    assert pos[-1, 2] < 0.0                              # the free end falls under gravity
    rows = _metrics(tmp_path)
    assert rows.shape == (3 * 5, 6) and (rows[:, 4] == 0).all()
