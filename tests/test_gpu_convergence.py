"""baselines.descend / run_convergence / `converge` on the GPU against the reference's own
outputs (tests/golden/convergence.npz from make_golden.convergence_fixture: harness.py:702-743
and baselines.py:139-189 run on the reference's native CPU path, including its Newton G*)."""

import json
from pathlib import Path

import numpy as np
import pytest
from click.testing import CliRunner

from paper_2403_06321_b200 import baselines, parse_scene, run_convergence, scene_build
from paper_2403_06321_b200.cli import main as cli_main
from paper_2403_06321_b200.solver import _collision, _INPUTS, device_context, initialize

pytestmark = pytest.mark.gpu

GOLD = np.load(Path(__file__).parent / "golden" / "harness.npz")
CONV = np.load(Path(__file__).parent / "golden" / "convergence.npz")
SCENES = ("base", "placed", "mixed", "contact")
METHODS = ("vbd", "vbd-cheb", "jacobi", "gd")
ITERS = int(CONV["iters"])
G_RTOL = 1e-9   # per-iteration G: fp64 device reduction vs the reference's host sum
X_TOL = 1e-9    # final iterate after 24 iterations, relative to the bounding-box diagonal


def _cfg(name):
    return parse_scene(str(GOLD[f"{name}_scene"]))


def _diag(x):
    return float(np.linalg.norm(x.max(0) - x.min(0)))


@pytest.mark.parametrize("name", SCENES)
def test_run_convergence_matches_reference(name):
    """The same start (DCD + warm start), the same G trace and relative loss per solver, the
    same final iterate; G* given as the reference's Newton optimum."""
    g_star = float(CONV[f"{name}_g_star"])
    res = run_convergence(_cfg(name), METHODS, ITERS, g_star=g_star)
    assert res["g_star"] == g_star and res["g_star_method"] == "given"
    diag = _diag(CONV[f"{name}_x0"])
    for m in METHODS:
        tr = res["traces"][m]
        np.testing.assert_allclose(tr.g, CONV[f"{name}_{m}_g"], rtol=G_RTOL, atol=0, err_msg=m)
        err = np.abs(tr.x_final - CONV[f"{name}_{m}_x"]).max() / diag
        assert err <= X_TOL, (m, err)
        want = CONV[f"{name}_{m}_loss"]
        np.testing.assert_allclose(res["relative_loss"][m], want, rtol=1e-6,
                                   atol=1e-9 * max(1.0, np.abs(want).max()), err_msg=m)
        assert tr.wall_ms[0] == 0.0 and np.all(np.diff(tr.wall_ms) >= 0)


@pytest.mark.parametrize("name", ("base", "mixed"))
def test_descend_from_reference_start(name):
    """descend from the reference's own frozen start (x0, y0) -- no detection involved."""
    system, state, params = scene_build(_cfg(name))
    x0, y0 = CONV[f"{name}_x0"], CONV[f"{name}_y0"]
    for m in METHODS:
        state.x, state.y = x0.copy(), y0.copy()
        p = params
        if m == "vbd-cheb" and p.rho == 0.0:
            from dataclasses import replace
            p = replace(p, rho=0.95)
        tr = baselines.descend(state, p, m, ITERS)
        np.testing.assert_allclose(tr.g, CONV[f"{name}_{m}_g"], rtol=G_RTOL, atol=0, err_msg=m)
        assert np.array_equal(state.x, tr.x_final)


@pytest.mark.parametrize("name", SCENES)
def test_warm_start_matches_reference(name):
    system, state, params = scene_build(_cfg(name))
    ctx = device_context(system, params.precision, params.device)
    _collision(ctx, system, params)
    state._bind(ctx)
    state._upload(_INPUTS)
    initialize(state, params)
    diag = _diag(CONV[f"{name}_x0"])
    assert np.abs(state.x - CONV[f"{name}_x0"]).max() / diag <= 1e-12
    np.testing.assert_allclose(state.y, CONV[f"{name}_y0"], rtol=1e-14, atol=1e-15)


def test_g_star_defaults_to_lowest_recorded_g():
    """Without a given G* (Newton is not provided) the lowest G of the traces stands in."""
    res = run_convergence(_cfg("base"), ["vbd", "jacobi"], 8)
    assert res["g_star_method"] == "min-trace"
    assert res["g_star"] == min(float(t.g.min()) for t in res["traces"].values())
    for m in ("vbd", "jacobi"):
        assert res["relative_loss"][m][0] == 1.0 and res["relative_loss"][m].min() >= 0.0


def test_newton_and_unknown_methods_rejected():
    system, state, params = scene_build(_cfg("base"))
    with pytest.raises(NotImplementedError):
        baselines.descend(state, params, "newton", 2)
    with pytest.raises(ValueError):
        baselines.descend(state, params, "cg", 2)


def test_cli_converge_writes_traces(tmp_path):
    p = tmp_path / "s.json"
    p.write_text(str(GOLD["base_scene"]))
    out = tmp_path / "c.csv"
    g_star = float(CONV["base_g_star"])
    res = CliRunner().invoke(cli_main, ["converge", "--scene", str(p), "--out", str(out),
                                        "--iters", str(ITERS), "--g-star", repr(g_star)])
    assert res.exit_code == 0, res.output
    summary = json.loads(res.output)
    assert summary["backend"] == "b200" and summary["g_star"] == g_star
    lines = out.read_text().splitlines()
    assert lines[0] == "solver,iteration,G,relative_loss,wall_ms"
    assert len(lines) == 1 + 4 * (ITERS + 1)
    rows = [ln.split(",") for ln in lines[1:]]
    for m in METHODS:
        g = np.array([float(r[2]) for r in rows if r[0] == m])
        np.testing.assert_allclose(g, CONV[f"base_{m}_g"], rtol=G_RTOL, atol=0)
        assert summary["final_G"][m] == pytest.approx(float(g[-1]), rel=1e-15)


def test_descend_zero_iterations_and_fp32():
    """n_iters = 0 records G_0 only and leaves x alone; an fp32 context follows the fp64
    reference trace to fp32 accuracy."""
    from dataclasses import replace
    system, state, params = scene_build(_cfg("base"))
    x0, y0 = CONV["base_x0"], CONV["base_y0"]
    state.x, state.y = x0.copy(), y0.copy()
    tr = baselines.descend(state, params, "vbd", 0)
    assert tr.g.shape == (1,) and tr.wall_ms.tolist() == [0.0]
    np.testing.assert_allclose(tr.g[0], CONV["base_vbd_g"][0], rtol=G_RTOL)
    assert np.array_equal(tr.x_final, x0)
    # fp32 build: the colour-sweep traces end within the north-star fp32 bar of the reference's
    # fp64 iterate (jacobi / gd accept-or-reject line searches on fp32 G are not compared)
    p32 = replace(params, precision="fp32")
    diag = _diag(x0)
    for m in ("vbd", "vbd-cheb"):
        state.x, state.y = x0.copy(), y0.copy()
        p = replace(p32, rho=0.95) if m == "vbd-cheb" and p32.rho == 0.0 else p32
        tr = baselines.descend(state, p, m, ITERS)
        err = np.abs(tr.x_final - CONV[f"base_{m}_x"]).max() / diag
        assert err <= 1e-5, (m, err)
