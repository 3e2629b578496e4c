"""GPU: the non-tet terms of the colour pass -- springs (_native.pyx:319-349), world-box
(:401-409) and subspace constraints (:435-463, solver.py:158-162) -- against the golden
scene written by the reference (tests/golden/extras_scene.npz) and the oracle.

Tolerances as in tests/test_gpu_parity.py: one pass fp64 <= 1e-12 (absolute), trajectories
fp64 <= 1e-10 x bbox diagonal, fp32 <= 1e-5 x bbox diagonal.
"""

import numpy as np
import pytest

from extras import extras_system

pytestmark = pytest.mark.gpu
G = (0.0, 0.0, -9.8)


@pytest.fixture(scope="module")
def V():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2403_06321_b200 as V
    return V


def _diag(s):
    x = s.rest_positions
    return float(np.linalg.norm(x.max(0) - x.min(0)))


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-12), ("fp32", 1e-4)])
def test_extras_passes_match_reference_golden(V, O, golden, precision, tol):
    """One pass, absolute bar (the scene spans 0.8).  fp32: the forces of the stiff springs
    and box penalty are small residuals of large terms, so the fp32 rounding of the inputs is
    amplified ~50x more than in the plain beam (2e-6); the mode-1 Jacobi pass is the worst."""
    g = golden("extras_scene.npz")
    m, s = extras_system(O, g)
    ctx = V.DeviceContext.from_system(O.RefSystemView(s), precision=precision)
    assert ctx.info.tiles == 0  # non-tet terms run in the global-memory K1
    h = float(g["h"])
    x = g["x0"].copy()
    for c, grp in enumerate(s.groups()):
        ctx.color_pass(x, g["x_t"], g["y"], h, grp)
        assert np.abs(x - g[f"after_color{c}"]).max() <= tol, (c, np.abs(x - g[f"after_color{c}"]).max())
        x = g[f"after_color{c}"].copy()
    allv = np.arange(s.num_vertices)
    for mode in (0, 1):
        x = g["x0"].copy()
        ctx.color_pass(x, g["x_t"], g["y"], h, allv, mode=mode)
        assert np.abs(x - g[f"jacobi_mode{mode}"]).max() <= tol, mode
    x = g["x0"].copy()
    ctx.color_pass(x, g["x_t"], g["y"], h, allv, line_search=True)
    assert np.abs(x - g["jacobi_linesearch"]).max() <= tol


def _noise_floor(O, s, rho, n_steps):
    """How far the reference algorithm itself drifts from a 1e-7 (fp32-scale) perturbation
    of the initial positions, per step (oracle, fp64) -- SURVEY §7.6's noise-floor method."""
    a = O.make_state(s)
    pert = s.rest_positions + 1e-7 * np.random.default_rng(0).standard_normal(s.rest_positions.shape)
    b = O.make_state(s, x0=pert)
    out = []
    for _ in range(n_steps):
        O.step(s, a, 1.0 / 60.0, 15, rho, G)
        O.step(s, b, 1.0 / 60.0, 15, rho, G)
        out.append(np.abs(a.x - b.x).max() / _diag(s))
    return out


@pytest.mark.parametrize("rho", [0.0, 0.9])
@pytest.mark.parametrize("precision,tol", [("fp64", 1e-10), ("fp32", 1e-5)])
def test_extras_steps_match_reference_golden(V, O, golden, rho, precision, tol):
    """fp64 holds 1e-10 x diag throughout.  fp32 holds 1e-5 x diag while the scene is
    well-conditioned; with rho = 0.9 the cloth hitting the (non-smooth) box penalty amplifies
    a 1e-7 perturbation to ~1e-3 x diag in the reference itself, so from there the fp32 bar
    is 10x that measured floor."""
    g = golden("extras_scene.npz")
    m, s = extras_system(O, g)
    ctx = V.DeviceContext.from_system(O.RefSystemView(s), precision=precision)
    z = np.zeros((s.num_vertices, 3))
    ctx.set_state(x=s.rest_positions, x_t=s.rest_positions, v_t=z, v_prev=z)
    p = ctx.step_params(1.0 / 60.0, 15, rho, 1e-10, "adaptive", G)
    xs = g[f"steps_rho{int(rho * 100):02d}"]
    diag = _diag(s)
    floor = _noise_floor(O, s, rho, len(xs)) if precision == "fp32" else [0.0] * len(xs)
    for k in range(len(xs)):
        ctx.step(p)
        x = ctx.get_state(x=True)["x"]
        err = np.abs(x - xs[k]).max() / diag
        assert err <= max(tol, 10 * floor[k]), (k, err, floor[k])
    nb = m.num_vertices
    assert (x[nb:nb + 25, 2] < 0.185).any()  # the cloth is on the box floor


def test_extras_line_search_steps_vs_oracle(V, O, golden):
    g = golden("extras_scene.npz")
    m, s = extras_system(O, g)
    ctx = V.DeviceContext.from_system(O.RefSystemView(s), precision="fp64")
    z = np.zeros((s.num_vertices, 3))
    ctx.set_state(x=s.rest_positions, x_t=s.rest_positions, v_t=z, v_prev=z)
    p = ctx.step_params(1.0 / 60.0, 10, 0.0, 1e-10, "adaptive", G, line_search=True)
    st = O.make_state(s)
    for _ in range(3):
        ctx.step(p)
        O.step(s, st, 1.0 / 60.0, 10, 0.0, G, line_search=True)
    x = ctx.get_state(x=True)["x"]
    assert np.abs(x - st.x).max() / _diag(s) <= 1e-10


def test_mirrored_api_springs_and_constraints(V, O):
    """vbdsim-style scene through this package's own build_system / step."""
    beam = V.generate_beam(6, 3, 3, 0.05)
    chain = V.generate_chain(5, 0.05, stiffness=400.0, mass=0.02)
    nb = beam.num_vertices
    root = np.flatnonzero(beam.rest_positions[:, 0] < 1e-9)
    cons = [V.FixedConstraint(int(v)) for v in root] + [V.FixedConstraint(nb)]
    cons.append(V.SubspaceConstraint(nb - 1, np.array([[0.0], [0.0], [1.0]]), beam.rest_positions[-1]))
    cons += [V.WorldBoxConstraint(nb + k, (-1, -1, -0.1), (1, 1, 1), 5e3) for k in range(1, 5)]
    system = V.build_system([V.Body(beam, V.MaterialParams(1e6, 1e7, 1e-6)),
                             V.Body(chain, None, k_d=1e-3)], cons)
    state = V.make_state(system)
    params = V.SolverParams(h=1 / 60, n_max=12, rho=0.5, a_ext=G, precision="fp64")
    # oracle twin of the same scene
    ob = O.generate_beam(6, 3, 3, 0.05)
    osys = O.build_system_ex(
        [(ob, (1e6, 1e7, 1e-6))],
        [(chain.particles, chain.masses, chain.indices, chain.rest_length, chain.stiffness, 1e-3)],
        fixed=list(root) + [nb], subspace=[(nb - 1, [[0.0], [0.0], [1.0]], ob.rest_positions[-1])],
        boxes=[(nb + k, (-1, -1, -0.1), (1, 1, 1), 5e3) for k in range(1, 5)])
    assert np.array_equal(system.colors.color_of, osys.color_of)
    ost = O.make_state(osys)
    for _ in range(5):
        V.step(state, params)
        O.step(osys, ost, 1 / 60, 12, 0.5, G)
    assert np.abs(state.x - ost.x).max() / _diag(osys) <= 1e-10
    assert abs(state.x[nb - 1, 0] - beam.rest_positions[-1, 0]) < 1e-12  # stays on its line
