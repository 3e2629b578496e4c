"""The mirrored vbdsim API (paper_2403_06321_b200) on the GPU: the reference's own step
invariants (pkg/tests/test_solver.py, test_acceptance.py #2/#7/#9) restated against our
package, plus the lazy host/device coherence of SimState."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
G = (0.0, 0.0, -9.8)


@pytest.fixture(scope="module")
def V():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2403_06321_b200 as V
    return V


def beam_state(V, nx=3, ny=2, nz=2, constraints=(), mat=None, spacing=0.1):
    mat = mat or V.MaterialParams(2e5, 8e5)
    mesh = V.generate_beam(nx, ny, nz, spacing, density=1000.0)
    if callable(constraints):
        constraints = constraints(mesh)
    system = V.build_system([V.Body(mesh, mat)], constraints)
    return system, V.make_state(system)


def test_build_system_matches_oracle(V, O):
    mesh = V.generate_beam(9, 4, 4, 0.05)
    fixed = np.flatnonzero(mesh.rest_positions[:, 0] < 1e-9)
    s = V.build_system([V.Body(mesh, V.MaterialParams(1e6, 1e7, 1e-6))],
                       [V.FixedConstraint(int(v)) for v in fixed])
    o = O.build_system([(O.generate_beam(9, 4, 4, 0.05), (1e6, 1e7, 1e-6))], fixed)
    for k in ("tets", "tet_w", "tet_vol", "masses", "t_off", "t_id", "t_slot", "color_off",
              "color_verts"):
        assert np.array_equal(getattr(s, k), getattr(o, k)), k
    assert np.array_equal(s.colors.color_of, o.color_of)
    assert np.array_equal(s.cons.kind, o.kind)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_rest_is_fixed_point(V, precision):
    system, state = beam_state(V, mat=V.MaterialParams(2e5, 8e5, k_d=0.01))
    p = V.SolverParams(h=1 / 60, n_max=4, a_ext=(0, 0, 0), precision=precision)
    V.step(state, p)
    tol = 1e-12 if precision == "fp64" else 1e-6
    assert np.allclose(state.x, system.rest_positions, atol=tol)
    assert np.allclose(state.v_t, 0.0, atol=1e-10 if precision == "fp64" else 1e-4)


def test_single_particle_is_implicit_euler(V):
    """Acceptance #2 (test_acceptance.py:249-268): inertia-only step is exact."""
    net = V.SpringNet(np.zeros((1, 3)), np.zeros((0, 2), np.int64), np.zeros(0), np.zeros(0),
                      np.array([2.5]))
    system = V.build_system([V.Body(net)])
    state = V.make_state(system)
    state.v_t = np.array([[0.3, -0.1, 0.2]])
    h = 1.0 / 60.0
    v_t = state.v_t.copy()
    y = state.x_t + h * v_t + h * h * np.array(G)
    V.step(state, V.SolverParams(h=h, n_max=1, a_ext=G))
    v_expect = v_t + h * np.array(G)
    assert np.abs(state.x - y).max() / np.abs(y).max() <= 1e-12
    assert np.abs(state.v_t - v_expect).max() / np.abs(v_expect).max() <= 1e-12


def test_velocity_update_and_step_index(V):
    system, state = beam_state(V, constraints=(V.FixedConstraint(0),))
    p = V.SolverParams(h=0.01, n_max=6, a_ext=G)
    x_before = state.x_t.copy()
    V.step(state, p)
    assert np.allclose(state.v_t, (state.x_t - x_before) / 0.01, atol=1e-12)
    assert state.step_index == 1


def test_fixed_vertices_hold(V):
    system, state = beam_state(V, 6, 3, 3, constraints=lambda m: [
        V.FixedConstraint(int(v)) for v in np.flatnonzero(m.rest_positions[:, 0] < 1e-9)])
    fixed = np.flatnonzero(system.cons.kind == 1)
    p = V.SolverParams(h=1 / 60, n_max=8, a_ext=G)
    for _ in range(5):
        V.step(state, p)
        assert np.array_equal(state.x[fixed], system.rest_positions[fixed])


def test_deterministic_repeat(V):
    results = []
    for _ in range(2):
        system, state = beam_state(V, constraints=(V.FixedConstraint(0), V.FixedConstraint(1)))
        p = V.SolverParams(h=1 / 60, n_max=10, rho=0.9, a_ext=G)
        for _ in range(5):
            V.step(state, p)
        results.append(state.x.copy())
    assert np.array_equal(results[0], results[1])


def test_nonfinite_diagnostics(V):
    system, state = beam_state(V)
    state.v_t[3, 2] = np.inf  # in-place host edit must reach the device
    p = V.SolverParams(h=0.01, n_max=3, a_ext=G)
    with pytest.raises(V.NonFiniteState) as exc:
        V.step(state, p)
    assert exc.value.iteration == 1
    assert exc.value.step == 0
    assert exc.value.vertex >= 0
    assert state.step_index == 0


def test_host_edits_between_steps_are_seen(V, O):
    """Lazy coherence: results equal to an always-synchronised oracle run."""
    system, state = beam_state(V, 9, 4, 4, spacing=0.05, mat=V.MaterialParams(1e6, 1e7, 1e-6))
    o = O.build_system([(O.generate_beam(9, 4, 4, 0.05), (1e6, 1e7, 1e-6))])
    ost = O.make_state(o)
    p = V.SolverParams(h=1 / 60, n_max=10, rho=0.9, a_ext=G)
    for k in range(4):
        if k == 2:
            kick = np.zeros_like(state.x)
            kick[:, 2] = 0.5
            state.v_t = state.v_t + kick
            ost.v_t = ost.v_t + kick
        V.step(state, p)
        O.step(o, ost, 1 / 60, 10, 0.9, G)
    assert np.abs(state.x - ost.x).max() <= 1e-10


def test_on_iteration_callback(V):
    system, state = beam_state(V, 9, 4, 4, spacing=0.05)
    seen = []
    p = V.SolverParams(h=1 / 60, n_max=5, rho=0.5, a_ext=G)
    V.step(state, p, on_iteration=lambda st, n: seen.append((n, st.x.copy())))
    assert [n for n, _ in seen] == [1, 2, 3, 4, 5]
    assert np.array_equal(seen[-1][1], state.x)
    system2, state2 = beam_state(V, 9, 4, 4, spacing=0.05)
    V.step(state2, p)
    assert np.array_equal(state2.x, state.x)


def test_initialize_modes(V):
    for mode in ("prev_pos", "inertia", "inertia_accel", "adaptive"):
        system, state = beam_state(V)
        rng = np.random.default_rng(1)
        state.v_t = rng.standard_normal(state.x_t.shape)
        state.v_prev = rng.standard_normal(state.x_t.shape)
        h = 0.01
        p = V.SolverParams(h=h, init_mode=mode, a_ext=G)
        x = V.initialize(state, p).copy()
        xt, vt, vp = state.x_t, state.v_t, state.v_prev
        a = np.array(G)
        if mode == "prev_pos":
            want = xt
        elif mode == "inertia":
            want = xt + h * vt
        elif mode == "inertia_accel":
            want = xt + h * vt + h * h * a
        else:
            a_t = (vt - vp) / h
            comp = a_t @ (a / np.linalg.norm(a))
            at = np.clip(comp / np.linalg.norm(a), 0, 1)
            want = xt + h * vt + (h * h) * at[:, None] * a
        assert np.allclose(x, want, atol=1e-14), mode


def test_local_solve_and_color_pass(V):
    system, state = beam_state(V)
    rng = np.random.default_rng(4)
    state.x = state.x + 0.02 * rng.standard_normal(state.x.shape)
    p = V.SolverParams(h=0.01, a_ext=G)
    state.y = V.inertia_target(state.x_t, state.v_t, p.a_ext_vec, p.h)
    for i in (0, 5, system.num_vertices - 1):
        delta = V.local_solve(i, state, p)
        ref = state.x.copy()
        V.color_pass(state, np.array([i]), p)
        assert np.allclose(state.x[i], ref[i] + delta, atol=1e-12)
        state.x = ref


def test_contacts_with_iteration_callback(V):
    """step(on_iteration=...) with contacts runs the same detection as the graph-free step."""
    system, a = beam_state(V)
    b = V.make_state(system)
    p = V.SolverParams(h=0.01, a_ext=(0, 0, -9.8), contact=V.ContactParams(k_c=1e5))
    V.step(a, p)
    V.step(b, p, on_iteration=lambda st, n: None)
    assert np.array_equal(a.x, b.x)
