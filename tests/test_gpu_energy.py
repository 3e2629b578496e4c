"""GPU: the incremental potential G(x) = 1/(2h^2)|x - y|_M^2 + E(x) on the device
(vbd_energy; _assembly.py:78-82, the per-iteration metric of harness.run_simulation,
harness.py:664-678) against values the reference's own baselines.energy recorded
(tests/golden/energy.npz) and the oracle.  Bars: relative 1e-12 (fp64); fp32 1e-5 relative
(the inertia term is |x - y|^2 of two fp32 positions a few 1e-3 apart)."""

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


def _beam(O):
    m = O.generate_beam(9, 4, 4, 0.05)
    return O.build_system([(m, (1e6, 1e7, 1e-6))], np.flatnonzero(m.rest_positions[:, 0] < 1e-9))


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-12), ("fp32", 1e-5)])
@pytest.mark.parametrize("scene", ["extras", "beam"])
def test_energy_matches_reference_golden(V, O, golden, precision, tol, scene):
    g = golden("energy.npz")
    s = extras_system(O, golden("extras_scene.npz"))[1] if scene == "extras" else _beam(O)
    ctx = V.DeviceContext.from_system(O.RefSystemView(s), precision=precision)
    for k in range(len(g[f"{scene}_G"])):
        ctx.set_state(x=g[f"{scene}_x"][k], y=g[f"{scene}_y"][k])
        got = ctx.energy(1 / 60)
        want = float(g[f"{scene}_G"][k])
        assert abs(got - want) <= tol * abs(want), (k, got, want)


def test_energy_per_iteration_metric(V, O):
    """step(on_iteration=cb) with cb calling energy(): the metrics path without a D2H of x."""
    mesh = V.generate_beam(9, 4, 4, 0.05)
    root = np.flatnonzero(mesh.rest_positions[:, 0] < 1e-9)
    system = V.build_system([V.Body(mesh, V.MaterialParams(1e6, 1e7, 1e-6))],
                            [V.FixedConstraint(int(v)) for v in root])
    state = V.make_state(system)
    params = V.SolverParams(h=1 / 60, n_max=10, rho=0.5, a_ext=G, precision="fp64")
    rows = []
    V.step(state, params, on_iteration=lambda st, n: rows.append(V.energy(st, params)))
    s = _beam(O)
    st = O.make_state(s)
    want = []
    O.step(s, st, 1 / 60, 10, 0.5, G, on_iteration=lambda o, n: want.append(
        O.variational_energy(s, o.x, o.y, 1 / 60)))
    assert len(rows) == 10
    assert np.allclose(rows, want, rtol=1e-11, atol=0)
    assert rows[-1] < rows[0]  # VBD decreases G within the step


def test_energy_per_iteration_with_contacts(V, golden):
    """The metrics path of a contact scene: device detection inside step(on_iteration=...),
    G including the contact penalty (_assembly.py:49-56), against the reference's values."""
    g = golden("energy.npz")
    n = 4
    light = V.generate_beam(n, n, n, 0.3 / (n - 1), density=10.0)
    heavy0 = V.generate_beam(n, n, n, 0.2 / (n - 1), density=2000.0)
    heavy = V.build_tet_mesh(heavy0.rest_positions + [0.05, 0.05, 0.3005], heavy0.tets, 2000.0)
    bottom = [i for i in range(light.num_vertices) if light.rest_positions[i, 2] < 1e-9]
    system = V.build_system([V.Body(light, V.MaterialParams(1e6, 1e7), k_d=0.01),
                             V.Body(heavy, V.MaterialParams(1e6, 1e7), k_d=0.01)],
                            [V.FixedConstraint(i) for i in bottom])
    params = V.SolverParams(h=1 / 120, n_max=10, a_ext=G, precision="fp64",
                            contact=V.ContactParams(k_c=1e6, mu_c=0.5, eps_v=1e-3))
    state = V.make_state(system)
    rows = []
    for _ in range(2):
        V.step(state, params, on_iteration=lambda st, k: rows.append(V.energy(st, params)))
    got = np.array(rows[::5])
    assert np.allclose(got, g["contact_G"], rtol=1e-8, atol=0), (got, g["contact_G"])
