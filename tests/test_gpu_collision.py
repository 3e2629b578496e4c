"""GPU: contact detection on the device (vbd_set_collision / vbd_detect_contacts, contact.py
restated) against the contact sets the reference itself built in its step
(tests/golden/contact_detection.npz), and the device-resident step() with contacts against
the reference's trajectory (tests/golden/contact_scene.npz)."""

import numpy as np
import pytest

from extras import contact_system

pytestmark = pytest.mark.gpu
G = (0.0, 0.0, -9.8)


@pytest.fixture(scope="module")
def V():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2403_06321_b200 as V
    return V


class _Coll:
    """collision_mesh / collision_map of a System whose vertices all belong to tet bodies."""

    def __init__(self, V, s):
        self.collision_mesh = V.build_tet_mesh(s.rest_positions, s.tets, 1.0)
        self.collision_map = np.arange(s.num_vertices)


def test_device_contact_sets_match_reference(V, O, golden):
    g = golden("contact_detection.npz")
    s = contact_system(O)
    ctx = V.DeviceContext.from_system(O.RefSystemView(s), precision="fp64")
    ctx.set_collision(_Coll(V, s), V.ContactParams(k_c=1e6, mu_c=0.5, eps_v=1e-3), 4)
    seen_ccd = 0
    for k in range(int(g["num"])):
        which = int(g[f"r{k}_which"])
        ctx.set_state(x=g[f"r{k}_x"], x_t=g[f"r{k}_x_t"])
        if which == 1:
            ctx.detect_contacts(0)  # the step's DCD set (CCD drops pairs it already tracks)
        idx, gam, nrm, ccd = ctx.detect_contacts(which)
        want = g[f"r{k}_idx"]
        assert np.array_equal(idx, want), (k, idx[:5], want[:5])
        if len(want):
            # CCD records come from a time of impact (cubic root + 20-step bisection); our
            # closed-form root and the reference's companion-matrix eigenvalue agree to ~1e-13,
            # which moves the impact geometry by ~1e-12
            tol = 1e-12 if which == 0 else 1e-9
            assert np.abs(gam - g[f"r{k}_gamma"]).max() <= tol, k
            assert np.abs(nrm - g[f"r{k}_normal"]).max() <= tol, k
            assert bool(ccd.all()) == (which == 1)
        if which == 0:
            assert np.array_equal(ctx.colliding(), g[f"r{k}_flags"]), k
        seen_ccd += which == 1 and len(want) > 0
    assert seen_ccd >= 3


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-8), ("fp32", 1e-4)])
def test_step_with_contacts_matches_reference(V, golden, precision, tol):
    """The heavy cube dropped on the light one through this package's own step()."""
    g = golden("contact_scene.npz")
    n = 4
    light = V.generate_beam(n, n, n, 0.3 / (n - 1), density=10.0)
    heavy0 = V.generate_beam(n, n, n, 0.2 / (n - 1), density=2000.0)
    heavy = V.build_tet_mesh(heavy0.rest_positions + [0.05, 0.05, 0.3005], heavy0.tets, 2000.0)
    bottom = [i for i in range(light.num_vertices) if light.rest_positions[i, 2] < 1e-9]
    system = V.build_system([V.Body(light, V.MaterialParams(1e6, 1e7), k_d=0.01),
                             V.Body(heavy, V.MaterialParams(1e6, 1e7), k_d=0.01)],
                            [V.FixedConstraint(i) for i in bottom])
    params = V.SolverParams(h=1 / 120, n_max=10, a_ext=G, precision=precision,
                            contact=V.ContactParams(k_c=1e6, mu_c=0.5, eps_v=1e-3))
    state = V.make_state(system)
    diag = float(np.linalg.norm(system.rest_positions.max(0) - system.rest_positions.min(0)))
    for k in range(len(g["steps"])):
        V.step(state, params)
        err = np.abs(state.x - g["steps"][k]).max() / diag
        assert err <= tol, (k, err)
    # the heavy cube rests on the light one instead of falling through it
    nl = light.num_vertices
    assert state.x[nl:, 2].min() > 0.29
