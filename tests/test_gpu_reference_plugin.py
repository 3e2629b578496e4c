"""The drop-in seam exercised with the UNMODIFIED reference package.

The reference is pip-installed into baseline/_ref (git-ignored; it travels to the GPU box),
``vbdsim._backend._impl`` is pointed at ``paper_2403_06321_b200.backend`` exactly as the
one-line change in INTEGRATION.md §1 would, and the reference's own solver is run with the
B200 kernel against the same solver with the reference's compiled kernel.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
G = (0.0, 0.0, -9.8)


@pytest.fixture(scope="module")
def ref():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    # build() installs the unmodified reference here; its absence is a failure, not a skip
    assert (REF / "vbdsim").exists(), "reference not installed in baseline/_ref (run build())"
    sys.path.insert(0, str(REF))
    import vbdsim
    from vbdsim import _backend
    assert vbdsim.backend_name() == "native"
    return vbdsim, _backend


@pytest.fixture
def with_b200(ref):
    vbdsim, _backend = ref
    import paper_2403_06321_b200.backend as b200
    native = _backend._impl

    class Swap:
        def __enter__(self):
            _backend._impl = b200
            return b200

        def __exit__(self, *a):
            _backend._impl = native
    return Swap


def _beam(vbdsim, nx=9, ny=4, nz=4, sp=0.05, mat=(1e6, 1e7, 1e-6)):
    m = vbdsim.generate_beam(nx, ny, nz, sp, density=1000.0)
    fixed = np.flatnonzero(m.rest_positions[:, 0] < 1e-9)
    s = vbdsim.build_system([vbdsim.Body(m, vbdsim.MaterialParams(*mat))],
                            [vbdsim.FixedConstraint(int(v)) for v in fixed])
    return m, s


@pytest.mark.parametrize("rho", [0.0, 0.9])
def test_reference_step_with_b200_backend(ref, with_b200, rho):
    vbdsim, _ = ref
    m, s = _beam(vbdsim)
    p = vbdsim.SolverParams(h=1 / 60, n_max=10, rho=rho, a_ext=G)
    a, b = vbdsim.make_state(s), vbdsim.make_state(s)
    for _ in range(5):
        vbdsim.step(a, p)
    with with_b200() as impl:
        assert vbdsim.backend_name() == "b200"
        for _ in range(5):
            vbdsim.step(b, p)
    diag = m.bbox_diagonal()
    assert np.abs(a.x - b.x).max() / diag <= 1e-10
    assert np.abs(a.v_t - b.v_t).max() <= 1e-8


@pytest.mark.parametrize("mode", [0, 1])
def test_reference_jacobi_pass_matches_native(ref, with_b200, mode):
    vbdsim, _backend = ref
    m, s = _beam(vbdsim, 13, 6, 6, 0.05, (2e5, 8e5, 2e-3))
    st = vbdsim.make_state(s)
    rng = np.random.default_rng(9)
    st.v_t = 0.4 * rng.standard_normal(st.x.shape)
    p = vbdsim.SolverParams(h=1 / 60, a_ext=G)
    st.y = vbdsim.inertia_target(st.x_t, st.v_t, p.a_ext_vec, p.h)
    vbdsim.initialize(st, p)
    group = np.arange(s.num_vertices, dtype=np.int64)
    xa, xb = st.x.copy(), st.x.copy()
    _backend._impl.color_pass(s, st.carr, xa, st.x_t, st.y, p.h, group, mode, n_threads=1)
    with with_b200() as impl:
        impl.color_pass(s, st.carr, xb, st.x_t, st.y, p.h, group, mode)
    assert np.abs(xa - xb).max() < 1e-12  # test_backends.py:78 bar


def test_reference_system_on_fast_path(ref):
    """A reference System packed straight into a device context and stepped resident."""
    vbdsim, _ = ref
    import paper_2403_06321_b200 as V
    m, s = _beam(vbdsim, 41, 11, 11, 0.025)
    p = vbdsim.SolverParams(h=1 / 60, n_max=10, a_ext=G)
    st = vbdsim.make_state(s)
    for _ in range(10):
        vbdsim.step(st, p)
    for precision, tol in (("fp64", 1e-10), ("fp32", 1e-5)):
        ctx = V.DeviceContext.from_system(s, precision=precision)
        z = np.zeros((s.num_vertices, 3))
        ctx.set_state(x=s.rest_positions, x_t=s.rest_positions, v_t=z, v_prev=z)
        ctx.step(ctx.step_params(1 / 60, 10, 0.0, 1e-10, "adaptive", G), n_steps=10)
        x = ctx.get_state(x=True)["x"]
        assert np.abs(x - st.x).max() / m.bbox_diagonal() <= tol, precision


def test_springs_through_the_plugin_match_native(ref, with_b200):
    """A tet cube hanging from a spring chain: the unmodified reference solver with the b200
    colour pass against the reference's own native backend."""
    vbdsim, _ = ref
    chain = vbdsim.generate_chain(4, 0.2, stiffness=900.0, mass=0.1)
    cube = vbdsim.generate_cube(3, 0.4, density=1000.0)
    s = vbdsim.build_system([vbdsim.Body(cube, vbdsim.MaterialParams(2e5, 8e5)),
                             vbdsim.Body(chain, None, k_d=0.001)],
                            [vbdsim.FixedConstraint(cube.num_vertices)])
    p = vbdsim.SolverParams(h=1 / 60, n_max=10, a_ext=G)
    a, b = vbdsim.make_state(s), vbdsim.make_state(s)
    for _ in range(5):
        vbdsim.step(a, p)
    with with_b200():
        for _ in range(5):
            vbdsim.step(b, p)
    diag = float(np.linalg.norm(s.rest_positions.max(0) - s.rest_positions.min(0)))
    assert np.abs(a.x - b.x).max() / diag <= 1e-10


def test_contact_scene_through_the_plugin_matches_native(ref, with_b200):
    """A heavy cube dropped onto a light one: the reference's own detection (broad phase,
    DCD, CCD, friction) with the b200 colour pass, against the native backend."""
    vbdsim, _ = ref
    n = 4
    light = vbdsim.generate_beam(n, n, n, 0.3 / (n - 1), density=10.0)
    heavy0 = vbdsim.generate_beam(n, n, n, 0.2 / (n - 1), density=2000.0)
    heavy = vbdsim.build_tet_mesh(heavy0.rest_positions + [0.05, 0.05, 0.3005], heavy0.tets, 2000.0)
    bottom = [i for i in range(light.num_vertices) if light.rest_positions[i, 2] < 1e-9]
    s = vbdsim.build_system([vbdsim.Body(light, vbdsim.MaterialParams(1e6, 1e7), k_d=0.01),
                             vbdsim.Body(heavy, vbdsim.MaterialParams(1e6, 1e7), k_d=0.01)],
                            [vbdsim.FixedConstraint(i) for i in bottom])
    p = vbdsim.SolverParams(h=1 / 120, n_max=10, threads=1, a_ext=G,
                            contact=vbdsim.ContactParams(k_c=1e6, mu_c=0.5, eps_v=1e-3))
    a, b = vbdsim.make_state(s), vbdsim.make_state(s)
    for _ in range(4):
        vbdsim.step(a, p)
    with with_b200():
        for _ in range(4):
            vbdsim.step(b, p)
    assert len(b.contact_set) > 0
    diag = float(np.linalg.norm(s.rest_positions.max(0) - s.rest_positions.min(0)))
    assert np.abs(a.x - b.x).max() / diag <= 1e-10
