"""K1R, the resident whole-step kernel for small scenes (csrc/vbd_resident.cuh).

The step of a small scene runs as ONE launch: REPL (one thread-block cluster, every CTA holds
a replica of all positions in shared memory, DSMEM broadcast + barrier.cluster per colour pass)
or GLOB (one CTA per SM, positions in L2, grid barrier).  Its per-vertex arithmetic is the K1
one, so it must be BITWISE equal to the per-colour graph path (VBD_RESIDENT=0), and through it
within the fp64 / fp32 bars of the oracle.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = (0.0, 0.0, -9.8)
H = 1.0 / 60.0


@pytest.fixture(scope="module")
def V():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2403_06321_b200 as V
    return V


def c1_system(O, nx=41, ny=11, nz=11, spacing=0.025, mat=(1e6, 1e7, 1e-6)):
    m = O.generate_beam(nx, ny, nz, spacing)
    fixed = np.flatnonzero(m.rest_positions[:, 0] < 1e-9)
    return m, O.build_system([(m, mat)], fixed)


def run(V, O, s, precision, resident, monkeypatch, n=3, rho=0.9, n_max=10, x0=None):
    monkeypatch.setenv("VBD_RESIDENT", resident)
    ctx = V.DeviceContext.from_system(O.RefSystemView(s), precision=precision)
    monkeypatch.delenv("VBD_RESIDENT")
    z = np.zeros((s.num_vertices, 3))
    x0 = s.rest_positions if x0 is None else x0
    ctx.set_state(x=x0, x_t=x0, v_t=z, v_prev=z)
    p = ctx.step_params(H, n_max, rho, 1e-10, "adaptive", G)
    for _ in range(n):
        ctx.step(p)
    info = ctx._info()
    out = ctx.get_state(x=True, v_t=True, v_prev=True, x_t=True)
    ctx.close()
    return out, info


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("rho", [0.0, 0.9])
def test_c1_cluster_resident_bitwise_equals_graph(V, O, precision, rho, monkeypatch):
    m, s = c1_system(O)
    a, ia = run(V, O, s, precision, "", monkeypatch, rho=rho)
    b, ib = run(V, O, s, precision, "0", monkeypatch, rho=rho)
    if precision == "fp32":
        assert ia.resident == 1 and ia.resident_ctas in (8, 16), (ia.resident, ia.resident_ctas)
    assert ib.resident == 0
    for k in ("x", "v_t", "v_prev", "x_t"):
        assert np.array_equal(a[k], b[k]), k
    st = O.make_state(s)
    for _ in range(3):
        O.step(s, st, H, 10, rho, G)
    tol = 1e-10 if precision == "fp64" else 1e-5
    assert np.abs(a["x"] - st.x).max() / m.bbox_diagonal() <= tol


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_grid_resident_bitwise_equals_graph(V, O, precision, monkeypatch):
    m, s = c1_system(O, 13, 6, 6, 0.05)
    a, ia = run(V, O, s, precision, "glob", monkeypatch)
    b, _ = run(V, O, s, precision, "0", monkeypatch)
    assert ia.resident == 2 and ia.resident_ctas > 16
    for k in ("x", "v_t", "v_prev", "x_t"):
        assert np.array_equal(a[k], b[k]), k


def test_resident_mixed_materials_per_vertex(V, O, monkeypatch):
    """one material per vertex off: per-entry damping from the kind records (UM = false)"""
    m, s = c1_system(O, 13, 6, 6, 0.05)
    rng = np.random.default_rng(3)
    pick = rng.random(len(s.tets)) < 0.5
    s.tet_mu = np.where(pick, 1e6, 3e6)
    s.tet_lam = np.where(pick, 1e7, 2e7)
    s.tet_kd = np.where(pick, 1e-6, 5e-6)
    # fp64: two materials double the kinds and the table no longer fits next to the replica,
    # so the fp64 case runs the grid-resident form (kinds + slots spread over the SMs)
    for prec, mode, want in (("fp32", "repl", 1), ("fp64", "glob", 2)):
        a, ia = run(V, O, s, prec, mode, monkeypatch)
        b, _ = run(V, O, s, prec, "0", monkeypatch)
        assert ia.resident == want
        assert np.array_equal(a["x"], b["x"])


def test_resident_extreme_init_and_nonfinite_report(V, O, monkeypatch):
    """random initial positions (inverted tets), rho 0.95: still bitwise; and a NaN start is
    reported with the same (step, iteration, vertex) as the graph path"""
    m, s = c1_system(O, 9, 9, 9, 0.05, (2e6, 1e7, 1e-6))
    lo, hi = m.rest_positions.min(0), m.rest_positions.max(0)
    x0 = np.random.default_rng(0).uniform(lo, hi, size=m.rest_positions.shape)
    a, _ = run(V, O, s, "fp64", "repl", monkeypatch, n=1, rho=0.95, n_max=100, x0=x0)
    b, _ = run(V, O, s, "fp64", "0", monkeypatch, n=1, rho=0.95, n_max=100, x0=x0)
    assert np.array_equal(a["x"], b["x"])
    x0[17] = np.nan
    res = []
    for mode in ("repl", "0"):
        monkeypatch.setenv("VBD_RESIDENT", mode)
        ctx = V.DeviceContext.from_system(O.RefSystemView(s), precision="fp32")
        monkeypatch.delenv("VBD_RESIDENT")
        z = np.zeros_like(x0)
        ctx.set_state(x=x0, x_t=x0, v_t=z, v_prev=z)
        with pytest.raises(V.NonFiniteState) as ei:
            ctx.step(ctx.step_params(H, 10, 0.0, 1e-10, "adaptive", G))
        res.append((ei.value.step, ei.value.iteration, ei.value.vertex))
        ctx.close()
    assert res[0] == res[1]


def test_device_generated_c1_bench_scene_resident(V, monkeypatch):
    """the bench's C1 workload (scenes.build) runs resident and equals the graph path"""
    from paper_2403_06321_b200.scenes import build, config
    cfg = config("c1")
    xs = []
    for mode in ("", "0"):
        monkeypatch.setenv("VBD_RESIDENT", mode)
        ctx, _ = build(cfg, precision="fp32")
        monkeypatch.delenv("VBD_RESIDENT")
        for _ in range(3):
            ctx.step(cfg.step_params())
        xs.append((ctx.get_state(x=True)["x"], ctx._info().resident))
        ctx.close()
    assert xs[0][1] == 1 and xs[1][1] == 0
    assert np.array_equal(xs[0][0], xs[1][0])


def test_device_generated_c2_bench_scene_grid_resident(V, monkeypatch):
    """the bench's C2 workload (37^3, rho 0.95, extreme init) runs grid-resident by default
    (too large for one cluster's replica, small enough to be launch-bound as a graph) and equals
    the graph path bitwise"""
    from paper_2403_06321_b200.scenes import build, config
    cfg = config("c2")
    xs = []
    for mode in ("", "0"):
        monkeypatch.setenv("VBD_RESIDENT", mode)
        ctx, _ = build(cfg, precision="fp32")
        monkeypatch.delenv("VBD_RESIDENT")
        for _ in range(2):
            ctx.step(cfg.step_params())
        xs.append((ctx.get_state(x=True, v_t=True), ctx._info().resident))
        ctx.close()
    assert xs[0][1] == 2 and xs[1][1] == 0
    assert np.array_equal(xs[0][0]["x"], xs[1][0]["x"]) and np.array_equal(xs[0][0]["v_t"], xs[1][0]["v_t"])
