"""GPU parity: the sm_100a path (through the C ABI) against the oracle and the
reference's golden vectors.

Tolerances (north_star, BASELINE.json):
  * colouring: bit-exact (integer work);
  * one colour pass, fp64: |dx| <= 1e-12 (the reference's own native-vs-NumPy bar,
    pkg/tests/test_backends.py:78);
  * trajectories: fp64 within 1e-10 x bbox diagonal, fp32 within 1e-5 x bbox
    diagonal, over 10 steps.
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


def beam_sys(O, nx=9, ny=4, nz=4, spacing=0.05, mat=(1e6, 1e7, 1e-6), fix=True):
    m = O.generate_beam(nx, ny, nz, spacing)
    fixed = np.flatnonzero(m.rest_positions[:, 0] < 1e-9) if fix else np.zeros(0, np.int64)
    s = O.build_system([(m, mat)], fixed)
    return m, s


def ctx_for(V, O, s, precision):
    return V.DeviceContext.from_system(O.RefSystemView(s), precision=precision)


# --------------------------------------------------------------------------------------
# colouring (K5) -- bit-exact


@pytest.mark.parametrize("name,build", [
    ("c1", lambda O: [O.generate_beam(41, 11, 11, 0.025)]),
    ("c2", lambda O: [O.generate_cube(37, 0.5)]),
    ("c3", lambda O: [O.generate_beam(3032, 4, 4, 0.01)] * 2),
    ("twobody", lambda O: [O.generate_beam(9, 4, 4, 0.05), O.generate_cube(5, 0.3)]),
    ("c4obj", lambda O: [O.generate_cube(15, 0.3)]),
])
def test_device_greedy_color_bit_exact(V, O, golden, name, build):
    g = golden(f"color_{name}.npz")
    meshes = build(O)
    off, tets = 0, []
    for m in meshes:
        tets.append(m.tets + off)
        off += m.num_vertices
    noff, nids = O.merged_adjacency(off, [np.concatenate(tets)])
    adj = V.VertexAdjacency(off, None, None, None, noff, nids)
    part = V.greedy_color(adj)
    assert np.array_equal(part.color_of, g["color_of"].astype(np.int64))
    assert part.num_colors == len(g["color_off"]) - 1


def test_device_greedy_color_custom_order(V, O):
    m = O.generate_beam(7, 5, 4, 0.1)
    noff, nids = O.merged_adjacency(m.num_vertices, [m.tets])
    order = np.random.default_rng(1).permutation(m.num_vertices)
    a, _ = O.greedy_color(noff, nids, order=order)
    part = V.greedy_color(V.VertexAdjacency(m.num_vertices, None, None, None, noff, nids),
                          order=order)
    assert np.array_equal(part.color_of, a)


@pytest.mark.parametrize("beams,golden_name", [
    ([(41, 11, 11, 0.025)], "c1"),
    ([(37, 37, 37, 0.5 / 36)], "c2"),
    ([(3032, 4, 4, 0.01), (3032, 4, 4, 0.01)], "c3"),
])
def test_device_generated_scene_coloring(V, golden, beams, golden_name):
    g = golden(f"color_{golden_name}.npz")
    bs = [V.Beam(*b, mu=1e6, lam=1e7, kd=1e-6, origin=(2.0 * k, 0, 0)) for k, b in enumerate(beams)]
    ctx = V.DeviceContext.from_beams(bs, precision="fp32")
    assert np.array_equal(ctx.colors(), g["color_of"].astype(np.int64))
    assert ctx.info.num_tets == int(g["t"])


# --------------------------------------------------------------------------------------
# one colour pass (K1) against the reference's golden outputs


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-12), ("fp32", 2e-6)])
def test_color_pass_matches_reference_golden(V, O, golden, precision, tol):
    g = golden("pass_beam_9_4_4.npz")
    m, s = beam_sys(O)
    ctx = ctx_for(V, O, s, precision)
    h = float(g["h"])
    x = g["x0"].copy()
    for c, grp in enumerate(s.groups()):
        ctx.color_pass(x, g["x_t"], g["y"], h, grp)
        err = np.abs(x - g[f"after_color{c}"]).max()
        assert err <= tol, (c, err)
        x = g[f"after_color{c}"].copy()  # per-pass parity on identical inputs
    allv = np.arange(s.num_vertices)
    for mode in (0, 1):
        x = g["x0"].copy()
        ctx.color_pass(x, g["x_t"], g["y"], h, allv, mode=mode)
        assert np.abs(x - g[f"jacobi_mode{mode}"]).max() <= tol, mode


def test_color_pass_fp64_vs_oracle_random_states(V, O):
    m, s = beam_sys(O, 13, 6, 6, 0.05, mat=(2e5, 8e5, 2e-3))
    ctx = ctx_for(V, O, s, "fp64")
    rng = np.random.default_rng(11)
    for trial in range(3):
        x0 = s.rest_positions * [1.3, 1.0, 0.9] + 0.01 * rng.standard_normal((s.num_vertices, 3))
        xt = s.rest_positions + 0.005 * rng.standard_normal((s.num_vertices, 3))
        y = xt + 0.002 * rng.standard_normal((s.num_vertices, 3))
        for grp in s.groups() + [np.arange(s.num_vertices), np.array([5, 17, 3])]:
            a, b = x0.copy(), x0.copy()
            O.color_pass(s, a, xt, y, H, grp)
            ctx.color_pass(b, xt, y, H, grp)
            assert np.abs(a - b).max() <= 1e-12


def test_color_pass_edge_cases(V, O):
    m, s = beam_sys(O)
    ctx = ctx_for(V, O, s, "fp64")
    x = s.rest_positions + 0.01
    before = x.copy()
    ctx.color_pass(x, s.rest_positions, s.rest_positions, H, np.zeros(0, np.int64))
    assert np.array_equal(x, before)  # ng == 0 is a no-op (_native.pyx:520-521)
    fixed = np.flatnonzero(s.kind == 1)
    ctx.color_pass(x, s.rest_positions, s.rest_positions, H, fixed)
    assert np.array_equal(x, before)  # fixed vertices never move (_native.pyx:424-426)
    ctx.color_pass(x, s.rest_positions, s.rest_positions, H, np.arange(s.num_vertices), eps_det=2.0)
    assert np.array_equal(x, before)  # det guard freezes every vertex (test_solver.py:236-245)
    with pytest.raises(TypeError):
        ctx.color_pass(x.astype(np.float32), s.rest_positions, s.rest_positions, H, [0])


# --------------------------------------------------------------------------------------
# whole steps (K2..K4 around K1, CUDA graph)


def run_ctx_steps(ctx, s, n_steps, h=H, n_max=10, rho=0.0, a=G, x0=None):
    ctx.set_state(x=s.rest_positions if x0 is None else x0,
                  x_t=s.rest_positions if x0 is None else x0,
                  v_t=np.zeros((s.num_vertices, 3)), v_prev=np.zeros((s.num_vertices, 3)))
    p = ctx.step_params(h, n_max, rho, 1e-10, "adaptive", a)
    xs = []
    for _ in range(n_steps):
        ctx.step(p)
        xs.append(ctx.get_state(x=True, v_t=True))
    return xs


@pytest.mark.parametrize("rho", [0.0, 0.9])
@pytest.mark.parametrize("precision,tol", [("fp64", 1e-10), ("fp32", 1e-5)])
def test_steps_match_reference_golden(V, O, golden, rho, precision, tol):
    g = golden(f"steps_beam_rho{int(rho * 100):02d}.npz")
    m, s = beam_sys(O)
    diag = m.bbox_diagonal()
    ctx = ctx_for(V, O, s, precision)
    xs = run_ctx_steps(ctx, s, 10, rho=rho)
    for k in range(10):
        err = np.abs(xs[k]["x"] - g["x"][k]).max() / diag
        assert err <= tol, (k, err)


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-10), ("fp32", 1e-5)])
def test_c1_ten_steps(V, O, golden, precision, tol):
    """BASELINE config 1 (cantilever 41x11x11, fixed root) over 10 steps."""
    g = golden("steps_c1.npz")
    m, s = beam_sys(O, 41, 11, 11, 0.025)
    diag = m.bbox_diagonal()
    ctx = ctx_for(V, O, s, precision)
    xs = run_ctx_steps(ctx, s, 10)
    assert np.abs(xs[0]["x"] - g["x_step1"]).max() / diag <= tol
    assert np.abs(xs[9]["x"] - g["x_step10"]).max() / diag <= tol


def test_extreme_init_fp64(V, O, golden):
    """Randomised initial positions, rho=0.95, n_max=100 (BASELINE config 2, small)."""
    g = golden("steps_extreme_cube6.npz")
    m = O.generate_cube(6, 0.5)
    s = O.build_system([(m, (2e6, 1e7, 1e-6))])
    diag = m.bbox_diagonal()
    ctx = ctx_for(V, O, s, "fp64")
    xs = run_ctx_steps(ctx, s, 3, n_max=100, rho=0.95, a=(0, 0, 0), x0=g["x0"])
    for k in range(3):
        err = np.abs(xs[k]["x"] - g["x"][k]).max() / diag
        assert err <= 1e-9, (k, err)  # chaotic scene: reference's own backends differ ~1e-9


def test_device_generated_c1_matches_oracle(V, O):
    """Device generator + packer + masses (fp64) vs the oracle's host-built scene."""
    m, s = beam_sys(O, 41, 11, 11, 0.025)
    diag = m.bbox_diagonal()
    ctx = V.DeviceContext.from_beams([V.Beam(41, 11, 11, 0.025, 1e6, 1e7, 1e-6, fix_min_x=True)],
                                     precision="fp64")
    assert ctx.info.num_fixed == 121
    p = ctx.step_params(H, 10, 0.0, 1e-10, "adaptive", G)
    st = O.make_state(s)
    for k in range(5):
        ctx.step(p)
        O.step(s, st, H, 10, 0.0, G)
    x = ctx.get_state(x=True)["x"]
    assert np.abs(x - st.x).max() / diag <= 1e-10


def test_step_bitwise_repeatable(V, O):
    m, s = beam_sys(O, 13, 6, 6, 0.05)
    outs = []
    for precision in ("fp32", "fp32", "fp64", "fp64"):
        ctx = ctx_for(V, O, s, precision)
        outs.append(run_ctx_steps(ctx, s, 3, rho=0.9)[-1]["x"])
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(outs[2], outs[3])


def test_multi_step_resident_equals_single_steps(V, O):
    m, s = beam_sys(O, 13, 6, 6, 0.05)
    a = ctx_for(V, O, s, "fp32")
    b = ctx_for(V, O, s, "fp32")
    run_ctx_steps(a, s, 0)
    run_ctx_steps(b, s, 0)
    p = a.step_params(H, 10, 0.9, 1e-10, "adaptive", G)
    a.step(p, n_steps=5)
    for _ in range(5):
        b.step(p)
    assert np.array_equal(a.get_state(x=True)["x"], b.get_state(x=True)["x"])


# --------------------------------------------------------------------------------------
# multi-GPU logic emulated on one GPU: slabs with halo exchange, object shards


def test_slab_decomposition_bitwise_equals_single_context(V):
    import torch
    beam = V.Beam(24, 7, 6, 0.02, 1e6, 1e7, 1e-6, fix_min_x=True)
    full = V.DeviceContext.from_beams([beam], precision="fp32")
    nx = beam.nx
    cuts = [0, 7, 15, nx]
    slabs = [V.DeviceContext.from_beams([beam], precision="fp32", slab=(cuts[r], cuts[r + 1]))
             for r in range(3)]
    p = full.step_params(1 / 120, 8, 0.9, 1e-10, "adaptive", G)
    for _ in range(3):
        full.step(p)
    from paper_2403_06321_b200.dist import SlabExchange
    ex = SlabExchange.local(slabs)
    for _ in range(3):
        ex.step(p)
    xf = full.get_state(x=True)["x"]
    plane = beam.ny * beam.nz
    for r, sctx in enumerate(slabs):
        xs = sctx.get_state(x=True)["x"]
        lo = max(cuts[r] - 1, 0)
        own = slice((cuts[r] - lo) * plane, (cuts[r + 1] - lo) * plane)
        assert np.array_equal(xs[own], xf[cuts[r] * plane:cuts[r + 1] * plane]), r


def test_object_sharding_bitwise_equals_single_context(V):
    cubes = [V.Beam(5, 5, 5, 0.05, 1e6, 1e7, 1e-6, origin=(0.5 * k, 0, 0)) for k in range(6)]
    la = np.zeros((6, 6))
    la[:, 3:] = np.linspace(-2, 2, 18).reshape(6, 3)
    whole = V.DeviceContext.from_beams(cubes, precision="fp32")
    whole.set_beam_velocities(la)
    parts = [V.DeviceContext.from_beams(cubes[:2], precision="fp32"),
             V.DeviceContext.from_beams(cubes[2:], precision="fp32")]
    parts[0].set_beam_velocities(la[:2])
    parts[1].set_beam_velocities(la[2:])
    p = whole.step_params(1 / 120, 10, 0.0, 1e-10, "adaptive", G)
    for c in [whole] + parts:
        c.step(p, n_steps=4)
    xw = whole.get_state(x=True)["x"]
    xp = np.concatenate([c.get_state(x=True)["x"] for c in parts])
    assert np.array_equal(xw, xp)


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-10), ("fp32", 1e-5)])
def test_twisting_beam_kinematic_bc(V, O, precision, tol):
    """BASELINE config 3 at 1/10 length: both ends clamped and rotated by rewriting x_t of
    the fixed vertices every step (as test_acceptance.py:471-473 drives the reference)."""
    from paper_2403_06321_b200.scenes import config, twist_targets
    cfg = config("c3", scale=0.1)
    b = cfg.beams[0]
    ctx = V.DeviceContext.from_beams([cfg.beams[0]], precision=precision)
    m = O.generate_beam(b.nx, b.ny, b.nz, b.spacing)
    plane = b.ny * b.nz
    fixed = np.concatenate([np.arange(plane), (b.nx - 1) * plane + np.arange(plane)])
    s = O.build_system([(m, (b.mu, b.lam, b.kd))], fixed)
    st = O.make_state(s)
    one = type(cfg)(cfg.name, (b,), cfg.h, cfg.n_max, cfg.rho, cfg.a_ext, twist_rev_s=cfg.twist_rev_s)
    p = ctx.step_params(cfg.h, cfg.n_max, cfg.rho, 1e-10, "adaptive", cfg.a_ext)
    for k in range(1, 11):
        idx, xyz = twist_targets(one, s.rest_positions, k * cfg.h)
        ctx.set_fixed_targets(idx, xyz)
        ctx.step(p)
        st.x_t[idx] = xyz
        st.x[idx] = xyz
        O.step(s, st, cfg.h, cfg.n_max, cfg.rho, cfg.a_ext)
    x = ctx.get_state(x=True)["x"]
    assert np.abs(x - st.x).max() / m.bbox_diagonal() <= tol
    # the clamped ends really turned
    assert np.abs(x[idx] - s.rest_positions[idx]).max() > 1e-3


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-12), ("fp32", 2e-6)])
def test_line_search_pass_matches_reference_golden(V, O, golden, precision, tol):
    """Jacobi pass with the 17-trial local line search (_native.pyx:481-492)."""
    g = golden("pass_beam_9_4_4.npz")
    m, s = beam_sys(O)
    ctx = ctx_for(V, O, s, precision)
    x = g["x0"].copy()
    ctx.color_pass(x, g["x_t"], g["y"], float(g["h"]), np.arange(s.num_vertices), line_search=True)
    assert np.abs(x - g["jacobi_linesearch"]).max() <= tol


def test_line_search_steps_vs_oracle(V, O):
    m, s = beam_sys(O, 13, 6, 6, 0.05)
    ctx = ctx_for(V, O, s, "fp64")
    st = O.make_state(s)
    z = np.zeros((s.num_vertices, 3))
    ctx.set_state(x=s.rest_positions, x_t=s.rest_positions, v_t=z, v_prev=z)
    p = ctx.step_params(1 / 30, 20, 0.0, 1e-10, "adaptive", G, line_search=True)
    for _ in range(3):
        ctx.step(p)
        O.step(s, st, 1 / 30, 20, 0.0, G, line_search=True)
    x = ctx.get_state(x=True)["x"]
    assert np.abs(x - st.x).max() / m.bbox_diagonal() <= 1e-10


def test_slab_p2p_bitwise_equals_single_context(V):
    """The fused peer-memory halo (K1 pushes + device phase barriers), three slabs of one
    process on separate streams, against one context."""
    beam = V.Beam(26, 7, 6, 0.02, 1e6, 1e7, 1e-6, fix_min_x=True)
    full = V.DeviceContext.from_beams([beam], precision="fp32")
    cuts = [0, 8, 17, beam.nx]
    slabs = [V.DeviceContext.from_beams([beam], precision="fp32", slab=(cuts[r], cuts[r + 1]))
             for r in range(3)]
    from paper_2403_06321_b200.dist import SlabP2P
    ex = SlabP2P.local(slabs)
    for rho in (0.9, 0.0):  # the phase count per step changes between the two
        p = full.step_params(1 / 120, 6, rho, 1e-10, "adaptive", G)
        for _ in range(3):
            full.step(p)
        for _ in range(3):
            ex.step(p)
        xf = full.get_state(x=True)["x"]
        plane = beam.ny * beam.nz
        for r, sctx in enumerate(slabs):
            xs = sctx.get_state(x=True)["x"]
            lo = max(cuts[r] - 1, 0)
            own = slice((cuts[r] - lo) * plane, (cuts[r + 1] - lo) * plane)
            assert np.array_equal(xs[own], xf[cuts[r] * plane:cuts[r + 1] * plane]), (rho, r)


def test_slab_p2p_disconnect_then_nccl_style_exchange(V):
    """bench.py's fallback: slabs connected for the P2P halo, then disconnected and stepped with
    the host-driven exchange -- no stale peer stores, still bitwise equal to one context."""
    beam = V.Beam(24, 7, 6, 0.02, 1e6, 1e7, 1e-6, fix_min_x=True)
    full = V.DeviceContext.from_beams([beam], precision="fp32")
    cuts = [0, 7, 15, beam.nx]
    slabs = [V.DeviceContext.from_beams([beam], precision="fp32", slab=(cuts[r], cuts[r + 1]))
             for r in range(3)]
    from paper_2403_06321_b200.dist import SlabExchange, SlabP2P
    SlabP2P.local(slabs)
    for sctx in slabs:
        sctx.p2p_disconnect()
    ex = SlabExchange.local(slabs)
    p = full.step_params(1 / 120, 8, 0.9, 1e-10, "adaptive", G)
    for _ in range(3):
        full.step(p)
        ex.step(p)
    xf = full.get_state(x=True)["x"]
    plane = beam.ny * beam.nz
    for r, sctx in enumerate(slabs):
        xs = sctx.get_state(x=True)["x"]
        lo = max(cuts[r] - 1, 0)
        own = slice((cuts[r] - lo) * plane, (cuts[r + 1] - lo) * plane)
        assert np.array_equal(xs[own], xf[cuts[r] * plane:cuts[r + 1] * plane]), r


def test_slab_p2p_irregular_mesh_k1t_x_bitwise(V, monkeypatch):
    """An irregular mesh (jittered rest positions, explicit layout -> K1T-X) decomposed into
    three slabs with the fused peer-memory halo: bitwise equal to one context."""
    monkeypatch.setenv("VBD_LAYOUT", "explicit")
    monkeypatch.setenv("VBD_RESIDENT", "0")
    beam = V.Beam(26, 7, 6, 0.02, 1e6, 1e7, 1e-6, fix_min_x=True, jitter=0.1)
    full = V.DeviceContext.from_beams([beam], precision="fp32")
    cuts = [0, 8, 17, beam.nx]
    slabs = [V.DeviceContext.from_beams([beam], precision="fp32", slab=(cuts[r], cuts[r + 1]))
             for r in range(3)]
    monkeypatch.delenv("VBD_LAYOUT")
    monkeypatch.delenv("VBD_RESIDENT")
    assert full.info.layout == 0 and full.info.tiles > 0
    from paper_2403_06321_b200.dist import SlabP2P
    ex = SlabP2P.local(slabs)
    p = full.step_params(1 / 120, 6, 0.9, 1e-10, "adaptive", G)
    for _ in range(3):
        full.step(p)
        ex.step(p)
    xf = full.get_state(x=True)["x"]
    plane = beam.ny * beam.nz
    for r, sctx in enumerate(slabs):
        xs = sctx.get_state(x=True)["x"]
        lo = max(cuts[r] - 1, 0)
        own = slice((cuts[r] - lo) * plane, (cuts[r + 1] - lo) * plane)
        assert np.array_equal(xs[own], xf[cuts[r] * plane:cuts[r + 1] * plane]), r


def test_slab_p2p_class_tiles_bitwise(V, monkeypatch):
    """Grid-class tiles (one lane per interior vertex, neighbours in registers) inside three
    slabs with the fused peer-memory halo: bitwise equal to one context (the slab boundary and
    ghost planes are plain vertices; every slab's interior is class tiles)."""
    for k, v in (("VBD_RESIDENT", "0"), ("VBD_TILE_V", "64"), ("VBD_ENTRY_ORDER", "code")):
        monkeypatch.setenv(k, v)
    beam = V.Beam(48, 14, 12, 0.02, 1e6, 1e7, 1e-6, fix_min_x=True)
    full = V.DeviceContext.from_beams([beam], precision="fp32")
    cuts = [0, 15, 31, beam.nx]
    slabs = [V.DeviceContext.from_beams([beam], precision="fp32", slab=(cuts[r], cuts[r + 1]))
             for r in range(3)]
    for k in ("VBD_RESIDENT", "VBD_TILE_V", "VBD_ENTRY_ORDER"):
        monkeypatch.delenv(k)
    assert full._info().class_tiles > 0 and all(sc._info().class_tiles > 0 for sc in slabs)
    from paper_2403_06321_b200.dist import SlabP2P
    ex = SlabP2P.local(slabs)
    p = full.step_params(1 / 120, 6, 0.9, 1e-10, "adaptive", G)
    for _ in range(3):
        full.step(p)
        ex.step(p)
    xf = full.get_state(x=True)["x"]
    plane = beam.ny * beam.nz
    for r, sctx in enumerate(slabs):
        xs = sctx.get_state(x=True)["x"]
        lo = max(cuts[r] - 1, 0)
        own = slice((cuts[r] - lo) * plane, (cuts[r + 1] - lo) * plane)
        assert np.array_equal(xs[own], xf[cuts[r] * plane:cuts[r + 1] * plane]), r
