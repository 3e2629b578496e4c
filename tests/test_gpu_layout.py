"""GPU: the two entry layouts of K1.

* explicit -- every (vertex, tet) entry carries its slot-weight rows (48 B fp32 / 96 B fp64);
* compact  -- the entry is one int4 {n0, n1, n2, kind} and each distinct (rows, volume,
  material) key lives once in a kind table.  Chosen automatically when the scene has at most
  VBD_KIND_CAP distinct keys (structured grids, instanced objects).

The compact layout is a lossless re-encoding running the same arithmetic, so it must give
results bitwise identical to the explicit layout; both are held to the oracle by the parity
suite (tests/test_gpu_parity.py runs whichever layout the scene selects, i.e. compact for
the generated grids) and here on an irregular mesh that must fall back to explicit.
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


def beam_sys(O, nx=13, ny=6, nz=6, spacing=0.05, mat=(1e6, 1e7, 1e-6)):
    m = O.generate_beam(nx, ny, nz, spacing)
    fixed = np.flatnonzero(m.rest_positions[:, 0] < 1e-9)
    return m, O.build_system([(m, mat)], fixed)


def make_ctx(V, O, s, precision, layout, monkeypatch, cap=None):
    """layout: "explicit" | "compact" (16-byte entries, K1 over global memory) | "auto"
    (compact + the K1T tile pipeline when the scene allows it)."""
    monkeypatch.setenv("VBD_LAYOUT", "explicit" if layout == "explicit" else "auto")
    monkeypatch.setenv("VBD_TILES", "0" if layout == "compact" else "1")
    if cap is not None:
        monkeypatch.setenv("VBD_KIND_CAP", str(cap))
    else:
        monkeypatch.delenv("VBD_KIND_CAP", raising=False)
    ctx = V.DeviceContext.from_system(O.RefSystemView(s), precision=precision)
    monkeypatch.delenv("VBD_LAYOUT")
    monkeypatch.delenv("VBD_TILES")
    return ctx


def steps(ctx, s, n, rho=0.9, n_max=10, line_search=False, x0=None):
    z = np.zeros((s.num_vertices, 3))
    x0 = s.rest_positions if x0 is None else x0
    ctx.set_state(x=x0, x_t=x0, v_t=z, v_prev=z)
    p = ctx.step_params(H, n_max, rho, 1e-10, "adaptive", G, line_search=line_search)
    for _ in range(n):
        ctx.step(p)
    return ctx.get_state(x=True, v_t=True)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_compact_selected_for_grids(V, O, precision, monkeypatch):
    m, s = beam_sys(O)
    ctx = make_ctx(V, O, s, precision, "auto", monkeypatch)
    assert ctx.info.layout == 1 and ctx.info.entry_bytes == 16
    if precision == "fp32":
        # a 5-tet grid has 10 rest shapes x 4 slots (fp32 rows round to identical bits)
        assert ctx.info.num_entry_kinds == 40
    ex = make_ctx(V, O, s, precision, "explicit", monkeypatch)
    assert ex.info.layout == 0 and ex.info.entry_bytes == (48 if precision == "fp32" else 96)
    assert ex.info.num_entry_kinds == 0


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("rho", [0.0, 0.9])
@pytest.mark.parametrize("layout", ["compact", "auto"])
def test_compact_bitwise_equals_explicit(V, O, precision, rho, layout, monkeypatch):
    m, s = beam_sys(O)
    ctx = make_ctx(V, O, s, precision, layout, monkeypatch)
    if precision == "fp32":  # fp64 grids have ~1e3 kinds (ulp-distinct rows): tiles off
        assert (ctx.info.tiles > 0) == (layout == "auto")
    a = steps(ctx, s, 5, rho=rho)
    b = steps(make_ctx(V, O, s, precision, "explicit", monkeypatch), s, 5, rho=rho)
    assert np.array_equal(a["x"], b["x"])
    assert np.array_equal(a["v_t"], b["v_t"])


@pytest.mark.parametrize("tv", [64, 32])
def test_tiles_cover_every_colour(V, O, monkeypatch, tv):
    """64-vertex tiles per colour (32 for small scenes); every neighbour list fits the 16-bit
    local index; and the two tile sizes give bitwise the same steps."""
    m, s = beam_sys(O, 21, 9, 7)
    monkeypatch.setenv("VBD_TILE_V", str(tv))
    monkeypatch.setenv("VBD_RESIDENT", "0")
    monkeypatch.setenv("VBD_TILE_CLASS", "0")  # (class tiles hold 128 vertices: own test below)
    ctx = make_ctx(V, O, s, "fp32", "auto", monkeypatch)
    monkeypatch.delenv("VBD_TILE_CLASS")
    counts = ctx.color_counts()
    assert ctx.info.tiles == sum((c + tv - 1) // tv for c in counts)
    assert 0 < ctx.info.tile_nbr_cap < 65536
    b_ctx = make_ctx(V, O, s, "fp32", "explicit", monkeypatch)
    monkeypatch.delenv("VBD_TILE_V")
    monkeypatch.delenv("VBD_RESIDENT")
    assert np.array_equal(steps(ctx, s, 3)["x"], steps(b_ctx, s, 3)["x"])


def test_compact_bitwise_equals_explicit_line_search(V, O, monkeypatch):
    m, s = beam_sys(O)
    a = steps(make_ctx(V, O, s, "fp64", "auto", monkeypatch), s, 2, rho=0.0, line_search=True)
    b = steps(make_ctx(V, O, s, "fp64", "explicit", monkeypatch), s, 2, rho=0.0, line_search=True)
    assert np.array_equal(a["x"], b["x"])


def test_compact_mixed_materials_per_vertex(V, O, monkeypatch):
    """Non-uniform material per vertex (damping per entry, material from the kind record)."""
    m, s = beam_sys(O)
    rng = np.random.default_rng(3)
    pick = rng.random(len(s.tets)) < 0.5
    s.tet_mu = np.where(pick, 1e6, 3e6)
    s.tet_lam = np.where(pick, 1e7, 2e7)
    s.tet_kd = np.where(pick, 1e-6, 5e-6)
    monkeypatch.setenv("VBD_UNIFORM_MAT", "0")
    a_ctx = make_ctx(V, O, s, "fp64", "auto", monkeypatch)
    c_ctx = make_ctx(V, O, s, "fp64", "compact", monkeypatch)
    b_ctx = make_ctx(V, O, s, "fp64", "explicit", monkeypatch)
    assert a_ctx.info.layout == 1 and a_ctx.info.num_materials == 2
    a = steps(a_ctx, s, 3)
    b = steps(b_ctx, s, 3)
    assert np.array_equal(a["x"], b["x"])
    assert np.array_equal(steps(c_ctx, s, 3)["x"], b["x"])
    st = O.make_state(s)
    for _ in range(3):
        O.step(s, st, H, 10, 0.9, G)
    assert np.abs(a["x"] - st.x).max() / m.bbox_diagonal() <= 1e-10


def test_irregular_mesh_falls_back_to_explicit(V, O, monkeypatch):
    """Jittered rest positions: every tet has its own shape, more kinds than the cap."""
    m = O.generate_beam(9, 5, 5, 0.05)
    rng = np.random.default_rng(0)
    pos = m.rest_positions + rng.uniform(-0.008, 0.008, m.rest_positions.shape)
    mj = O.build_tet_mesh(pos, m.tets, 1000.0)
    fixed = np.flatnonzero(pos[:, 0] < 0.01)
    s = O.build_system([(mj, (1e6, 1e7, 1e-6))], fixed)
    ctx = make_ctx(V, O, s, "fp32", "auto", monkeypatch, cap=256)
    assert ctx.info.layout == 0
    roomy = make_ctx(V, O, s, "fp32", "auto", monkeypatch)  # default cap: fits
    assert roomy.info.layout == 1 and roomy.info.num_entry_kinds > 256
    st = O.make_state(s)
    for _ in range(4):
        O.step(s, st, H, 10, 0.9, G)
    diag = mj.bbox_diagonal()
    for c in (ctx, roomy):
        x = steps(c, s, 4)["x"]
        assert np.abs(x - st.x).max() / diag <= 1e-5


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_device_generated_c5_like_block_is_compact(V, precision):
    """fp64 too: the generator forms grid edges from integer cell offsets, so every cell of a
    shape has bitwise the same Dm^-1 (40 kinds, the kind table in shared memory)."""
    ctx = V.DeviceContext.from_beams([V.Beam(40, 40, 40, 0.01, 2e6, 2e7, 1e-7, fix_min_x=True)],
                                     precision=precision)
    assert ctx.info.layout == 1 and ctx.info.num_entry_kinds <= 64


def hub_system(O, n_spokes=240):
    """A beam plus one hub vertex shared by n_spokes tets (degree far above a 5-tet grid's 32):
    the tile build must decline or handle it, and every layout must still agree bitwise."""
    m = O.generate_beam(9, 5, 5, 0.05)
    rng = np.random.default_rng(3)
    pos = m.rest_positions
    hub = np.array([[0.2, 0.1, 0.35]])
    pts = np.concatenate([pos, hub])
    hub_id = len(pos)
    tets = [list(t) for t in m.tets]
    top = np.flatnonzero(pos[:, 2] > 0.19)
    for _ in range(n_spokes):
        a, b, c = rng.choice(top, 3, replace=False)
        t = [hub_id, a, b, c]
        d = np.linalg.det(np.stack([pts[t[1]] - pts[t[0]], pts[t[2]] - pts[t[0]], pts[t[3]] - pts[t[0]]]))
        if abs(d) < 1e-7:
            continue
        tets.append(t if d > 0 else [t[0], t[2], t[1], t[3]])
    mesh = O.build_tet_mesh(pts, np.asarray(tets, dtype=np.int64), 1000.0)
    fixed = np.flatnonzero(pts[:, 0] < 1e-9)
    return O.build_system([(mesh, (1e5, 1e6, 1e-6))], fixed)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_high_degree_vertex_all_layouts_bitwise(V, O, precision, monkeypatch):
    s = hub_system(O)
    a = steps(make_ctx(V, O, s, precision, "auto", monkeypatch), s, 3, rho=0.5, n_max=6)
    b = steps(make_ctx(V, O, s, precision, "explicit", monkeypatch), s, 3, rho=0.5, n_max=6)
    c = steps(make_ctx(V, O, s, precision, "compact", monkeypatch), s, 3, rho=0.5, n_max=6)
    assert np.array_equal(a["x"], b["x"]) and np.array_equal(a["x"], c["x"])
    assert np.isfinite(a["x"]).all()


@pytest.mark.parametrize("kg", ["0", "1"])
def test_fp64_tiles_exact_grid_bitwise(V, O, kg, monkeypatch):
    """An fp64 grid with exactly representable spacing has few kinds: the 2-lane tiles run with
    the kind table in shared memory at 2 CTAs/SM (32-byte positions), or with VBD_TILE_KG=1
    from global memory -- both bitwise equal to the explicit layout."""
    m = O.generate_beam(11, 5, 5, 0.25)
    s = O.build_system([(m, (1e6, 1e7, 1e-6))], np.flatnonzero(m.rest_positions[:, 0] < 1e-9))
    monkeypatch.setenv("VBD_TILE_KG", kg)
    monkeypatch.setenv("VBD_TILE_W", "2")  # global kinds are compiled for the 2-lane kernel
    ctx = make_ctx(V, O, s, "fp64", "auto", monkeypatch)
    monkeypatch.delenv("VBD_TILE_KG")
    monkeypatch.delenv("VBD_TILE_W")
    assert ctx.info.tiles > 0 and ctx.info.num_entry_kinds < 100
    a = steps(ctx, s, 4, rho=0.9)
    b = steps(make_ctx(V, O, s, "fp64", "explicit", monkeypatch), s, 4, rho=0.9)
    assert np.array_equal(a["x"], b["x"])


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_irregular_mesh_tiles_bitwise(V, O, precision, seed, monkeypatch):
    """Jittered rest shapes with the default kind cap: thousands of kinds, so the tiles read
    their records from global memory (KG) and every tile's bank placement (DSATUR) sees an
    irregular conflict graph.  Tiles == explicit layout bitwise; both within the north-star
    bar of the oracle."""
    m = O.generate_beam(10, 5, 4, 0.05)
    rng = np.random.default_rng(seed)
    pos = m.rest_positions + rng.uniform(-0.01, 0.01, m.rest_positions.shape)
    mj = O.build_tet_mesh(pos, m.tets, 1000.0)
    s = O.build_system([(mj, (1e6, 1e7, 1e-6))], np.flatnonzero(pos[:, 0] < 0.01))
    monkeypatch.setenv("VBD_TILE_W", "2")  # global kinds are compiled for the 2-lane kernel
    t = make_ctx(V, O, s, precision, "auto", monkeypatch)
    monkeypatch.delenv("VBD_TILE_W")
    assert t.info.tiles > 0 and t.info.num_entry_kinds > 1000
    a = steps(t, s, 4, rho=0.9)
    b = steps(make_ctx(V, O, s, precision, "explicit", monkeypatch), s, 4, rho=0.9)
    assert np.array_equal(a["x"], b["x"])
    st = O.make_state(s)
    for _ in range(4):
        O.step(s, st, H, 10, 0.9, G)
    tol = 1e-10 if precision == "fp64" else 1e-5
    assert np.abs(a["x"] - st.x).max() / mj.bbox_diagonal() <= tol


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-10), ("fp32", 1e-5)])
def test_device_generated_jittered_beam_vs_oracle(V, O, precision, tol):
    """Beam.jitter (the c5j bench scene's irregular rest shapes): every tet its own rest shape,
    so the entry dictionary overflows and the explicit layout runs (fp32: rest edges from the
    rows per entry).  Five steps against the oracle built from the device's rest positions."""
    b = V.Beam(12, 6, 6, 0.05, 2e6, 2e7, 1e-7, fix_min_x=True, jitter=0.1)
    ctx = V.DeviceContext.from_beams([b], precision=precision)
    rest = ctx.get_state(x=True)["x"]
    grid = O.generate_beam(12, 6, 6, 0.05)
    assert np.abs(rest - grid.rest_positions).max() <= 0.1 * 0.05 + 1e-15
    assert (rest[:, 0][grid.rest_positions[:, 0] < 1e-9] == 0.0).all()
    mesh = O.build_tet_mesh(rest, grid.tets, 1000.0)
    fixed = np.flatnonzero(rest[:, 0] < 1e-9)
    s = O.build_system([(mesh, (2e6, 2e7, 1e-7))], fixed)
    assert np.array_equal(ctx.colors(), s.color_of)
    st = O.make_state(s)
    p = ctx.step_params(1 / 240, 10, 0.0, 1e-10, "adaptive", G)
    for _ in range(5):
        ctx.step(p)
        O.step(s, st, 1 / 240, 10, 0.0, G)
    assert ctx.info.layout == 0 or ctx.info.num_entry_kinds > 1000
    err = np.abs(ctx.get_state(x=True)["x"] - st.x).max() / mesh.bbox_diagonal()
    assert err <= tol, err
    ctx.close()


@pytest.mark.parametrize("rho", [0.0, 0.9])
def test_k1t_explicit_rows_bitwise_equals_explicit_k1(V, monkeypatch, rho):
    """K1T-X (irregular mesh through the tile pipeline, rows streamed per slot, constants and
    rest edges derived on the fly) is bitwise the explicit-layout global K1 (VBD_TILES_X=0)."""
    b = V.Beam(14, 9, 7, 0.05, 2e6, 2e7, 1e-7, fix_min_x=True, jitter=0.1)
    out = []
    for xr in ("1", "0"):
        monkeypatch.setenv("VBD_TILES_X", xr)
        monkeypatch.setenv("VBD_RESIDENT", "0")
        monkeypatch.setenv("VBD_LAYOUT", "explicit")  # (a mesh this small fits the entry dictionary)
        ctx = V.DeviceContext.from_beams([b], precision="fp32")
        for k in ("VBD_TILES_X", "VBD_RESIDENT", "VBD_LAYOUT"):
            monkeypatch.delenv(k)
        assert ctx.info.layout == 0
        assert (ctx.info.tiles > 0) == (xr == "1")
        p = ctx.step_params(1 / 240, 10, rho, 1e-10, "adaptive", G)
        for _ in range(3):
            ctx.step(p)
        out.append(ctx.get_state(x=True, v_t=True))
        ctx.close()
    assert np.array_equal(out[0]["x"], out[1]["x"]) and np.array_equal(out[0]["v_t"], out[1]["v_t"])


def class_run(V, monkeypatch, beams, mode, n=3, rho=0.9, n_max=10, h=1 / 240):
    """mode: "class" (K1T with grid-class tiles), "plain" (K1T, VBD_TILE_CLASS=0), "global"
    (the compact global K1)."""
    monkeypatch.setenv("VBD_TILE_CLASS", "0" if mode == "plain" else "1")
    monkeypatch.setenv("VBD_TILE_V", "64")  # class tiles ride on the 64-vertex tile configuration
    monkeypatch.setenv("VBD_ENTRY_ORDER", "code")  # (small scenes keep the kind-hash order)
    monkeypatch.setenv("VBD_RESIDENT", "0")
    monkeypatch.setenv("VBD_TILES", "0" if mode == "global" else "1")
    ctx = V.DeviceContext.from_beams(beams, precision="fp32")
    for k in ("VBD_TILE_CLASS", "VBD_TILE_V", "VBD_RESIDENT", "VBD_TILES", "VBD_ENTRY_ORDER"):
        monkeypatch.delenv(k)
    info = ctx._info()
    p = ctx.step_params(h, n_max, rho, 1e-10, "adaptive", G)
    for _ in range(n):
        ctx.step(p)
    out = ctx.get_state(x=True, v_t=True, v_prev=True)
    ctx.close()
    return out, info


@pytest.mark.parametrize("rho", [0.0, 0.9])
def test_class_tiles_bitwise_equal_plain_tiles(V, monkeypatch, rho):
    """K1T class tiles (interior vertices of the 5-tet grid, one lane per vertex, each distinct
    neighbour loaded once into registers, entries from compile-time indices) are bitwise the
    2-lane tiles (VBD_TILE_CLASS=0) and the global compact K1."""
    beams = [V.Beam(40, 17, 15, 0.01, 2e6, 2e7, 1e-7, fix_min_x=True)]
    a, ia = class_run(V, monkeypatch, beams, "class", rho=rho)
    b, ib = class_run(V, monkeypatch, beams, "plain", rho=rho)
    c, _ = class_run(V, monkeypatch, beams, "global", rho=rho)
    assert ia.class_tiles > 0 and ia.class_records == 40
    # interior vertices: (40 - 1) x 15 x 13 solved interior of 39 x 17 x 15 solved
    assert ia.class_vertices == 38 * 15 * 13
    assert ib.class_tiles == 0
    for k in ("x", "v_t", "v_prev"):
        assert np.array_equal(a[k], b[k]), k
        assert np.array_equal(a[k], c[k]), k


def test_class_tiles_several_instances_and_beams(V, monkeypatch):
    """two beams with different materials and spacings (two instances per class), a twisted
    start (large strains), rho 0.95: still bitwise the plain tiles"""
    beams = [V.Beam(33, 12, 12, 0.01, 2e6, 2e7, 1e-7, fix_min_x=True),
             V.Beam(29, 14, 11, 0.013, 5e5, 4e6, 3e-7, fix_min_x=True, origin=(0.0, 0.3, 0.0))]
    a, ia = class_run(V, monkeypatch, beams, "class", n=4, rho=0.95, h=1 / 120)
    b, _ = class_run(V, monkeypatch, beams, "plain", n=4, rho=0.95, h=1 / 120)
    assert ia.class_tiles > 0 and ia.class_records == 80
    for k in ("x", "v_t", "v_prev"):
        assert np.array_equal(a[k], b[k]), k


def test_class_tiles_from_system_vs_oracle(V, O, monkeypatch):
    """through build_system (the reference's API): class tiles on, 3 steps within the fp32 bar
    of the fp64 oracle, and bitwise the plain tiles"""
    m, s = beam_sys(O, 41, 15, 13, 0.01, (2e6, 2e7, 1e-7))
    xs = []
    for mode in ("1", "0"):
        monkeypatch.setenv("VBD_TILE_CLASS", mode)
        monkeypatch.setenv("VBD_TILE_V", "64")
        monkeypatch.setenv("VBD_RESIDENT", "0")
        monkeypatch.setenv("VBD_ENTRY_ORDER", "code")
        ctx = V.DeviceContext.from_system(O.RefSystemView(s), precision="fp32")
        for k in ("VBD_TILE_CLASS", "VBD_TILE_V", "VBD_RESIDENT", "VBD_ENTRY_ORDER"):
            monkeypatch.delenv(k)
        assert (ctx._info().class_tiles > 0) == (mode == "1")
        xs.append(steps(ctx, s, 3)["x"])
        ctx.close()
    assert np.array_equal(xs[0], xs[1])
    st = O.make_state(s)
    for _ in range(3):
        O.step(s, st, H, 10, 0.9, G)
    assert np.abs(xs[0] - st.x).max() / m.bbox_diagonal() <= 1e-5


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_entry_orders_bitwise_across_layouts(V, O, precision, monkeypatch):
    """both per-vertex entry orders (rest-edge sign pattern / kind hash) give layouts that agree
    bitwise with each other's explicit layout, and stay within the oracle bars"""
    m, s = beam_sys(O)
    st = O.make_state(s)
    for _ in range(3):
        O.step(s, st, H, 10, 0.9, G)
    tol = 1e-10 if precision == "fp64" else 1e-5
    for order in ("code", "hash"):
        monkeypatch.setenv("VBD_ENTRY_ORDER", order)
        a = steps(make_ctx(V, O, s, precision, "auto", monkeypatch), s, 3)["x"]
        b = steps(make_ctx(V, O, s, precision, "explicit", monkeypatch), s, 3)["x"]
        monkeypatch.delenv("VBD_ENTRY_ORDER")
        assert np.array_equal(a, b), order
        assert np.abs(a - st.x).max() / m.bbox_diagonal() <= tol
