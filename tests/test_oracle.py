"""The oracle (oracle/) pinned against the reference: golden vectors written by
the reference itself (tests/golden/make_golden.py) and, when oracle/_ref is
present, the reference's compiled colour-pass kernel run live on the same inputs.
CPU only."""

import numpy as np
import pytest

G = (0.0, 0.0, -9.8)


def _beam_system(O, nx=9, ny=4, nz=4, spacing=0.05, mat=(1e6, 1e7, 1e-6)):
    m = O.generate_beam(nx, ny, nz, spacing)
    fixed = np.flatnonzero(m.rest_positions[:, 0] < 1e-9)
    return m, fixed, O.build_system([(m, mat)], fixed)


def test_mesh_arrays_match_reference(O, golden):
    g = golden("mesh_beam_5_3_3.npz")
    m = O.generate_beam(5, 3, 3, 0.1)
    for k in ("rest_positions", "tets", "rest_volumes", "inv_rest_shape", "masses"):
        assert np.array_equal(getattr(m, k), g[k]), k
    off, ids, slots = O.incidence_from_elements(m.tets, m.num_vertices)
    assert np.array_equal(off, g["elem_offsets"])
    assert np.array_equal(ids, g["elem_ids"])
    assert np.array_equal(slots, g["elem_slots"])
    noff, nids = O.merged_adjacency(m.num_vertices, [m.tets])
    assert np.array_equal(noff, g["neighbor_offsets"])
    assert np.array_equal(nids, g["neighbor_ids"])
    s = O.build_system([(m, (2e5, 8e5, 0.01))])
    assert np.array_equal(s.tet_w, g["tet_w"])
    assert np.array_equal(s.color_of, g["color_of"])
    assert np.array_equal(s.color_verts, g["color_verts"])


def test_beam_connectivity_c_matches_python_loop(O):
    for dims in ((2, 2, 2), (3, 4, 5), (6, 2, 3)):
        assert np.array_equal(O.beam_tets(*dims), O.beam_tets_py(*dims))


@pytest.mark.parametrize("name,build", [
    ("c1", lambda O: [O.generate_beam(41, 11, 11, 0.025)]),
    ("c2", lambda O: [O.generate_cube(37, 0.5)]),
    ("c3", lambda O: [O.generate_beam(3032, 4, 4, 0.01)] * 2),
    ("twobody", lambda O: [O.generate_beam(9, 4, 4, 0.05), O.generate_cube(5, 0.3)]),
    ("c4obj", lambda O: [O.generate_cube(15, 0.3)]),
])
def test_greedy_color_bit_exact(O, golden, name, build):
    g = golden(f"color_{name}.npz")
    s = O.build_system([(m, (1e6, 1e7, 1e-6)) for m in build(O)])
    assert s.num_vertices == int(g["n"]) and len(s.tets) == int(g["t"])
    assert np.array_equal(s.color_of, g["color_of"].astype(np.int64))
    assert np.array_equal(s.color_off, g["color_off"])


def test_greedy_c_matches_literal_python(O):
    m = O.generate_beam(7, 5, 4, 0.1)
    noff, nids = O.merged_adjacency(m.num_vertices, [m.tets])
    a, _ = O.greedy_color(noff, nids)
    b, _ = O.greedy_color_py(noff, nids)
    assert np.array_equal(a, b)


def test_color_pass_bit_exact(O, golden):
    g = golden("pass_beam_9_4_4.npz")
    m, fixed, s = _beam_system(O)
    assert np.array_equal(fixed, g["fixed"])
    h = float(g["h"])
    x = g["x0"].copy()
    for c, grp in enumerate(s.groups()):
        O.color_pass(s, x, g["x_t"], g["y"], h, grp)
        assert np.array_equal(x, g[f"after_color{c}"]), c
    allv = np.arange(s.num_vertices)
    for mode in (0, 1):
        x = g["x0"].copy()
        O.color_pass(s, x, g["x_t"], g["y"], h, allv, mode=mode)
        assert np.array_equal(x, g[f"jacobi_mode{mode}"])
    x = g["x0"].copy()
    O.color_pass(s, x, g["x_t"], g["y"], h, allv, line_search=True)
    assert np.array_equal(x, g["jacobi_linesearch"])


@pytest.mark.parametrize("rho", [0.0, 0.9])
def test_step_trajectory_bit_exact(O, golden, rho):
    g = golden(f"steps_beam_rho{int(rho * 100):02d}.npz")
    m, fixed, s = _beam_system(O)
    st = O.make_state(s)
    for k in range(10):
        O.step(s, st, 1.0 / 60.0, 10, rho, G)
        assert np.array_equal(st.x, g["x"][k]), k
        assert np.array_equal(st.v_t, g["v"][k]), k


def test_c1_ten_steps_bit_exact(O, golden):
    g = golden("steps_c1.npz")
    m, fixed, s = _beam_system(O, 41, 11, 11, 0.025)
    st = O.make_state(s)
    for k in range(10):
        O.step(s, st, 1.0 / 60.0, 10, 0.0, G)
        if k == 0:
            assert np.array_equal(st.x, g["x_step1"])
    assert np.array_equal(st.x, g["x_step10"])


def test_extreme_init_bit_exact(O, golden):
    g = golden("steps_extreme_cube6.npz")
    m = O.generate_cube(6, 0.5)
    s = O.build_system([(m, (2e6, 1e7, 1e-6))])
    st = O.make_state(s, x0=g["x0"])
    for k in range(3):
        O.step(s, st, 1.0 / 60.0, 100, 0.95)
        assert np.array_equal(st.x, g["x"][k]), k


def test_thread_count_independent(O):
    m, fixed, s = _beam_system(O, 13, 6, 6)
    rng = np.random.default_rng(3)
    x0 = s.rest_positions + 0.003 * rng.standard_normal(s.rest_positions.shape)
    y = s.rest_positions.copy()
    outs = []
    for nt in (1, 2, 7):
        x = x0.copy()
        O.color_pass(s, x, s.rest_positions, y, 1 / 60, np.arange(s.num_vertices), n_threads=nt)
        outs.append(x)
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_oracle_matches_reference_kernel_live(O):
    ref = O.ref_native()
    if ref is None:
        pytest.skip("oracle/_ref not built (make -C oracle ref)")
    m, fixed, s = _beam_system(O, 13, 6, 6)
    a, b = O.make_state(s), O.make_state(s)
    for _ in range(3):
        O.step(s, a, 1 / 30, 20, 0.95, G)
        O.step(s, b, 1 / 30, 20, 0.95, G, kernel=ref, n_threads=1)
        assert np.array_equal(a.x, b.x)


# ------------------------------------------------------------------------------------
# springs, subspace and world-box constraints (_native.pyx:319-349, 401-409, 435-463)

def test_extras_passes_bit_exact(O, golden):
    from extras import extras_system
    g = golden("extras_scene.npz")
    m, s = extras_system(O, g)
    h = float(g["h"])
    x = g["x0"].copy()
    for c, grp in enumerate(s.groups()):
        O.color_pass(s, x, g["x_t"], g["y"], h, grp)
        assert np.array_equal(x, g[f"after_color{c}"]), c
    allv = np.arange(s.num_vertices)
    for mode in (0, 1):
        x = g["x0"].copy()
        O.color_pass(s, x, g["x_t"], g["y"], h, allv, mode=mode)
        assert np.array_equal(x, g[f"jacobi_mode{mode}"]), mode
    x = g["x0"].copy()
    O.color_pass(s, x, g["x_t"], g["y"], h, allv, line_search=True)
    assert np.array_equal(x, g["jacobi_linesearch"])


@pytest.mark.parametrize("rho", [0.0, 0.9])
def test_extras_steps_bit_exact(O, golden, rho):
    from extras import extras_system
    g = golden("extras_scene.npz")
    m, s = extras_system(O, g)
    st = O.make_state(s)
    xs = g[f"steps_rho{int(rho * 100):02d}"]
    for k in range(len(xs)):
        O.step(s, st, 1.0 / 60.0, 15, rho, G)
        assert np.array_equal(st.x, xs[k]), k
    # the cloth reached the box floor and the subspace vertices stayed on their subspaces
    nb = m.num_vertices
    assert (st.x[nb:nb + 25, 2] < 0.185).any()
    assert abs(st.x[nb - 1, 0] - m.rest_positions[-1, 0]) < 1e-12
    assert abs(st.x[nb - 2, 2] - m.rest_positions[-2, 2]) < 1e-12


def test_energy_bit_exact(O, golden):
    """G = 1/(2h^2)|x - y|_M^2 + E(x) (_assembly.py:78-82) at iterates recorded by the
    reference's own baselines.energy."""
    from extras import extras_system
    g = golden("energy.npz")
    m, s = extras_system(O, golden("extras_scene.npz"))
    for k in range(len(g["extras_G"])):
        assert O.variational_energy(s, g["extras_x"][k], g["extras_y"][k], 1 / 60) == g["extras_G"][k]
    m, fixed, sb = _beam_system(O)
    for k in range(len(g["beam_G"])):
        assert O.variational_energy(sb, g["beam_x"][k], g["beam_y"][k], 1 / 60) == g["beam_G"][k]


def test_contact_passes_bit_exact(O, golden):
    """Colour passes with contact + friction terms (_native.pyx:351-399, gammas refreshed
    for DCD vertex-triangle anchors, :134-172) recorded at the reference's kernel seam."""
    from extras import ContactCall, contact_system
    g = golden("contact_scene.npz")
    s = contact_system(O)
    h = float(g["h"])
    for k in range(int(g["num_calls"])):
        x = g[f"call{k}_x0"].copy()
        O.color_pass(s, x, g[f"call{k}_x_t"], g[f"call{k}_y"], h, g[f"call{k}_group"],
                     carr=ContactCall(g, k), mu_c=float(g[f"call{k}_mu_c"]),
                     eps_v=float(g[f"call{k}_eps_v"]))
        assert np.array_equal(x, g[f"call{k}_x1"]), k
        assert not np.array_equal(x, g[f"call{k}_x0"])


# --------------------------------------------------------------------------------------
# BASELINE configs' own settings (tests/golden/make_golden.py::config_fixtures)


def c2_full_system(O):
    m = O.generate_cube(37, 0.5)
    s = O.build_system([(m, (2e6, 1e7, 1e-6))])
    lo, hi = m.rest_positions.min(0), m.rest_positions.max(0)
    x0 = np.random.default_rng(0).uniform(lo, hi, size=m.rest_positions.shape)
    return m, s, x0


def test_c2_full_color_passes_bit_exact(O, golden):
    """C2 at full size (37^3): the first iteration's colour passes on identical inputs."""
    g = golden("c2_full.npz")
    m, s, x0 = c2_full_system(O)
    x = x0.copy()
    for c, grp in enumerate(s.groups()):
        O.color_pass(s, x, x0, x0, 1.0 / 60.0, grp)
        assert np.array_equal(x[grp], g[f"after_color{c}"]), c


def test_c2_full_first_step_bit_exact(O, golden):
    g = golden("c2_full.npz")
    m, s, x0 = c2_full_system(O)
    st = O.make_state(s, x0=x0)
    O.step(s, st, 1.0 / 60.0, 100, 0.95, (0.0, 0.0, 0.0))
    assert np.array_equal(st.x, g["x_step1"])


def test_c4_object_steps_bit_exact(O, golden):
    """The first C4 object (cube 15, z=1, rigid velocity) at C4's material/h/n_max."""
    g = golden("c4obj_steps.npz")
    m0 = O.generate_cube(15, 0.3)
    m = O.build_tet_mesh(m0.rest_positions + np.array([0.0, 0.0, 1.0]), m0.tets, 1000.0)
    s = O.build_system([(m, (1e6, 1e7, 1e-7))], [])
    st = O.make_state(s, v0=g["v0"])
    want = dict(zip(g["steps"].tolist(), g["x"]))
    for k in range(1, 11):
        O.step(s, st, 1.0 / 120.0, 60, 0.0, G)
        if k in want:
            assert np.array_equal(st.x, want[k]), k


def test_c5_block_first_step_bit_exact(O, golden):
    """32^3 block with C5's material, h, n_max and fixed face."""
    g = golden("c5block_steps.npz")
    m, fixed, s = _beam_system(O, 32, 32, 32, 0.01, mat=(2e6, 2e7, 1e-7))
    assert np.array_equal(fixed, g["fixed"])
    st = O.make_state(s)
    O.step(s, st, 1.0 / 240.0, 40, 0.0, G)
    assert np.array_equal(st.x, g["x"][0])


def test_fp32_oracle_is_the_same_algorithm_in_binary32(O):
    """liboracle_f32.so (the fp32 sensitivity yardstick of test_gpu_configs) runs the same
    restatement in binary32: on a well-conditioned beam pass it agrees with the fp64 oracle to
    fp32 rounding, and its result is exactly representable in float32."""
    m, fixed, s = _beam_system(O)
    rng = np.random.default_rng(3)
    x0 = s.rest_positions + rng.normal(scale=1e-3, size=s.rest_positions.shape)
    diag = m.bbox_diagonal()
    for grp in s.groups():
        x = x0.copy()
        O.color_pass(s, x, s.rest_positions, s.rest_positions, 1.0 / 60.0, grp)
        r = O.color_pass_fp32(s, x0, s.rest_positions, s.rest_positions, 1.0 / 60.0, grp)
        assert np.array_equal(r.astype(np.float32).astype(np.float64), r)
        err = np.abs(r - x[grp]).max() / diag
        assert 0 < err < 1e-5, err
