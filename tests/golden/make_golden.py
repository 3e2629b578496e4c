"""Regenerate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container (where /root/reference exists):

    make -C oracle ref            # the reference's compiled kernel -> oracle/_ref
    python tests/golden/make_golden.py

It imports the unmodified reference package (/root/reference/pkg/src/vbdsim),
with its compiled ``_native`` extension supplied by oracle/_ref (built from the
reference's own committed ``_native.c``), and records inputs + outputs of the
functions on the hot path:

* generate_beam/build_tet_mesh arrays          (harness.py:42-76, mesh.py:128-170)
* incidence and merged adjacency               (mesh.py:232-267, _system.py:147-169)
* greedy_color on the BASELINE configs C1/C2/C3 (mesh.py:270-302)
* color_pass outputs for every colour group, all-vertex Jacobi pass (mode 0/1)
  and the line-search variant               (_native.pyx:513-589)
* step() trajectories                          (solver.py:291-324)

The fixtures are small (.npz) and committed; the GPU box never reads
/root/reference.
"""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from oracle import oracle as O  # noqa: E402

native = O.ref_native()
if native is None:
    raise SystemExit("build the reference kernel first: make -C oracle ref")
sys.modules["vbdsim._native"] = native

import vbdsim  # noqa: E402
from vbdsim import (Body, FixedConstraint, MaterialParams, SolverParams,  # noqa: E402
                    build_system, color_pass, generate_beam, generate_cube,
                    inertia_target, initialize, make_state, step)
from vbdsim._system import _merged_adjacency  # noqa: E402
from vbdsim.mesh import incidence  # noqa: E402

assert vbdsim.backend_name() == "native"
G = (0.0, 0.0, -9.8)


def save(name, **arrays):
    np.savez_compressed(OUT / name, **arrays)
    print("wrote", name, sum(a.nbytes for a in map(np.asarray, arrays.values())), "bytes")


def mesh_fixture():
    m = generate_beam(5, 3, 3, 0.1, density=1000.0)
    adj = incidence(m)
    sysm = build_system([Body(m, MaterialParams(2e5, 8e5, 0.01))])
    madj = _merged_adjacency(m.num_vertices, [m.tets])
    noff, nids = madj.neighbor_offsets, madj.neighbor_ids
    save("mesh_beam_5_3_3.npz", rest_positions=m.rest_positions, tets=m.tets,
         rest_volumes=m.rest_volumes, inv_rest_shape=m.inv_rest_shape, masses=m.masses,
         elem_offsets=adj.elem_offsets, elem_ids=adj.elem_ids, elem_slots=adj.elem_slots,
         neighbor_offsets=noff, neighbor_ids=nids, tet_w=sysm.tet_w,
         color_of=sysm.colors.color_of, color_off=sysm.color_off, color_verts=sysm.color_verts)


def coloring_fixtures():
    scenes = {
        "c1": [generate_beam(41, 11, 11, 0.025)],
        "c2": [generate_cube(37, 0.5)],
        "c3": [generate_beam(3032, 4, 4, 0.01), generate_beam(3032, 4, 4, 0.01)],
        "twobody": [generate_beam(9, 4, 4, 0.05), generate_cube(5, 0.3)],
        "c4obj": [generate_cube(15, 0.3)],
    }
    for name, meshes in scenes.items():
        s = build_system([Body(m, MaterialParams(1e6, 1e7, 1e-6)) for m in meshes])
        save(f"color_{name}.npz", color_of=s.colors.color_of.astype(np.int8),
             color_off=s.color_off, n=np.int64(s.num_vertices), t=np.int64(len(s.tets)))


def beam_system(nx=9, ny=4, nz=4, spacing=0.05, mat=(1e6, 1e7, 1e-6)):
    m = generate_beam(nx, ny, nz, spacing, density=1000.0)
    fixed = np.flatnonzero(m.rest_positions[:, 0] < 1e-9)
    s = build_system([Body(m, MaterialParams(*mat))], [FixedConstraint(int(v)) for v in fixed])
    return m, fixed, s


def pass_fixture():
    m, fixed, s = beam_system()
    st = make_state(s)
    rng = np.random.default_rng(7)
    st.v_t = 0.3 * rng.standard_normal(st.x.shape)
    p = SolverParams(h=1.0 / 60.0, a_ext=G, threads=1)
    st.y = inertia_target(st.x_t, st.v_t, p.a_ext_vec, p.h)
    initialize(st, p)
    st.x = np.ascontiguousarray(st.x + 0.004 * rng.standard_normal(st.x.shape))
    x0 = st.x.copy()
    outs = {}
    off = s.color_off
    x = x0.copy()
    for g in range(s.colors.num_colors):
        st.x = x
        color_pass(st, s.color_verts[off[g]:off[g + 1]], p)
        outs[f"after_color{g}"] = st.x.copy()
        x = st.x.copy()
    allv = np.arange(s.num_vertices, dtype=np.int64)
    for mode in (0, 1):
        st.x = x0.copy()
        color_pass(st, allv, p, mode=mode)
        outs[f"jacobi_mode{mode}"] = st.x.copy()
    st.x = x0.copy()
    color_pass(st, allv, SolverParams(h=1.0 / 60.0, a_ext=G, threads=1, line_search=True))
    outs["jacobi_linesearch"] = st.x.copy()
    save("pass_beam_9_4_4.npz", x0=x0, x_t=st.x_t, y=st.y, fixed=fixed, h=np.float64(p.h),
         mu=np.float64(1e6), lam=np.float64(1e7), kd=np.float64(1e-6), **outs)


def step_fixtures():
    # C1-like: small cantilever under gravity, plain and Chebyshev-accelerated
    for rho in (0.0, 0.9):
        m, fixed, s = beam_system()
        st = make_state(s)
        p = SolverParams(h=1.0 / 60.0, n_max=10, rho=rho, a_ext=G, threads=1)
        xs, vs = [], []
        for _ in range(10):
            step(st, p)
            xs.append(st.x.copy())
            vs.append(st.v_t.copy())
        save(f"steps_beam_rho{int(rho * 100):02d}.npz", x=np.array(xs), v=np.array(vs),
             fixed=fixed, n_max=np.int64(10), rho=np.float64(rho), h=np.float64(p.h))
    # BASELINE config 1 at full size, 10 steps
    m = generate_beam(41, 11, 11, 0.025, density=1000.0)
    fixed = np.flatnonzero(m.rest_positions[:, 0] < 1e-9)
    s = build_system([Body(m, MaterialParams(1e6, 1e7, 1e-6))],
                     [FixedConstraint(int(v)) for v in fixed])
    st = make_state(s)
    p = SolverParams(h=1.0 / 60.0, n_max=10, a_ext=G, threads=1)
    xs = []
    for k in range(10):
        step(st, p)
        if k in (0, 9):
            xs.append(st.x.copy())
    save("steps_c1.npz", x_step1=xs[0], x_step10=xs[1], fixed=fixed)
    # extreme initialisation (BASELINE config 2 at reduced size)
    m = generate_cube(6, 0.5, density=1000.0)
    s = build_system([Body(m, MaterialParams(2e6, 1e7, 1e-6))])
    rng = np.random.default_rng(0)
    lo, hi = m.rest_positions.min(0), m.rest_positions.max(0)
    x0 = rng.uniform(lo, hi, size=m.rest_positions.shape)
    st = make_state(s, x0=x0)
    p = SolverParams(h=1.0 / 60.0, n_max=100, rho=0.95, threads=1)
    xs = []
    for _ in range(3):
        step(st, p)
        xs.append(st.x.copy())
    save("steps_extreme_cube6.npz", x0=x0, x=np.array(xs))


def extras_scene():
    """A beam + a spring cloth + a spring chain, with fixed, subspace and world-box
    constraints: the non-tet terms of _assemble / _solve_vertex (_native.pyx:319-349,
    401-409, 435-463) and _local_energy (:226-257)."""
    from vbdsim import SubspaceConstraint, WorldBoxConstraint, build_spring_net, generate_chain
    m = generate_beam(7, 3, 3, 0.05, density=1000.0)
    P = 5
    xs_, ys_ = np.meshgrid(np.arange(P), np.arange(P), indexing="ij")
    parts = np.stack([0.5 + 0.05 * xs_.ravel(), 0.05 * ys_.ravel(), np.full(P * P, 0.2)], 1)
    rows = []
    for i in range(P):
        for j in range(P):
            v = i * P + j
            for w in ([v + P] if i + 1 < P else []) + ([v + 1] if j + 1 < P else []) + \
                     ([v + P + 1] if i + 1 < P and j + 1 < P else []):
                rows.append([v, w, float(np.linalg.norm(parts[v] - parts[w])), 500.0])
    cloth = build_spring_net(parts, rows, np.full(P * P, 0.01))
    chain = generate_chain(6, 0.04, 300.0, mass=0.02)
    nb, nc = m.num_vertices, cloth.num_vertices
    fixed = [int(v) for v in np.flatnonzero(m.rest_positions[:, 0] < 1e-9)] + [nb, nb + nc]
    cons = [FixedConstraint(v) for v in fixed]
    cons.append(SubspaceConstraint(nb - 1, np.array([[0.0], [0.0], [1.0]]), m.rest_positions[-1]))
    cons.append(SubspaceConstraint(nb - 2, np.array([[1.0, 0.0], [0.0, 1.0], [0.0, 0.0]]),
                                   m.rest_positions[-2]))
    boxes = [(nb + v, (-1.0, -1.0, 0.185), (2.0, 2.0, 1.0), 1e4) for v in range(nc)]
    cons += [WorldBoxConstraint(v, lo, hi, k) for v, lo, hi, k in boxes]
    s = build_system([Body(m, MaterialParams(1e6, 1e7, 1e-6)),
                      Body(cloth, k_d=1e-3), Body(chain, k_d=5e-4)], cons)
    sub = [(nb - 1, [[0.0], [0.0], [1.0]], m.rest_positions[-1]),
           (nb - 2, [[1.0, 0.0], [0.0, 1.0], [0.0, 0.0]], m.rest_positions[-2])]
    return m, cloth, chain, fixed, sub, boxes, s


def extras_fixture():
    m, cloth, chain, fixed, sub, boxes, s = extras_scene()
    st = make_state(s)
    rng = np.random.default_rng(11)
    st.v_t = 0.2 * rng.standard_normal(st.x.shape)
    p = SolverParams(h=1.0 / 60.0, a_ext=G, threads=1)
    st.y = inertia_target(st.x_t, st.v_t, p.a_ext_vec, p.h)
    initialize(st, p)
    st.x = np.ascontiguousarray(st.x + 0.004 * rng.standard_normal(st.x.shape))
    x0 = st.x.copy()
    outs = {}
    off = s.color_off
    x = x0.copy()
    for g in range(s.colors.num_colors):
        st.x = x
        color_pass(st, s.color_verts[off[g]:off[g + 1]], p)
        outs[f"after_color{g}"] = st.x.copy()
        x = st.x.copy()
    allv = np.arange(s.num_vertices, dtype=np.int64)
    for mode in (0, 1):
        st.x = x0.copy()
        color_pass(st, allv, p, mode=mode)
        outs[f"jacobi_mode{mode}"] = st.x.copy()
    st.x = x0.copy()
    color_pass(st, allv, SolverParams(h=1.0 / 60.0, a_ext=G, threads=1, line_search=True))
    outs["jacobi_linesearch"] = st.x.copy()
    # trajectories: the cloth falls onto the box floor, the chain swings
    trajs = {}
    for rho in (0.0, 0.9):
        st2 = make_state(s)
        p2 = SolverParams(h=1.0 / 60.0, n_max=15, rho=rho, a_ext=G, threads=1)
        xs = []
        for _ in range(8):
            step(st2, p2)
            xs.append(st2.x.copy())
        trajs[f"steps_rho{int(rho * 100):02d}"] = np.array(xs)
    save("extras_scene.npz", x0=x0, x_t=st.x_t, y=st.y, h=np.float64(p.h),
         cloth_parts=cloth.particles, cloth_idx=cloth.indices, cloth_l0=cloth.rest_length,
         cloth_k=cloth.stiffness, cloth_m=cloth.masses, chain_parts=chain.particles,
         chain_idx=chain.indices, chain_l0=chain.rest_length, chain_k=chain.stiffness,
         chain_m=chain.masses, fixed=np.array(fixed), color_of=s.colors.color_of,
         **outs, **trajs)


def energy_fixture():
    """G = baselines.energy (_assembly.py:78-82) at a few iterates of the extras scene and
    of the beam (metrics path of harness.run_simulation, harness.py:664-678)."""
    from vbdsim import baselines
    out = {}
    for name, scene in (("extras", lambda: extras_scene()[-1]), ("beam", lambda: beam_system()[2]),
                        ("contact", lambda: contact_scene()[0])):
        s = scene()
        st = make_state(s)
        p = SolverParams(h=1.0 / 60.0, n_max=10, rho=0.5, a_ext=G, threads=1)
        if name == "contact":
            p = contact_scene()[1]
        xs, ys, gs = [], [], []

        def rec(state, n):
            xs.append(state.x.copy())
            ys.append(state.y.copy())
            gs.append(baselines.energy(state, p))
        for _ in range(2):
            step(st, p, on_iteration=rec)
        out[f"{name}_x"] = np.array(xs[::5])
        out[f"{name}_y"] = np.array(ys[::5])
        out[f"{name}_G"] = np.array(gs[::5])
    save("energy.npz", **out)


def contact_scene():
    """A heavy cube resting on a light cube with a fixed base (a small version of the
    reference's extreme-mass-ratio acceptance scene, test_acceptance.py:419-433)."""
    from vbdsim import ContactParams, build_tet_mesh
    n = 4
    light = generate_beam(n, n, n, 0.3 / (n - 1), density=10.0)
    heavy0 = generate_beam(n, n, n, 0.2 / (n - 1), density=2000.0)
    heavy = build_tet_mesh(heavy0.rest_positions + [0.05, 0.05, 0.3005], heavy0.tets, 2000.0)
    bottom = [i for i in range(light.num_vertices) if light.rest_positions[i, 2] < 1e-9]
    s = build_system([Body(light, MaterialParams(1e6, 1e7), k_d=0.01),
                      Body(heavy, MaterialParams(1e6, 1e7), k_d=0.01)],
                     [FixedConstraint(i) for i in bottom])
    p = SolverParams(h=1.0 / 120.0, n_max=10, threads=1, a_ext=G,
                     contact=ContactParams(k_c=1e6, mu_c=0.5, eps_v=1e-3))
    return s, p


def contact_fixture():
    """Colour passes with contacts (_native.pyx:351-399) recorded at the kernel seam, and the
    trajectory of the reference's own step() (DCD/CCD, solver.py:241-324)."""
    from vbdsim import _backend
    s, p = contact_scene()
    native = _backend._impl
    calls = []
    seen = [0]

    class Rec:
        NAME = native.NAME

        @staticmethod
        def color_pass(system, carr, x, x_t, y, h, group, mode=0, **kw):
            before = x.copy()
            native.color_pass(system, carr, x, x_t, y, h, group, mode, **kw)
            seen[0] += 1
            if carr is not None and carr.count and len(calls) < 8 and len(group) > 20 and seen[0] % 19 == 1:
                calls.append(dict(x0=before, x_t=x_t.copy(), y=y.copy(), group=np.array(group),
                                  x1=x.copy(), mu_c=kw["mu_c"], eps_v=kw["eps_v"], idx=carr.idx,
                                  gamma=carr.gamma, refresh=carr.refresh, normal=carr.normal,
                                  tangent=carr.tangent, k_c=carr.k_c, cv_off=carr.cv_off,
                                  cv_cid=carr.cv_cid, cv_slot=carr.cv_slot))
    _backend._impl = Rec
    try:
        st = make_state(s)
        xs, counts, flags = [], [], []
        for _ in range(4):
            step(st, p)
            xs.append(st.x.copy())
            counts.append(len(st.contact_set))
    finally:
        _backend._impl = native
    out = {"steps": np.array(xs), "contact_counts": np.array(counts), "h": np.float64(p.h)}
    for k, c in enumerate(calls):
        for name, v in c.items():
            out[f"call{k}_{name}"] = np.asarray(v)
    out["num_calls"] = np.int64(len(calls))
    save("contact_scene.npz", **out)
    contact_detection_fixture()


def contact_detection_fixture():
    """The reference's own contact sets right after each DCD / CCD pass of the contact scene
    (solver.py:241-279, contact.py): inputs x_t, x and the records in order."""
    from vbdsim import solver as S
    s, p = contact_scene()
    rec = []
    dcd0, ccd0 = S._detect_dcd, S._detect_ccd

    def snap(tag, state):
        cs = state.contact_set
        lst = cs.dcd if tag == "dcd" else cs.ccd
        rec.append(dict(kind=tag, x_t=state.x_t.copy(), x=state.x.copy(),
                        idx=np.array([c.indices for c in lst], dtype=np.int64).reshape(-1, 4),
                        gamma=np.array([c.gammas() for c in lst]).reshape(-1, 4),
                        normal=np.array([c.normal for c in lst]).reshape(-1, 3),
                        ee=np.array([c.kind == "ee" for c in lst], dtype=bool),
                        flags=cs.colliding_flag.copy()))

    def dcd(state, params):
        dcd0(state, params)
        snap("dcd", state)

    def ccd(state, params):
        ccd0(state, params)
        snap("ccd", state)
    S._detect_dcd, S._detect_ccd = dcd, ccd
    try:
        st = make_state(s)
        for _ in range(4):
            step(st, p)
    finally:
        S._detect_dcd, S._detect_ccd = dcd0, ccd0
    out = {"num": np.int64(len(rec))}
    for k, r in enumerate(rec):
        out[f"r{k}_which"] = np.int64(0 if r["kind"] == "dcd" else 1)
        for name in ("x_t", "x", "idx", "gamma", "normal", "ee", "flags"):
            out[f"r{k}_{name}"] = r[name]
    save("contact_detection.npz", **out)


# --------------------------------------------------------------------------------------------
# harness: scene schema, scene_build, frames, run_simulation, CLI (harness.py, cli.py)

HARNESS_BASE = {
    "objects": [{"generator": {"kind": "beam", "nx": 3, "ny": 2, "nz": 2, "spacing": 0.1},
                 "material": {"mu": 1e5, "lambda": 4e5, "k_d": 0.001}, "density": 1000.0}],
    "gravity": [0.0, 0.0, -9.8],
    "constraints": [{"kind": "fixed", "object": 0, "box": [[-1e-6, -1e-6, -1e-6], [1e-6, 0.2, 0.2]]}],
    "solver": {"h": 0.005, "n_max": 6},
    "frames": 2,
    "output": {"format": "bin", "every": 1},
}


def harness_scenes():
    """Scenes run through the reference's run_simulation (small enough for its CPU path)."""
    import copy
    import json
    base = copy.deepcopy(HARNESS_BASE)
    placed = {
        "objects": [{"generator": {"kind": "beam", "nx": 6, "ny": 3, "nz": 3, "spacing": 0.05},
                     "material": {"mu": 2e5, "lambda": 1e6, "k_d": 1e-4}, "density": 800.0,
                     "translate": [0.5, -0.2, 1.0], "rotate_deg": [10.0, 20.0, 30.0],
                     "scale": [1.2, 1.0, 0.9], "velocity": [0.1, 0.0, -0.3],
                     "initial_stretch": [1.05, 0.98, 1.0]}],
        "gravity": [0.0, -9.8, 0.0],
        "constraints": [{"kind": "fixed", "object": 0, "vertices": [0, 1, 2]}],
        "solver": {"S": 2, "n_max": 5, "rho": 0.5, "line_search": "local_backtracking"},
        "frames": 2, "output": {"format": "obj", "every": 1}}
    mixed = {
        "objects": [{"generator": {"kind": "beam", "nx": 5, "ny": 3, "nz": 3, "spacing": 0.05},
                     "material": {"mu": 1e5, "lambda": 5e5}},
                    {"generator": {"kind": "chain", "count": 6, "spacing": 0.04, "stiffness": 800.0,
                                   "mass": 0.05},
                     "material": {"mu": 1.0, "lambda": 1.0, "k_d": 1e-3},
                     "translate": [0.0, 0.5, 0.3], "scale": 1.5},
                    {"generator": {"kind": "cube", "n": 3, "edge": 0.1}, "material":
                     {"mu": 3e5, "lambda": 1e6}, "translate": [0.5, 0.0, 0.0]}],
        "gravity": [0.0, 0.0, -9.8],
        "constraints": [{"kind": "fixed", "object": 0, "box": [[-1, -1, -1], [1e-9, 1, 1]]},
                        {"kind": "fixed", "object": 1, "vertices": [0]},
                        {"kind": "subspace", "object": 0, "vertex": 44, "basis": [[0, 0, 1]]},
                        {"kind": "subspace", "object": 2, "vertex": 26,
                         "basis": [[1, 0, 0], [0, 1, 0]], "anchor": [0.6, 0.1, 0.1]},
                        {"kind": "world_box", "lo": [-5, -5, -0.02], "hi": [5, 5, 5], "k_b": 1e4},
                        {"kind": "world_box", "object": 2, "lo": [-5, -5, 0.0], "hi": [5, 5, 5],
                         "k_b": 5e3}],
        "solver": {"h": 1 / 120, "n_max": 8, "init_mode": "inertia", "eps_det": 1e-9},
        "frames": 3, "output": {"format": "bin", "every": 2}}
    contact = {
        "objects": [{"generator": {"kind": "cube", "n": 4, "edge": 0.3},
                     "material": {"mu": 5e4, "lambda": 2e5, "k_d": 1e-4}, "density": 10.0},
                    {"generator": {"kind": "cube", "n": 4, "edge": 0.2},
                     "material": {"mu": 5e5, "lambda": 2e6, "k_d": 1e-4}, "density": 2000.0,
                     "translate": [0.05, 0.05, 0.3005], "velocity": [0.0, 0.0, -0.5]}],
        "gravity": [0.0, 0.0, -9.8],
        "constraints": [{"kind": "fixed", "object": 0, "box": [[-1, -1, -1], [1, 1, 1e-9]]}],
        "contact": {"k_c": 1e6, "mu_c": 0.3, "eps_v": 1e-2, "dcd_radius": 2e-3},
        "solver": {"h": 1 / 120, "n_max": 8, "n_col": 3},
        "frames": 3, "output": {"format": "bin", "every": 1}}
    return {"base": json.dumps(base), "placed": json.dumps(placed), "mixed": json.dumps(mixed),
            "contact": json.dumps(contact)}


HARNESS_BAD = [
    '{nope',
    '{"objects": []}',
    '{"objects": [{"generator": {"kind": "beam", "nx": 3, "ny": 2, "nz": 2, "spacing": 0.1}}]}',
    '{"objects": [{"generator": {"kind": "tube"}, "material": {"mu": 1, "lambda": 1}}]}',
    '{"objects": [{"generator": {"kind": "beam", "nx": 1, "ny": 2, "nz": 2, "spacing": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}}]}',
    '{"objects": [{"generator": {"kind": "beam", "nx": 3, "ny": 2, "nz": 2, "spacing": "a"}, '
    '"material": {"mu": 1, "lambda": 1}}]}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": -1}}]}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}, "scale": [1, 0, 1]}]}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}, "translate": [1, 2]}]}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}}], "solver": {"h": "fast"}}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}}], "solver": {"h": -0.5}}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}}], "solver": {"rho": 1.0}}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}}], "solver": {"S": 0}}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}}], "solver": {"n_max": 2.5}}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}}], "solver": {"line_search": "on"}}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}}], "solver": {"init_mode": "zero"}}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}}], "solver": {"dt": 0.1}}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}}], "contact": {"mu_c": 0.1}}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}}], "contact": {"k_c": 1e7, "mu_c": -2.0}}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}}], "constraints": [{"kind": "fixed", "object": 0}]}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}}], "constraints": [{"kind": "fixed", "object": 3, '
    '"vertices": [0]}]}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}}], "constraints": [{"kind": "subspace", "object": 0, '
    '"vertex": 0, "basis": [[1, 0]]}]}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}}], "constraints": [{"kind": "world_box", '
    '"lo": [0, 0, 0], "hi": [1, 1, 1]}]}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}}], "frames": -1}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}}], "output": {"format": "vtk"}}',
    '{"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}, '
    '"material": {"mu": 1, "lambda": 1}}], "warp_speed": 9}',
    '[1, 2]',
]


def harness_fixture():
    """Reference outputs of parse_scene/serialize_scene (incl. the error for each bad document),
    scene_build, export_frame and run_simulation (metrics rows minus wall_ms and the last
    frame) -- harness.py:95-691 -- plus the `color` command's JSON (cli.py:94-118)."""
    import json
    import tempfile
    from click.testing import CliRunner
    from vbdsim import harness as H
    from vbdsim.cli import main as cli_main
    from vbdsim.errors import SchemaError
    out = {}
    for name, text in harness_scenes().items():
        cfg = H.parse_scene(text)
        out[f"{name}_scene"] = np.str_(text)
        out[f"{name}_ser"] = np.str_(H.serialize_scene(cfg))
        system, state, params = H.scene_build(cfg)
        for f in ("rest_positions", "masses", "tets", "springs", "sp_l0", "sp_k", "sp_kd",
                  "color_verts", "color_off"):
            out[f"{name}_{f}"] = np.asarray(getattr(system, f))
        for f in system.cons._fields:
            out[f"{name}_cons_{f}"] = np.asarray(getattr(system.cons, f))
        out[f"{name}_x0"] = state.x.copy()
        out[f"{name}_v0"] = state.v_t.copy()
        out[f"{name}_faces"] = H._surface_faces(system)
        with tempfile.TemporaryDirectory() as d:
            H.run_simulation(cfg, d)
            rows = [ln.split(",") for ln in open(f"{d}/metrics.csv").read().splitlines()[1:]]
            out[f"{name}_metrics"] = np.array([[float(c) for c in r[:-1]] for r in rows])
            files = sorted(p.name for p in Path(d).glob("frame_*"))
            out[f"{name}_frame_files"] = np.array(files)
            pos, fac = H.load_frame(Path(d) / files[-1])
            out[f"{name}_last_x"] = pos
            out[f"{name}_last_faces"] = fac
    errs = []
    for text in HARNESS_BAD:
        try:
            H.parse_scene(text)
            errs.append(("none", ""))
        except SchemaError as e:
            errs.append(("SchemaError", str(e)))
        except ValueError as e:
            errs.append(("ValueError", str(e)))
    out["bad_scenes"] = np.array(HARNESS_BAD)
    out["bad_kind"] = np.array([e[0] for e in errs])
    out["bad_msg"] = np.array([e[1] for e in errs])
    rng = np.random.default_rng(5)
    pos = rng.standard_normal((11, 3))
    fac = rng.integers(0, 11, (7, 3))
    with tempfile.TemporaryDirectory() as d:
        H.export_frame(pos, fac, f"{d}/f.bin")
        H.export_frame(pos, fac, f"{d}/f.obj")
        out["frame_pos"], out["frame_faces"] = pos, fac
        out["frame_bin"] = np.frombuffer(Path(f"{d}/f.bin").read_bytes(), dtype=np.uint8)
        out["frame_obj"] = np.str_(Path(f"{d}/f.obj").read_text())
        m = generate_beam(4, 3, 3, 0.1, density=1000.0)
        Path(f"{d}/m.node").write_text("# nodes\n" + "\n".join(
            f"{i} {float(p[0])!r} {float(p[1])!r} {float(p[2])!r}" for i, p in enumerate(m.rest_positions)))
        Path(f"{d}/m.ele").write_text("\n".join(f"{i} {t[0]} {t[1]} {t[2]} {t[3]} 0"
                                                for i, t in enumerate(m.tets)) + "\n\n")
        out["mesh_node"] = np.str_(Path(f"{d}/m.node").read_text())
        out["mesh_ele"] = np.str_(Path(f"{d}/m.ele").read_text())
        res = CliRunner().invoke(cli_main, ["color", "--nodes", f"{d}/m.node", "--eles", f"{d}/m.ele"])
        assert res.exit_code == 0, res.output
        out["color_json"] = np.str_(json.dumps(json.loads(res.output), sort_keys=True))
    save("harness.npz", **out)


def convergence_fixture():
    """Reference run_convergence (harness.py:702-743: the Newton optimum G* and a G trace per
    solver through baselines.descend, baselines.py:152-189) on the harness scenes, with the
    frozen start (x, y after DCD and the warm start) and each solver's final iterate."""
    from dataclasses import replace
    from vbdsim import baselines as B
    from vbdsim import harness as H
    from vbdsim.solver import _detect_dcd
    out = {}
    iters = 24  # three global line searches for jacobi / gd
    for name, text in harness_scenes().items():
        cfg = H.parse_scene(text)
        res = H.run_convergence(cfg, ["vbd", "vbd-cheb", "jacobi", "gd", "newton"], iters)
        out[f"{name}_g_star"] = np.float64(res["g_star"])
        system, state, params = H.scene_build(cfg)
        state.y = inertia_target(state.x_t, state.v_t, params.a_ext_vec, params.h)
        _detect_dcd(state, params)
        initialize(state, params)
        out[f"{name}_x0"], out[f"{name}_y0"] = state.x.copy(), state.y.copy()
        for m in ("vbd", "vbd-cheb", "jacobi", "gd"):
            tr = res["traces"][m]
            out[f"{name}_{m}_g"] = tr.g
            out[f"{name}_{m}_x"] = tr.x_final
            out[f"{name}_{m}_loss"] = res["relative_loss"][m]
            # the same trace again from the stored start (the trace is deterministic)
            st = H._clone_state(state)
            p = replace(params, rho=0.95) if m == "vbd-cheb" and params.rho == 0.0 else params
            assert np.array_equal(B.descend(st, p, m, iters).g, tr.g), (name, m)
    out["iters"] = np.int64(iters)
    save("convergence.npz", **out)


def config_fixtures():
    """Parity at the BASELINE configs' own settings.

    * c2_full.npz -- C2 at full size: generate_cube(37, 0.5), mu=2e6 lam=1e7 kd=1e-6,
      x0 = default_rng(0).uniform(bbox) (regenerated by the tests from the mesh), h=1/60,
      no gravity.  Per-colour-pass outputs of the first iteration of the first step on
      identical inputs (x = x_t = y = x0; only the colour's own rows are stored) and x after
      the first step at n_max=100, rho=0.95.
    * c4obj_steps.npz -- the first C4 object: generate_cube(15, 0.3) translated to z=1,
      mu=1e6 lam=1e7 kd=1e-7, h=1/120, n_max=60, gravity, seeded rigid velocity
      v = lin + ang x (x - centre); x after steps 1, 5, 10.
    * c5block_steps.npz -- a 32^3 block with C5's material, h, n_max and BCs:
      generate_beam(32,32,32,0.01), x=0 face fixed, mu=2e6 lam=2e7 kd=1e-7, h=1/240,
      n_max=40, gravity; x after steps 1 and 10.
    """
    from vbdsim import build_tet_mesh
    # C2
    m = generate_cube(37, 0.5, density=1000.0)
    s = build_system([Body(m, MaterialParams(2e6, 1e7, 1e-6))])
    lo, hi = m.rest_positions.min(0), m.rest_positions.max(0)
    x0 = np.random.default_rng(0).uniform(lo, hi, size=m.rest_positions.shape)
    st = make_state(s, x0=x0)
    p = SolverParams(h=1.0 / 60.0, n_max=100, rho=0.95, threads=1)
    out = {}
    off = s.color_off
    x = x0.copy()
    for g in range(s.colors.num_colors):
        grp = s.color_verts[off[g]:off[g + 1]]
        st.x = x.copy()
        color_pass(st, grp, p)
        out[f"after_color{g}"] = st.x[grp].copy()
        x = st.x.copy()
    st = make_state(s, x0=x0)
    step(st, p)
    # the reference's own noise floor on these inputs: its NumPy backend (same algorithm,
    # different rounding) against its native backend, per pass and after the first step
    from vbdsim import _backend
    from vbdsim import _numpy_core
    native = _backend._impl
    _backend._impl = _numpy_core
    try:
        fmax, fq = [], []
        x = x0.copy()
        for g in range(s.colors.num_colors):
            grp = s.color_verts[off[g]:off[g + 1]]
            stn = make_state(s, x0=x0)
            stn.x = x.copy()
            color_pass(stn, grp, p)
            d = np.abs(stn.x[grp] - out[f"after_color{g}"])
            fmax.append(d.max())
            fq.append(np.quantile(d, 0.999))
            x[grp] = out[f"after_color{g}"]
        stn = make_state(s, x0=x0)
        step(stn, p)
        diag = np.linalg.norm(st.x.max(0) - st.x.min(0))
        floor_step1 = np.abs(stn.x - st.x).max() / diag
    finally:
        _backend._impl = native
    save("c2_full.npz", x_step1=st.x, floor_pass_max=np.array(fmax),
         floor_pass_p999=np.array(fq), floor_step1=np.float64(floor_step1), **out)
    # one C4 object
    rng = np.random.default_rng(0)
    lin = rng.uniform(-1, 1, (10368, 3))[0]
    ang = 4.0 * rng.uniform(-1, 1, (10368, 3))[0]
    m0 = generate_cube(15, 0.3, density=1000.0)
    m = build_tet_mesh(m0.rest_positions + np.array([0.0, 0.0, 1.0]), m0.tets, 1000.0)
    c = np.array([0.0, 0.0, 1.0]) + 0.5 * (0.3 / 14) * 14
    r = m.rest_positions - c
    v0 = np.stack([lin[0] + (ang[1] * r[:, 2] - ang[2] * r[:, 1]),
                   lin[1] + (ang[2] * r[:, 0] - ang[0] * r[:, 2]),
                   lin[2] + (ang[0] * r[:, 1] - ang[1] * r[:, 0])], 1)
    s = build_system([Body(m, MaterialParams(1e6, 1e7, 1e-7))])
    st = make_state(s, v0=v0)
    p = SolverParams(h=1.0 / 120.0, n_max=60, a_ext=G, threads=1)
    xs = []
    for k in range(10):
        step(st, p)
        if k in (0, 4, 9):
            xs.append(st.x.copy())
    save("c4obj_steps.npz", la=np.concatenate([lin, ang]), v0=v0, x=np.array(xs),
         steps=np.array([1, 5, 10]))
    # C5 material / h / BCs on a 32^3 block
    m, fixed, s = beam_system(32, 32, 32, 0.01, mat=(2e6, 2e7, 1e-7))
    st = make_state(s)
    p = SolverParams(h=1.0 / 240.0, n_max=40, a_ext=G, threads=1)
    xs = []
    for k in range(10):
        step(st, p)
        if k in (0, 9):
            xs.append(st.x.copy())
    save("c5block_steps.npz", x=np.array(xs), steps=np.array([1, 10]), fixed=fixed)


if __name__ == "__main__":
    which = set(sys.argv[1:]) or {"mesh", "coloring", "pass", "steps", "extras", "energy", "contact", "harness",
                                 "convergence", "configs"}
    for name, fn in (("mesh", mesh_fixture), ("coloring", coloring_fixtures), ("pass", pass_fixture),
                     ("steps", step_fixtures), ("extras", extras_fixture), ("energy", energy_fixture),
                     ("contact", contact_fixture), ("harness", harness_fixture),
                     ("convergence", convergence_fixture), ("configs", config_fixtures)):
        if name in which:
            fn()
