"""CPU oracle for the VBD hot path -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker.  It is imported only by ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg; the product package (``paper_2403_06321_b200``)
never imports it and has no CPU fallback.

It restates, in NumPy plus the plain-C kernel ``oracle/vbd_oracle.c``, the
reference's algorithm for the path named in BASELINE.json:

* ``generate_beam`` / ``generate_cube``  <- pkg/src/vbdsim/harness.py:28-76
* ``build_tet_mesh`` (orientation fix, Dm^-1, volumes, lumped masses)
                                          <- pkg/src/vbdsim/mesh.py:128-170
* ``incidence_from_elements``            <- mesh.py:232-267
* ``merged_adjacency``                   <- pkg/src/vbdsim/_system.py:147-169
* ``greedy_color``                       <- mesh.py:270-302 (C: oracle_greedy_color)
* ``build_system`` (flat arrays, slot weights, colour groups)
                                          <- _system.py:139-144, 204-303
* ``color_pass``                         <- pkg/src/vbdsim/_native.pyx:513-589 (C)
* ``inertia_target``/``initialize``/``chebyshev_omega``/``accelerate``/``step``
                                          <- pkg/src/vbdsim/solver.py:120-177, 221-232, 282-324

Parity of this restatement is pinned by tests/test_oracle.py against golden
vectors written by the reference itself (tests/golden/make_golden.py) and,
live, against the reference's compiled kernel (``oracle/_ref``, built from the
reference's own ``_native.c`` by ``oracle/Makefile``).
"""

from __future__ import annotations

import ctypes
import importlib.util
import os
import subprocess
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
FIXED = 1
SUBSPACE = 2

# harness.py:30-33 -- 5-tet split of a hex cell, alternated by cell parity.
_CELL_EVEN = ((0, 3, 5, 6), (1, 0, 3, 5), (2, 0, 3, 6), (4, 0, 5, 6), (7, 3, 5, 6))
_CELL_ODD = ((1, 2, 4, 7), (0, 1, 2, 4), (3, 1, 2, 7), (5, 1, 4, 7), (6, 2, 4, 7))


# --------------------------------------------------------------------------
# native pieces

_lib = None


def lib():
    """ctypes handle on oracle/liboracle.so (built by ``make -C oracle``)."""
    global _lib
    if _lib is not None:
        return _lib
    path = HERE / "liboracle.so"
    if not path.exists():
        subprocess.run(["make", "-C", str(HERE)], check=True, capture_output=True)
    L = ctypes.CDLL(str(path))
    P = ctypes.c_void_p
    i64, f64, c_int = ctypes.c_int64, ctypes.c_double, ctypes.c_int
    L.oracle_color_pass.argtypes = [i64, P, P, P, P, P, P, P, P, P, P, P, P, P, P,
                                    f64, P, i64, c_int, c_int, f64, c_int]
    L.oracle_color_pass.restype = c_int
    L.oracle_color_pass_ex.argtypes = ([i64, P, P, P, P, P, P, P, P, P, P, P, P, P, P,
                                        f64, P, i64, c_int, c_int, f64, c_int] + [P] * 21
                                       + [f64, f64])
    L.oracle_color_pass_ex.restype = c_int
    L.oracle_local_energy.argtypes = [P, P, P, P, P, P, P, P, P, P, f64, i64, P]
    L.oracle_local_energy.restype = f64
    L.oracle_greedy_color.argtypes = [i64, P, P, P, P]
    L.oracle_greedy_color.restype = i64
    L.oracle_beam_tets.argtypes = [i64, i64, i64, P]
    L.oracle_beam_tets.restype = None
    _lib = L
    return L


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def ref_native():
    """The reference's own compiled colour-pass kernel (oracle/_ref), or None.

    Built by ``make -C oracle ref`` from /root/reference/pkg/src/vbdsim/_native.c
    (the reference's committed Cython output) with the reference's flags.  It is
    loaded standalone: only its ``color_pass``/``max_threads`` are used, always
    with an explicit contact-array object so it never imports reference Python.
    """
    ref = HERE / "_ref"
    hits = sorted(ref.glob("_native*.so")) if ref.exists() else []
    if not hits:
        return None
    spec = importlib.util.spec_from_file_location("_native", str(hits[0]))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


# --------------------------------------------------------------------------
# mesh construction (mesh.py / harness.py restated)

@dataclass
class Mesh:
    rest_positions: np.ndarray
    tets: np.ndarray
    rest_volumes: np.ndarray
    inv_rest_shape: np.ndarray
    masses: np.ndarray

    @property
    def num_vertices(self):
        return len(self.rest_positions)

    def bbox_diagonal(self):
        return float(np.linalg.norm(self.rest_positions.max(0) - self.rest_positions.min(0)))


def beam_tets(nx, ny, nz):
    """Raw connectivity of generate_beam (harness.py:54-66), via the C oracle."""
    t = np.empty(((nx - 1) * (ny - 1) * (nz - 1) * 5, 4), dtype=np.int64)
    lib().oracle_beam_tets(nx, ny, nz, _p(t))
    return t


def beam_tets_py(nx, ny, nz):
    """Pure-Python loop restatement of harness.py:54-66 (small sizes only)."""
    def vid(ax, ay, az):
        return (ax * ny + ay) * nz + az
    out = []
    for cx in range(nx - 1):
        for cy in range(ny - 1):
            for cz in range(nz - 1):
                corners = [vid(cx + dx, cy + dy, cz + dz)
                           for dx in (0, 1) for dy in (0, 1) for dz in (0, 1)]
                pat = _CELL_EVEN if (cx + cy + cz) % 2 == 0 else _CELL_ODD
                out.extend([corners[k] for k in t] for t in pat)
    return np.asarray(out, dtype=np.int64)


def build_tet_mesh(pos, tets, density):
    """mesh.py:128-170 restated (same NumPy kernels => same rounding)."""
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    tets = np.ascontiguousarray(tets, dtype=np.int64)
    d = pos[tets[:, 1:]] - pos[tets[:, :1]]
    vol = np.linalg.det(np.swapaxes(d, 1, 2)) / 6.0
    flip = vol < 0.0
    if np.any(flip):
        tets = tets.copy()
        tets[flip] = tets[flip][:, [0, 2, 1, 3]]
        vol = np.abs(vol)
    d_m = np.swapaxes(pos[tets[:, 1:]] - pos[tets[:, :1]], 1, 2)
    inv = np.linalg.inv(d_m)
    masses = np.zeros(len(pos))
    np.add.at(masses, tets.ravel(), np.repeat(density * vol / 4.0, 4))
    return Mesh(pos, tets, vol, inv, masses)


def generate_beam(nx, ny, nz, spacing, density=1000.0):
    """harness.py:42-67."""
    ix, iy, iz = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    pos = spacing * np.stack([ix, iy, iz], axis=-1).reshape(-1, 3).astype(np.float64)
    return build_tet_mesh(pos, beam_tets(nx, ny, nz), density)


def generate_cube(n, edge, density=1000.0):
    """harness.py:70-76."""
    return generate_beam(n, n, n, edge / (n - 1), density)


def incidence_from_elements(elements, n):
    """mesh.py:232-267: vertex->element CSR (ascending element id) + neighbours."""
    elements = np.asarray(elements, dtype=np.int64)
    num, arity = elements.shape
    verts = elements.ravel()
    eids = np.repeat(np.arange(num, dtype=np.int64), arity)
    slots = np.tile(np.arange(arity, dtype=np.int64), num)
    order = np.lexsort((eids, verts))
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(verts, minlength=n), out=off[1:])
    return off, np.ascontiguousarray(eids[order]), np.ascontiguousarray(slots[order])


def merged_adjacency(n, element_arrays):
    """_system.py:147-169: distinct-neighbour CSR over all element vertex pairs."""
    pairs = []
    for el in element_arrays:
        if len(el) == 0:
            continue
        pa, pb = np.triu_indices(el.shape[1], k=1)
        u, v = el[:, pa].ravel(), el[:, pb].ravel()
        pairs.append(np.stack([np.concatenate([u, v]), np.concatenate([v, u])], axis=1))
    uniq = np.unique(np.concatenate(pairs), axis=0) if pairs else np.zeros((0, 2), np.int64)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(uniq[:, 0], minlength=n), out=off[1:])
    return off, np.ascontiguousarray(uniq[:, 1])


def greedy_color(noff, nids, order=None):
    """mesh.py:270-302 via the C restatement; returns (color_of, groups)."""
    n = len(noff) - 1
    col = np.empty(n, dtype=np.int64)
    o = None if order is None else np.ascontiguousarray(order, dtype=np.int64)
    nc = lib().oracle_greedy_color(n, _p(np.ascontiguousarray(noff, dtype=np.int64)),
                                   _p(np.ascontiguousarray(nids, dtype=np.int64)), _p(o), _p(col))
    return col, tuple(np.flatnonzero(col == c) for c in range(nc))


def greedy_color_py(noff, nids):
    """Literal pure-Python restatement of mesh.py:276-295 (small graphs)."""
    n = len(noff) - 1
    deg = np.diff(noff)
    order = np.lexsort((np.arange(n), -deg))
    col = np.full(n, -1, dtype=np.int64)
    for i in order:
        used = col[nids[noff[i]:noff[i + 1]]]
        used = used[used >= 0]
        c = 0
        if used.size:
            taken = np.zeros(used.max() + 2, dtype=bool)
            taken[used] = True
            c = int(np.argmin(taken))
        col[i] = c
    nc = int(col.max()) + 1 if n else 0
    return col, tuple(np.flatnonzero(col == c) for c in range(nc))


# --------------------------------------------------------------------------
# flat system (_system.py:204-303, tet bodies only)

@dataclass
class System:
    num_vertices: int
    masses: np.ndarray
    rest_positions: np.ndarray
    tets: np.ndarray
    tet_w: np.ndarray
    tet_vol: np.ndarray
    tet_mu: np.ndarray
    tet_lam: np.ndarray
    tet_kd: np.ndarray
    t_off: np.ndarray
    t_id: np.ndarray
    t_slot: np.ndarray
    color_of: np.ndarray
    color_off: np.ndarray
    color_verts: np.ndarray
    kind: np.ndarray
    body_slices: tuple = ()
    # springs (_system.py:117-123) and constraints (_system.py:76-83); empty by default
    springs: np.ndarray = None
    sp_l0: np.ndarray = None
    sp_k: np.ndarray = None
    sp_kd: np.ndarray = None
    s_off: np.ndarray = None
    s_id: np.ndarray = None
    s_slot: np.ndarray = None
    sub_dim: np.ndarray = None
    sub_basis: np.ndarray = None
    sub_anchor: np.ndarray = None
    box_k: np.ndarray = None
    box_lo: np.ndarray = None
    box_hi: np.ndarray = None

    def __post_init__(self):
        n = self.num_vertices
        if self.springs is None:
            self.springs = np.zeros((0, 2), dtype=np.int64)
            self.sp_l0 = self.sp_k = self.sp_kd = np.zeros(0)
            self.s_off = np.zeros(n + 1, dtype=np.int64)
            self.s_id = np.zeros(0, dtype=np.int64)
            self.s_slot = np.zeros(0, dtype=np.int64)
        if self.sub_dim is None:
            self.sub_dim = np.zeros(n, dtype=np.int64)
            self.sub_basis = np.zeros((n, 3, 2))
            self.sub_anchor = np.zeros((n, 3))
        if self.box_k is None:
            self.box_k = np.zeros(n)
            self.box_lo = np.zeros((n, 3))
            self.box_hi = np.zeros((n, 3))

    @property
    def has_extras(self):
        return bool(len(self.springs) or (self.kind == SUBSPACE).any() or (self.box_k > 0).any())

    @property
    def num_colors(self):
        return len(self.color_off) - 1

    def groups(self):
        return [self.color_verts[self.color_off[g]:self.color_off[g + 1]]
                for g in range(self.num_colors)]


def slot_weight_rows(inv):
    """_system.py:139-144."""
    w = np.empty((len(inv), 4, 3))
    w[:, 1:, :] = inv
    w[:, 0, :] = -inv.sum(axis=1)
    return w


def build_system_ex(tet_bodies, spring_bodies=(), fixed=(), subspace=(), boxes=()):
    """_system.py:204-303 with spring nets and constraints (compile_constraints,
    _system.py:172-201).  tet_bodies: (Mesh, (mu, lam, kd)); spring_bodies:
    (particles (P,3), masses (P,), indices (S,2), rest_length (S,), stiffness (S,), kd);
    fixed: vertex ids; subspace: (vertex, basis (3,L), anchor (3,)); boxes:
    (vertex, lo (3,), hi (3,), k_b).  Vertices are numbered tet bodies first, then
    spring bodies, in the given order (as Body order in the reference)."""
    base = build_system(tet_bodies, fixed=()) if tet_bodies else None
    n_t = base.num_vertices if base else 0
    pos = [base.rest_positions] if base else []
    mass = [base.masses] if base else []
    sp, l0, k, kd = [], [], [], []
    off = n_t
    for parts, masses, idx, rest, stiff, damp in spring_bodies:
        pos.append(np.asarray(parts, dtype=np.float64))
        mass.append(np.asarray(masses, dtype=np.float64))
        sp.append(np.asarray(idx, dtype=np.int64) + off)
        l0.append(np.asarray(rest, dtype=np.float64))
        k.append(np.asarray(stiff, dtype=np.float64))
        kd.append(np.full(len(idx), float(damp)))
        off += len(parts)
    N = off
    cat = lambda parts, shape, dt=np.float64: (np.ascontiguousarray(np.concatenate(parts).astype(dt))
                                               if parts else np.zeros(shape, dtype=dt))
    springs = cat(sp, (0, 2), np.int64)
    tets = base.tets if base else np.zeros((0, 4), dtype=np.int64)
    t_off, t_id, t_slot = incidence_from_elements(tets, N)
    s_off, s_id, s_slot = incidence_from_elements(springs, N)
    noff, nids = merged_adjacency(N, [tets, springs])
    col, groups = greedy_color(noff, nids)
    color_off = np.zeros(len(groups) + 1, dtype=np.int64)
    np.cumsum([len(g) for g in groups], out=color_off[1:])
    kind = np.zeros(N, dtype=np.uint8)
    sub_dim = np.zeros(N, dtype=np.int64)
    sub_basis = np.zeros((N, 3, 2))
    sub_anchor = np.zeros((N, 3))
    box_k, box_lo, box_hi = np.zeros(N), np.zeros((N, 3)), np.zeros((N, 3))
    for v in fixed:
        kind[int(v)] = FIXED
    for v, basis, anchor in subspace:
        b = np.asarray(basis, dtype=np.float64).reshape(3, -1)
        if kind[v] == FIXED:
            continue
        kind[v] = SUBSPACE
        sub_dim[v] = b.shape[1]
        sub_basis[v, :, :b.shape[1]] = b
        sub_anchor[v] = anchor
    for v, lo, hi, kb in boxes:
        box_k[v], box_lo[v], box_hi[v] = kb, lo, hi
    z = lambda shape: np.zeros(shape)
    return System(N, cat(mass, (0,)), cat(pos, (0, 3)), tets,
                  base.tet_w if base else z((0, 4, 3)), base.tet_vol if base else z(0),
                  base.tet_mu if base else z(0), base.tet_lam if base else z(0),
                  base.tet_kd if base else z(0), t_off, t_id, t_slot, col, color_off,
                  np.ascontiguousarray(np.concatenate(groups)) if groups else np.zeros(0, np.int64),
                  kind, base.body_slices if base else (), springs, cat(l0, (0,)), cat(k, (0,)),
                  cat(kd, (0,)), s_off, s_id, s_slot, sub_dim, sub_basis, sub_anchor,
                  box_k, box_lo, box_hi)


def build_system(bodies, fixed=()):
    """bodies: list of (Mesh, (mu, lam, kd)); fixed: vertex ids (FixedConstraint)."""
    off = 0
    pos, mass, tets, tw, tv, mu, lam, kd, slices = [], [], [], [], [], [], [], [], []
    for mesh, (m_mu, m_lam, m_kd) in bodies:
        n = mesh.num_vertices
        slices.append(slice(off, off + n))
        pos.append(mesh.rest_positions)
        mass.append(mesh.masses)
        tets.append(mesh.tets + off)
        tw.append(slot_weight_rows(mesh.inv_rest_shape))
        tv.append(mesh.rest_volumes)
        t = len(mesh.tets)
        mu.append(np.full(t, m_mu))
        lam.append(np.full(t, m_lam))
        kd.append(np.full(t, m_kd))
        off += n
    N = off
    cat = lambda parts: np.ascontiguousarray(np.concatenate(parts))
    tets_a = cat(tets)
    t_off, t_id, t_slot = incidence_from_elements(tets_a, N)
    noff, nids = merged_adjacency(N, [tets_a])
    col, groups = greedy_color(noff, nids)
    color_off = np.zeros(len(groups) + 1, dtype=np.int64)
    np.cumsum([len(g) for g in groups], out=color_off[1:])
    kind = np.zeros(N, dtype=np.uint8)
    kind[np.asarray(list(fixed), dtype=np.int64)] = FIXED
    return System(N, cat(mass), cat(pos), tets_a, cat(tw), cat(tv), cat(mu), cat(lam), cat(kd),
                  t_off, t_id, t_slot, col, color_off, cat(groups), kind, tuple(slices))


# --------------------------------------------------------------------------
# colour pass + time step

def color_pass(system, x, x_t, y, h, group, mode=0, line_search=False, eps_det=1e-10,
               n_threads=0, carr=None, mu_c=0.0, eps_v=1e-2):
    """_native.pyx:513-589, in place on x (C, fp64).  ``carr``: a ContactArrays look-alike
    (count, idx, gamma, refresh, normal, tangent, k_c, cv_off, cv_cid, cv_slot)."""
    if x.dtype != np.float64 or not x.flags["C_CONTIGUOUS"]:
        raise TypeError("x must be C-contiguous float64")
    g = np.ascontiguousarray(group, dtype=np.int64)
    s = system
    has_c = carr is not None and carr.count > 0
    if s.has_extras or has_c:
        c = carr if has_c else None
        dts = (np.int64, np.float64, np.uint8, np.float64, np.float64, np.float64, np.int64, np.int64,
               np.int64)
        keep = [np.ascontiguousarray(getattr(c, k), dtype=dt) for k, dt in zip(
            ("idx", "gamma", "refresh", "normal", "tangent", "k_c", "cv_off", "cv_cid", "cv_slot"),
            dts)] if c else []
        rc = lib().oracle_color_pass_ex(
            s.num_vertices, _p(x), _p(np.ascontiguousarray(x_t)), _p(np.ascontiguousarray(y)),
            _p(s.masses), _p(s.tets), _p(s.tet_w), _p(s.tet_vol), _p(s.tet_mu), _p(s.tet_lam),
            _p(s.tet_kd), _p(s.t_off), _p(s.t_id), _p(s.t_slot), _p(s.kind), float(h), _p(g),
            len(g), int(mode), int(bool(line_search)), float(eps_det), int(n_threads),
            _p(s.springs), _p(s.sp_l0), _p(s.sp_k), _p(s.sp_kd), _p(s.s_off), _p(s.s_id),
            _p(s.s_slot), _p(s.sub_dim), _p(s.sub_basis), _p(s.box_k), _p(s.box_lo), _p(s.box_hi),
            *([_p(a) for a in keep] if c else [None] * 9), float(mu_c), float(eps_v))
        del keep
        if rc != 0:
            raise MemoryError("oracle colour pass failed")
        return
    rc = lib().oracle_color_pass(
        s.num_vertices, _p(x), _p(np.ascontiguousarray(x_t)), _p(np.ascontiguousarray(y)),
        _p(s.masses), _p(s.tets), _p(s.tet_w), _p(s.tet_vol), _p(s.tet_mu), _p(s.tet_lam),
        _p(s.tet_kd), _p(s.t_off), _p(s.t_id), _p(s.t_slot), _p(s.kind), float(h), _p(g),
        len(g), int(mode), int(bool(line_search)), float(eps_det), int(n_threads))
    if rc != 0:
        raise MemoryError("oracle colour pass failed")


_lib32 = None


def color_pass_fp32(system, x, x_t, y, h, group, eps_det=1e-10):
    """The same colour pass with every real in binary32 (liboracle_f32.so, tets only): the
    reference ALGORITHM in fp32 arithmetic.  Used only as the fp32 sensitivity yardstick on
    ill-conditioned inputs; returns the group's new rows (float64 copy of the fp32 result)."""
    global _lib32
    if _lib32 is None:
        path = HERE / "liboracle_f32.so"
        if not path.exists():
            subprocess.run(["make", "-C", str(HERE), "liboracle_f32.so"], check=True, capture_output=True)
        L = ctypes.CDLL(str(path))
        P = ctypes.c_void_p
        L.oracle_color_pass.argtypes = [ctypes.c_int64, P, P, P, P, P, P, P, P, P, P, P, P, P, P,
                                        ctypes.c_float, P, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_float, ctypes.c_int]
        L.oracle_color_pass.restype = ctypes.c_int
        _lib32 = L
    s = system
    if s.has_extras:
        raise NotImplementedError("color_pass_fp32: tets only")
    f = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    keep = [f(x), f(x_t), f(y), f(s.masses), f(s.tet_w), f(s.tet_vol), f(s.tet_mu), f(s.tet_lam),
            f(s.tet_kd)]
    x32, xt32, y32, m32, w32, v32, mu32, la32, kd32 = keep
    g = np.ascontiguousarray(group, dtype=np.int64)
    rc = _lib32.oracle_color_pass(s.num_vertices, _p(x32), _p(xt32), _p(y32), _p(m32), _p(s.tets), _p(w32),
                                  _p(v32), _p(mu32), _p(la32), _p(kd32), _p(s.t_off), _p(s.t_id),
                                  _p(s.t_slot), _p(s.kind), float(h), _p(g), len(g), 0, 0, float(eps_det), 0)
    if rc != 0:
        raise MemoryError("oracle fp32 colour pass failed")
    return x32[g].astype(np.float64)


def step_fp32(system, st, h, n_max, rho=0.0, a_ext=(0.0, 0.0, 0.0), eps_det=1e-10):
    """step() with every real in binary32: float32 state and K2 / blend / velocity arithmetic,
    colour passes through color_pass_fp32 (tets only, adaptive init, no contact).  The fp32
    sensitivity yardstick for chaotic scenes (C2 extreme init), never a parity reference."""
    f = np.float32
    a = np.asarray(a_ext, dtype=f)
    h32 = f(h)
    xt, vt, vp = (np.asarray(v, dtype=f) for v in (st.x_t, st.v_t, st.v_prev))
    y = xt + h32 * vt + (h32 * h32) * a
    norm = f(np.linalg.norm(a))
    if norm == 0:
        x = xt + h32 * vt
    else:
        at = (vt - vp) / h32
        comp = at @ (a / norm)
        x = xt + h32 * vt + ((h32 * h32) * np.clip(comp / norm, 0, 1).astype(f))[:, None] * a
    x[system.kind == 1] = xt[system.kind == 1]
    x = np.ascontiguousarray(x, dtype=f)
    prev1, pp = x.copy(), None
    for n in range(1, n_max + 1):
        for g in system.groups():
            x[g] = color_pass_fp32(system, x, xt, y, h, g, eps_det).astype(f)
        omega = chebyshev_omega(rho, n)
        if omega != 1.0 and pp is not None:
            x[...] = f(omega) * (x - pp) + pp
        pp = prev1
        prev1 = x.copy()
    v = (x - xt) / h32
    st.v_prev, st.v_t, st.x_t, st.x = st.v_t, v.astype(np.float64), x.astype(np.float64), x.astype(np.float64)
    st.step_index += 1
    return st


def local_energy(system, x, y, h, i, p):
    s = system
    p = np.ascontiguousarray(p, dtype=np.float64)
    return lib().oracle_local_energy(_p(x), _p(y), _p(s.masses), _p(s.tets), _p(s.tet_w),
                                     _p(s.tet_vol), _p(s.tet_mu), _p(s.tet_lam), _p(s.t_off),
                                     _p(s.t_id), float(h), int(i), _p(p))


class _EmptyContacts:
    """Zero-contact ContactArrays look-alike (_system.py:86-96) for oracle/_ref."""

    def __init__(self, n):
        z = np.zeros(0, dtype=np.int64)
        self.count = 0
        self.idx = np.zeros((0, 4), dtype=np.int64)
        self.gamma = np.zeros((0, 4))
        self.refresh = np.zeros(0, dtype=np.uint8)
        self.normal = np.zeros((0, 3))
        self.tangent = np.zeros((0, 3, 2))
        self.k_c = np.zeros(0)
        self.cv_off = np.zeros(n + 1, dtype=np.int64)
        self.cv_cid = z
        self.cv_slot = z.copy()


class RefSystemView:
    """Duck-typed reference ``System`` (_system.py:99-133) over oracle arrays, so
    the reference's own compiled kernel can be driven on identical inputs."""

    def __init__(self, s: System):
        n = s.num_vertices
        z = np.zeros(0, dtype=np.int64)
        self.num_vertices = n
        self.masses, self.tets, self.tet_w = s.masses, s.tets, s.tet_w
        self.tet_vol, self.tet_mu, self.tet_lam, self.tet_kd = s.tet_vol, s.tet_mu, s.tet_lam, s.tet_kd
        self.t_off, self.t_id, self.t_slot = s.t_off, s.t_id, s.t_slot
        self.color_off, self.color_verts = s.color_off, s.color_verts
        self.rest_positions = s.rest_positions
        self.springs, self.sp_l0, self.sp_k, self.sp_kd = s.springs, s.sp_l0, s.sp_k, s.sp_kd
        self.s_off, self.s_id, self.s_slot = s.s_off, s.s_id, s.s_slot
        del z

        class _Cons:
            pass
        c = _Cons()
        c.kind = s.kind
        c.sub_dim, c.sub_basis, c.sub_anchor = s.sub_dim, s.sub_basis, s.sub_anchor
        c.box_k, c.box_lo, c.box_hi = s.box_k, s.box_lo, s.box_hi
        self.cons = c
        self.carr = _EmptyContacts(n)


def inertia_target(x_t, v_t, a_ext, h):
    """solver.py:120-122."""
    return np.asarray(x_t) + h * np.asarray(v_t) + h * h * np.asarray(a_ext)


def chebyshev_omega(rho, n):
    """solver.py:167-177."""
    if n < 1:
        raise ValueError("iteration index must be >= 1")
    if rho == 0.0 or n == 1:
        return 1.0
    omega = 2.0 / (2.0 - rho * rho)
    for _ in range(3, n + 1):
        omega = 4.0 / (4.0 - rho * rho * omega)
    return omega


@dataclass
class State:
    x_t: np.ndarray
    v_t: np.ndarray
    v_prev: np.ndarray
    x: np.ndarray
    y: np.ndarray
    step_index: int = 0
    x_prev1: np.ndarray = None
    x_pp: np.ndarray = None


def make_state(system, x0=None, v0=None):
    """solver.py:111-117."""
    x = np.array(system.rest_positions if x0 is None else x0, dtype=np.float64)
    v = np.zeros_like(x) if v0 is None else np.array(v0, dtype=np.float64)
    return State(x.copy(), v.copy(), v.copy(), x.copy(), x.copy())


def initialize(system, st, h, a_ext, init_mode="adaptive"):
    """solver.py:125-164."""
    a = np.asarray(a_ext, dtype=np.float64)
    st.y = inertia_target(st.x_t, st.v_t, a, h)
    if init_mode == "prev_pos":
        x = st.x_t.copy()
    elif init_mode == "inertia":
        x = st.x_t + h * st.v_t
    elif init_mode == "inertia_accel":
        x = st.y.copy()
    else:
        norm = float(np.linalg.norm(a))
        if norm == 0.0:
            x = st.x_t + h * st.v_t
        else:
            a_t = (st.v_t - st.v_prev) / h
            comp = a_t @ (a / norm)
            a_tilde = np.clip(comp / norm, 0.0, 1.0)
            x = st.x_t + h * st.v_t + (h * h) * a_tilde[:, None] * a
    fixed = system.kind == FIXED
    x[fixed] = st.x_t[fixed]
    for i in np.flatnonzero(system.kind == SUBSPACE):  # solver.py:158-162
        dim = system.sub_dim[i]
        b = system.sub_basis[i][:, :dim]
        anchor = system.sub_anchor[i]
        x[i] = anchor + b @ (b.T @ (x[i] - anchor))
    st.x = np.ascontiguousarray(x)
    return st.x


class NonFinite(Exception):
    def __init__(self, step, iteration, vertex):
        super().__init__(f"non-finite at step {step} iteration {iteration} vertex {vertex}")
        self.step, self.iteration, self.vertex = step, iteration, vertex


def step(system, st, h, n_max, rho=0.0, a_ext=(0.0, 0.0, 0.0), eps_det=1e-10,
         init_mode="adaptive", kernel=None, n_threads=0, on_iteration=None, line_search=False):
    """solver.py:291-324 without contact.  ``kernel`` selects the colour-pass
    implementation: None -> the C restatement, or the reference's compiled
    module (``ref_native()``)."""
    a = np.asarray(a_ext, dtype=np.float64)
    st.y = inertia_target(st.x_t, st.v_t, a, h)
    initialize(system, st, h, a, init_mode)
    st.x_prev1 = st.x.copy()
    st.x_pp = None
    groups = system.groups()
    view = RefSystemView(system) if kernel is not None else None
    for n in range(1, n_max + 1):
        for g in groups:
            if kernel is None:
                color_pass(system, st.x, st.x_t, st.y, h, g, 0, line_search, eps_det, n_threads)
            else:
                kernel.color_pass(view, view.carr, st.x, st.x_t, st.y, h, g, 0,
                                  line_search=line_search, eps_det=eps_det, mu_c=0.0, eps_v=1e-2,
                                  n_threads=n_threads)
        omega = chebyshev_omega(rho, n)
        if omega != 1.0 and st.x_pp is not None:
            st.x[...] = omega * (st.x - st.x_pp) + st.x_pp
        st.x_pp = st.x_prev1
        st.x_prev1 = st.x.copy()
        if not np.isfinite(st.x).all():
            bad = np.flatnonzero(~np.isfinite(st.x).all(axis=1))
            raise NonFinite(st.step_index, n, int(bad[0]))
        if on_iteration is not None:
            on_iteration(st, n)
    v = (st.x - st.x_t) / h
    st.v_prev = st.v_t
    st.v_t = v
    st.x_t = st.x.copy()
    st.step_index += 1
    return st


# --------------------------------------------------------------------------
# incremental potential G (metrics path, _assembly.py:29-82 restated, no contacts)

def variational_energy(system, x, y, h):
    """G(x) = 1/(2 h^2) |x - y|_M^2 + E(x) with E = tets + springs + box
    (_assembly.py:29-38, 41-46, 59-67, 70-82), the same NumPy operations."""
    s = system
    x = np.asarray(x)
    dx = x - np.asarray(y)
    inertia = 0.5 / (h * h) * float((s.masses[:, None] * dx * dx).sum())
    e = 0.0
    if len(s.tets):
        f = np.einsum("tsa,tsb->tab", x[s.tets], s.tet_w)
        i_c = np.einsum("tab,tab->t", f, f)
        j = np.linalg.det(f)
        gamma = 1.0 + s.tet_mu / s.tet_lam
        psi = 0.5 * s.tet_mu * (i_c - 3.0) + 0.5 * s.tet_lam * (j - gamma) ** 2
        e += float((s.tet_vol * psi).sum())
    if len(s.springs):
        d = x[s.springs[:, 0]] - x[s.springs[:, 1]]
        length = np.linalg.norm(d, axis=1)
        e += float((0.5 * s.sp_k * (length - s.sp_l0) ** 2).sum())
    k = s.box_k
    active = k > 0.0
    if active.any():
        xa = x[active]
        below = np.maximum(s.box_lo[active] - xa, 0.0)
        above = np.maximum(xa - s.box_hi[active], 0.0)
        e += float(0.5 * (k[active][:, None] * (below ** 2 + above ** 2)).sum())
    return inertia + e
