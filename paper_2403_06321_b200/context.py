"""DeviceContext: one packed scene resident on one B200 (wraps ``vbd_ctx*``).

Built either from reference-layout System arrays (duck-typed: a System of this
package *or* of the reference package works) or from procedural beams generated
on the device (BASELINE configs C4/C5, tens of millions of vertices).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import NonFiniteState

FIXED, SUBSPACE = 1, 2


@dataclass(frozen=True)
class Beam:
    """generate_beam(nx, ny, nz, spacing, density) translated by origin, with a material."""

    nx: int
    ny: int
    nz: int
    spacing: float
    mu: float
    lam: float
    kd: float = 0.0
    density: float = 1000.0
    origin: tuple = (0.0, 0.0, 0.0)
    fix_min_x: bool = False
    fix_max_x: bool = False
    jitter: float = 0.0  # rest-position jitter, fraction of spacing (irregular mesh; 0 = grid)

    def desc(self):
        d = _lib.BeamDesc()
        d.nx, d.ny, d.nz = self.nx, self.ny, self.nz
        d.spacing, d.density = self.spacing, self.density
        d.origin = (ctypes.c_double * 3)(*map(float, self.origin))
        d.mu, d.lam, d.kd = self.mu, self.lam, self.kd
        d.fix_min_x = 1 if self.fix_min_x else 0
        d.fix_max_x = 1 if self.fix_max_x else 0
        d.jitter = float(self.jitter)
        return d

    @property
    def num_vertices(self):
        return self.nx * self.ny * self.nz

    @property
    def num_tets(self):
        return 5 * (self.nx - 1) * (self.ny - 1) * (self.nz - 1)


def _extra_terms(system, n):
    """Spring and constraint arrays of a System (reference or mirrored) for the C ABI:
    springs (_system.py:117-123), subspace and world-box constraints (_system.py:76-83)."""
    out = {}
    springs = getattr(system, "springs", None)
    if springs is not None and len(springs):
        out.update(springs=_lib.i64c(springs).reshape(-1, 2), sp_l0=_lib.f64c(system.sp_l0),
                   sp_k=_lib.f64c(system.sp_k), sp_kd=_lib.f64c(system.sp_kd))
    cons = system.cons
    if np.any(np.asarray(cons.kind) == SUBSPACE):
        out.update(sub_dim=_lib.i64c(cons.sub_dim), sub_basis=_lib.f64c(cons.sub_basis, (n, 3, 2)),
                   sub_anchor=_lib.f64c(cons.sub_anchor, (n, 3)))
    if np.any(np.asarray(cons.box_k) > 0.0):
        out.update(box_k=_lib.f64c(cons.box_k), box_lo=_lib.f64c(cons.box_lo, (n, 3)),
                   box_hi=_lib.f64c(cons.box_hi, (n, 3)))
    return out


class DeviceContext:
    def __init__(self, handle, keepalive=None):
        self._h = ctypes.c_void_p(handle)
        self._keep = keepalive
        self.info = self._info()
        self.n = self.info.num_vertices

    # -- construction -----------------------------------------------------------------
    @classmethod
    def from_system(cls, system, precision="fp64", device=0):
        n = int(system.num_vertices)
        arrs = dict(
            tets=_lib.i64c(system.tets).reshape(-1, 4),
            tet_w=_lib.f64c(system.tet_w).reshape(-1, 4, 3),
            tet_vol=_lib.f64c(system.tet_vol), tet_mu=_lib.f64c(system.tet_mu),
            tet_lam=_lib.f64c(system.tet_lam), tet_kd=_lib.f64c(system.tet_kd),
            masses=_lib.f64c(system.masses),
            kind=np.ascontiguousarray(system.cons.kind, dtype=np.uint8),
            t_off=_lib.i64c(system.t_off), t_id=_lib.i64c(system.t_id),
            t_slot=_lib.i64c(system.t_slot), color_off=_lib.i64c(system.color_off),
            color_verts=_lib.i64c(system.color_verts))
        rp = getattr(system, "rest_positions", None)
        if rp is not None:
            arrs["rest_positions"] = _lib.f64c(rp, (n, 3))
        arrs.update(_extra_terms(system, n))
        d = _lib.SystemDesc()
        d.num_vertices = n
        d.num_tets = len(arrs["tets"])
        for k, v in arrs.items():
            setattr(d, k, _lib.ptr(v))
        d.num_colors = len(arrs["color_off"]) - 1
        d.num_springs = len(arrs["springs"]) if "springs" in arrs else 0
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().vbd_ctx_create(ctypes.byref(d), device, _lib.PREC[precision],
                                             ctypes.byref(h)))
        return cls(h.value)

    @classmethod
    def from_beams(cls, beams, precision="fp32", device=0, slab=None):
        arr = (_lib.BeamDesc * len(beams))(*[b.desc() for b in beams])
        lo, hi = (0, 0) if slab is None else slab
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().vbd_ctx_create_beams(arr, len(beams), lo, hi, device,
                                                   _lib.PREC[precision], ctypes.byref(h)))
        return cls(h.value, keepalive=list(beams))

    def set_contacts(self, carr=None, mu_c=0.0, eps_v=1e-2):
        """Contact set for subsequent colour passes (a ContactArrays, _system.py:86-96)."""
        L = _lib.lib()
        if carr is None or not getattr(carr, "count", 0):
            _lib.check(L.vbd_set_contacts(self._h, 0, *([None] * 9), 0.0, 1e-2))
            self._contacts = None
            return
        keep = dict(idx=_lib.i64c(carr.idx), gamma=_lib.f64c(carr.gamma),
                    refresh=np.ascontiguousarray(carr.refresh, dtype=np.uint8),
                    normal=_lib.f64c(carr.normal), tangent=_lib.f64c(carr.tangent),
                    k_c=_lib.f64c(carr.k_c), cv_off=_lib.i64c(carr.cv_off),
                    cv_cid=_lib.i64c(carr.cv_cid), cv_slot=_lib.i64c(carr.cv_slot))
        _lib.check(L.vbd_set_contacts(self._h, int(carr.count), *[_lib.ptr(keep[k]) for k in (
            "idx", "gamma", "refresh", "normal", "tangent", "k_c", "cv_off", "cv_cid", "cv_slot")],
            float(mu_c), float(eps_v)))
        self._contacts = carr

    def set_collision(self, system=None, contact=None, n_col=4):
        """Device contact detection for step(): the collision surface of ``system`` (its
        collision mesh, mapped to global ids) and ContactParams ``contact``; None disables."""
        L = _lib.lib()
        mesh = getattr(system, "collision_mesh", None) if system is not None else None
        if contact is None or mesh is None or len(mesh.surface_tris) == 0:
            _lib.check(L.vbd_set_collision(self._h, 0, None, 0, None, 1.0, 1.0, 0.0, 1e-2, 0.0, 0, 0.0, 1))
            return
        cmap = np.asarray(system.collision_map, dtype=np.int64)
        tris = _lib.i64c(cmap[mesh.surface_tris])
        edges = _lib.i64c(cmap[mesh.surface_edges]).reshape(-1, 2)
        if len(mesh.surface_edges):  # contact.py:205-215: 1.5 x the median rest surface edge
            e = mesh.rest_positions[mesh.surface_edges]
            cell = 1.5 * float(np.median(np.linalg.norm(e[:, 1] - e[:, 0], axis=1)))
        else:
            cell = float(mesh.bbox_diagonal()) or 1.0
        md = contact.max_depth
        _lib.check(L.vbd_set_collision(self._h, len(tris), _lib.ptr(tris), len(edges), _lib.ptr(edges),
                                       cell, float(contact.k_c), float(contact.mu_c), float(contact.eps_v),
                                       float(contact.dcd_radius), 0 if md is None else 1,
                                       0.0 if md is None else float(md), int(n_col)))

    def detect_contacts(self, which, cap=100000):
        """One detection pass (0: DCD at x_t, 1: CCD x_t -> x): (idx, gamma, normal, is_ccd)."""
        n = ctypes.c_int64()
        idx = np.zeros((cap, 4), np.int64)
        gam = np.zeros((cap, 4))
        nrm = np.zeros((cap, 3))
        ccd = np.zeros(cap, np.int32)
        _lib.check(_lib.lib().vbd_detect_contacts(self._h, int(which), cap, ctypes.byref(n), _lib.ptr(idx),
                                                  _lib.ptr(gam), _lib.ptr(nrm), _lib.ptr(ccd)))
        k = min(n.value, cap)
        return idx[:k], gam[:k], nrm[:k], ccd[:k].astype(bool)

    def colliding(self):
        out = np.zeros(self.n, np.uint8)
        _lib.check(_lib.lib().vbd_get_colliding(self._h, _lib.ptr(out)))
        return out.astype(bool)

    def energy(self, h):
        """G(x) = 1/(2h^2)|x - y|_M^2 + E(x) at the device iterate (_assembly.py:78-82)."""
        g = ctypes.c_double()
        _lib.check(_lib.lib().vbd_energy(self._h, float(h), ctypes.byref(g)))
        return g.value

    def metrics(self, h):
        """(G, active contact count, max contact gap) at the device iterate in one reduction
        (the per-iteration columns of harness.py:664-670)."""
        g, n, d = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double()
        _lib.check(_lib.lib().vbd_energy_metrics(self._h, float(h), ctypes.byref(g), ctypes.byref(n),
                                                 ctypes.byref(d)))
        return g.value, int(n.value), d.value

    DESCEND_METHODS = {"vbd": 0, "vbd-cheb": 1, "jacobi": 2, "gd": 3}

    def descend(self, method, n_iters, h, rho=0.0, eps_det=1e-10, line_search=False):
        """baselines.descend (baselines.py:152-189) on the device from the resident x and y:
        returns (G per iteration (n_iters+1,), cumulative device ms (n_iters+1,))."""
        if method not in self.DESCEND_METHODS:
            raise ValueError(f"unknown solver {method!r}")
        g = np.zeros(int(n_iters) + 1)
        w = np.zeros(int(n_iters) + 1)
        _lib.check(_lib.lib().vbd_descend(self._h, self.DESCEND_METHODS[method], int(n_iters), float(h),
                                          float(rho), float(eps_det), 1 if line_search else 0,
                                          _lib.ptr(g), _lib.ptr(w)))
        return g, w

    def close(self):
        if self._h and self._h.value:
            _lib.check(_lib.lib().vbd_ctx_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- info ---------------------------------------------------------------------------
    def _info(self):
        i = _lib.CtxInfo()
        _lib.check(_lib.lib().vbd_ctx_get_info(self._h, ctypes.byref(i)))
        return i

    @property
    def num_colors(self):
        return int(self.info.num_colors)

    def color_counts(self):
        return [int(self.info.color_count[k]) for k in range(min(self.num_colors, 64))]

    def colors(self):
        out = np.empty(self.n, dtype=np.int64)
        _lib.check(_lib.lib().vbd_get_colors(self._h, _lib.ptr(out)))
        return out

    @property
    def stream(self):
        s = ctypes.c_void_p()
        _lib.check(_lib.lib().vbd_get_stream(self._h, ctypes.byref(s)))
        return s.value or 0

    def set_stream(self, handle):
        _lib.check(_lib.lib().vbd_set_stream(self._h, ctypes.c_void_p(handle or None)))

    # -- state --------------------------------------------------------------------------
    def set_state(self, x=None, x_t=None, v_t=None, v_prev=None, y=None):
        shape = (self.n, 3)
        arrs = [None if a is None else _lib.f64c(a, shape) for a in (x, x_t, v_t, v_prev, y)]
        _lib.check(_lib.lib().vbd_set_state(self._h, *[_lib.ptr(a) for a in arrs]))

    def get_state(self, x=True, x_t=False, v_t=False, v_prev=False, y=False, out=None):
        names = ("x", "x_t", "v_t", "v_prev", "y")
        want = dict(zip(names, (x, x_t, v_t, v_prev, y)))
        res = {}
        for k in names:
            if want[k]:
                res[k] = out[k] if out is not None and k in out else np.empty((self.n, 3))
        _lib.check(_lib.lib().vbd_get_state(self._h, *[_lib.ptr(res.get(k)) for k in names]))
        return res

    def set_fixed_targets(self, idx, xyz):
        i = _lib.i64c(idx).ravel()
        p = _lib.f64c(xyz, (len(i), 3))
        _lib.check(_lib.lib().vbd_set_fixed_targets(self._h, len(i), _lib.ptr(i), _lib.ptr(p)))

    def set_beam_velocities(self, lin_ang):
        a = _lib.f64c(lin_ang)
        _lib.check(_lib.lib().vbd_set_beam_velocities(self._h, _lib.ptr(a)))

    # -- hot path -----------------------------------------------------------------------
    @staticmethod
    def step_params(h, n_max, rho=0.0, eps_det=1e-10, init_mode="adaptive", a_ext=(0, 0, 0),
                    line_search=False):
        p = _lib.StepParams()
        p.line_search = 1 if line_search else 0
        p.h, p.n_max, p.rho, p.eps_det = float(h), int(n_max), float(rho), float(eps_det)
        p.init_mode = _lib.INIT_MODES[init_mode]
        p.a_ext = (ctypes.c_double * 3)(*map(float, a_ext))
        return p

    def step(self, params, n_steps=1, step_index=0):
        r = _lib.StepResult()
        _lib.check(_lib.lib().vbd_step(self._h, ctypes.byref(params), int(n_steps),
                                       ctypes.byref(r)))
        if r.nonfinite:
            raise NonFiniteState("non-finite vertex position", step=step_index + r.step,
                                 iteration=r.iteration, vertex=int(r.vertex))
        return r

    def initialize(self, params):
        _lib.check(_lib.lib().vbd_initialize(self._h, ctypes.byref(params)))

    def step_begin(self, params):
        _lib.check(_lib.lib().vbd_step_begin(self._h, ctypes.byref(params)))

    def step_color(self, color, iteration):
        _lib.check(_lib.lib().vbd_step_color(self._h, int(color), int(iteration)))

    def step_iter_end(self, iteration):
        _lib.check(_lib.lib().vbd_step_iter_end(self._h, int(iteration)))

    def step_end(self, step_index=0, raise_nonfinite=True):
        r = _lib.StepResult()
        _lib.check(_lib.lib().vbd_step_end(self._h, ctypes.byref(r)))
        if r.nonfinite and raise_nonfinite:
            raise NonFiniteState("non-finite vertex position", step=step_index,
                                 iteration=r.iteration, vertex=int(r.vertex))
        return r

    def color_pass(self, x, x_t, y, h, group, mode=0, line_search=False, eps_det=1e-10):
        if x.dtype != np.float64 or not x.flags["C_CONTIGUOUS"]:
            raise TypeError("x must be C-contiguous float64")  # _native.pyx:522-523
        g = _lib.i64c(group).ravel()
        xt = _lib.f64c(x_t, x.shape)
        yy = _lib.f64c(y, x.shape)
        _lib.check(_lib.lib().vbd_color_pass(self._h, _lib.ptr(x), _lib.ptr(xt), _lib.ptr(yy),
                                             float(h), _lib.ptr(g), len(g), int(mode),
                                             1 if line_search else 0, float(eps_det)))

    # -- halo (multi-GPU slabs) ---------------------------------------------------------
    def halo_count(self, side, color):
        ns, nr = ctypes.c_int64(0), ctypes.c_int64(0)
        _lib.check(_lib.lib().vbd_halo_count(self._h, side, color, ctypes.byref(ns),
                                             ctypes.byref(nr)))
        return ns.value, nr.value

    def halo_pack(self, side, color, dev_ptr):
        _lib.check(_lib.lib().vbd_halo_pack(self._h, side, color, ctypes.c_void_p(dev_ptr)))

    def halo_unpack(self, side, color, dev_ptr):
        _lib.check(_lib.lib().vbd_halo_unpack(self._h, side, color, ctypes.c_void_p(dev_ptr)))

    # -- fused P2P halo (multi-GPU slabs over peer memory) -------------------------------
    def ghost_blocks(self, side):
        nc = max(self.num_colors, 1)
        b, n, bd = (np.zeros(nc, np.int64) for _ in range(3))
        _lib.check(_lib.lib().vbd_halo_ghost_blocks(self._h, side, _lib.ptr(b), _lib.ptr(n),
                                                    _lib.ptr(bd)))
        return b[: self.num_colors], n[: self.num_colors], bd[: self.num_colors]

    def p2p_local_ptrs(self):
        pos, fl = ctypes.c_void_p(), ctypes.c_void_p()
        _lib.check(_lib.lib().vbd_halo_p2p_local(self._h, ctypes.byref(pos), ctypes.byref(fl)))
        return pos.value, fl.value

    def p2p_export(self):
        a, b = ctypes.create_string_buffer(64), ctypes.create_string_buffer(64)
        _lib.check(_lib.lib().vbd_halo_p2p_export(self._h, a, b))
        return a.raw, b.raw

    @staticmethod
    def ipc_open(device, handle):
        p = ctypes.c_void_p()
        _lib.check(_lib.lib().vbd_ipc_open(int(device), ctypes.c_char_p(handle), ctypes.byref(p)))
        return p.value

    def p2p_connect(self, side, peer_pos, peer_flags, peer_begin, peer_count):
        b = _lib.i64c(peer_begin)
        n = _lib.i64c(peer_count)
        _lib.check(_lib.lib().vbd_halo_p2p_connect(self._h, side, ctypes.c_void_p(peer_pos),
                                                   ctypes.c_void_p(peer_flags), _lib.ptr(b),
                                                   _lib.ptr(n)))

    def p2p_disconnect(self):
        """Drop both peer mappings (the K1 epilogue stops pushing into neighbour ghosts)."""
        for side in (0, 1):
            _lib.check(_lib.lib().vbd_halo_p2p_connect(self._h, side, None, None, None, None))

    def step_p2p_launch(self, params):
        _lib.check(_lib.lib().vbd_step_p2p_launch(self._h, ctypes.byref(params)))

    def step_p2p_finish(self, step_index=0):
        r = _lib.StepResult()
        _lib.check(_lib.lib().vbd_step_p2p_finish(self._h, ctypes.byref(r)))
        if r.nonfinite:
            raise NonFiniteState("non-finite vertex position", step=step_index,
                                 iteration=r.iteration, vertex=int(r.vertex))
        return r

    # -- measurement --------------------------------------------------------------------
    def profile_color_pass(self, h, reps=5):
        ms = np.zeros(max(self.num_colors, 1))
        _lib.check(_lib.lib().vbd_profile_color_pass(self._h, float(h), int(reps), _lib.ptr(ms)))
        return ms[: self.num_colors]
