"""Implicit-Euler stepping by per-vertex block descent on the B200.

Mirrors pkg/src/vbdsim/solver.py (SolverParams, SimState, make_state, step,
inertia_target, initialize, chebyshev_omega, accelerate, color_pass,
local_solve).  ``step`` runs the whole time step on the GPU as one CUDA graph:
K2 (inertia target + warm start), n_max x (one K1 colour pass per colour, K3
Chebyshev blend + non-finite check), K4 velocity commit.

SimState keeps the reference's attribute interface (x_t, v_t, v_prev, x, y as
(N,3) float64 arrays) with lazy host/device coherence: arrays stay resident on
the device between steps and are copied to the host only when read; anything
read or assigned on the host is re-uploaded before the next step.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .context import DeviceContext
from .errors import NonFiniteState
from .system import FIXED, SUBSPACE, compile_constraints

INIT_MODES = ("prev_pos", "inertia", "inertia_accel", "adaptive")
PRECISIONS = ("fp64", "fp32")
_FIELDS = ("x_t", "v_t", "v_prev", "x", "y")
_INPUTS = ("x_t", "v_t", "v_prev")


@dataclass(frozen=True)
class ContactParams:
    """solver.py ContactParams: penalty stiffness, friction, DCD radius and depth bound;
    detection and contact terms run on the device."""

    k_c: float
    mu_c: float = 0.0
    eps_v: float = 1e-2
    dcd_radius: float = 1e-3
    max_depth: float = None

    def __post_init__(self):
        if self.k_c <= 0.0:
            raise ValueError("k_c must be positive")
        if self.mu_c < 0.0:
            raise ValueError("mu_c must be >= 0")
        if self.eps_v <= 0.0:
            raise ValueError("eps_v must be positive")
        if self.dcd_radius < 0.0:
            raise ValueError("dcd_radius must be >= 0")


@dataclass(frozen=True)
class SolverParams:
    """solver.py:51-85 plus ``precision`` ("fp64" parity build, "fp32" performance
    build) and ``device`` (CUDA ordinal)."""

    h: float
    substeps: int = 1
    n_max: int = 10
    n_col: int = 4
    rho: float = 0.0
    eps_det: float = 1e-10
    line_search: bool = False
    init_mode: str = "adaptive"
    a_ext: tuple = (0.0, 0.0, 0.0)
    threads: int = 0
    contact: ContactParams = None
    precision: str = "fp64"
    device: int = 0

    def __post_init__(self):
        if self.h <= 0.0:
            raise ValueError("h must be positive")
        if self.substeps < 1:
            raise ValueError("substeps must be >= 1")
        if self.n_max < 1:
            raise ValueError("n_max must be >= 1")
        if self.n_col < 1:
            raise ValueError("n_col must be >= 1")
        if not 0.0 <= self.rho < 1.0:
            raise ValueError("rho must be in [0, 1)")
        if self.eps_det < 0.0:
            raise ValueError("eps_det must be >= 0")
        if self.init_mode not in INIT_MODES:
            raise ValueError(f"init_mode must be one of {INIT_MODES}")
        if self.precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {PRECISIONS}")
        object.__setattr__(self, "a_ext", tuple(float(v) for v in np.reshape(self.a_ext, 3)))

    @property
    def a_ext_vec(self) -> np.ndarray:
        return np.asarray(self.a_ext)


def device_context(system, precision="fp64", device=0) -> DeviceContext:
    """The packed device scene for ``system`` (cached on the System object)."""
    cache = getattr(system, "_contexts", None)
    if cache is None:
        cache = {}
        try:
            system._contexts = cache
        except AttributeError:
            pass
    key = (precision, device)
    ctx = cache.get(key)
    if ctx is None:
        ctx = DeviceContext.from_system(system, precision=precision, device=device)
        ctx.owner = None
        cache[key] = ctx
    return ctx


def _evict(ctx):
    """Make the host copy of ctx's current owner authoritative before reuse."""
    owner = ctx.owner() if getattr(ctx, "owner", None) is not None else None
    if owner is not None:
        owner._detach()
    ctx.owner = None


class SimState:
    """Mutable per-simulation state (solver.py:88-108) with lazy device coherence."""

    def __init__(self, system, x_t, v_t, v_prev, x, y, step_index=0):
        self.system = system
        self._h = {"x_t": x_t, "v_t": v_t, "v_prev": v_prev, "x": x, "y": y}
        self._stale_host = set()
        self._stale_dev = set(_FIELDS)
        self._ctx = None
        self.step_index = step_index
        self.contact_set = None
        self.carr = None
        self._x_prev1 = None
        self._x_pp = None

    # coherence ---------------------------------------------------------------------
    def _pull(self, names):
        names = [n for n in names if n in self._stale_host]
        if not names:
            return
        got = self._ctx.get_state(**{n: True for n in _FIELDS if n in names},
                                  **{n: False for n in _FIELDS if n not in names})
        for n in names:
            self._h[n] = got[n]
            self._stale_host.discard(n)

    def _detach(self):
        self._pull(list(self._stale_host))
        self._stale_dev = set(_FIELDS)
        self._ctx = None

    def _bind(self, ctx):
        if self._ctx is not ctx:
            if self._ctx is not None:
                self._detach()
            _evict(ctx)
            self._ctx = ctx
            self._stale_dev = set(_FIELDS)
            ctx.owner = weakref.ref(self)

    def _upload(self, names):
        todo = [n for n in names if n in self._stale_dev]
        if todo:
            self._ctx.set_state(**{n: self._h[n] for n in todo})
            for n in todo:
                self._stale_dev.discard(n)


def _field(name):
    def get(self):
        if name in self._stale_host:
            self._pull([name])
        self._stale_dev.add(name)  # the caller may mutate the returned array
        return self._h[name]

    def put(self, value):
        self._h[name] = np.ascontiguousarray(value, dtype=np.float64)
        self._stale_host.discard(name)
        self._stale_dev.add(name)
    return property(get, put)


for _n in _FIELDS:
    setattr(SimState, _n, _field(_n))


def make_state(system, x0=None, v0=None) -> SimState:
    """solver.py:111-117."""
    x = np.array(system.rest_positions if x0 is None else x0, dtype=np.float64)
    v = np.zeros_like(x) if v0 is None else np.array(v0, dtype=np.float64)
    if x.shape != (system.num_vertices, 3) or v.shape != x.shape:
        raise ValueError("state arrays must be (N,3)")
    return SimState(system, x.copy(), v.copy(), v.copy(), x.copy(), x.copy())


def inertia_target(x_t, v_t, a_ext, h: float) -> np.ndarray:
    """y = x_t + h v_t + h^2 a_ext (solver.py:120-122); K2 computes it on the device."""
    return np.asarray(x_t) + h * np.asarray(v_t) + h * h * np.asarray(a_ext)


def chebyshev_omega(rho: float, n: int) -> float:
    """solver.py:167-177 (the step's K3 weights come from the same recurrence)."""
    if n < 1:
        raise ValueError("iteration index must be >= 1")
    if rho == 0.0 or n == 1:
        return 1.0
    omega = 2.0 / (2.0 - rho * rho)
    for _ in range(3, n + 1):
        omega = 4.0 / (4.0 - rho * rho * omega)
    return omega


def _check_supported(state, params):
    """Contacts: detection runs on the device (vbd_set_collision) when the system has a
    collision surface (solver.py:235-238)."""


def _dparams(params):
    return DeviceContext.step_params(params.h, params.n_max, params.rho, params.eps_det,
                                     params.init_mode, params.a_ext, params.line_search)


def initialize(state, params) -> np.ndarray:
    """Warm start (solver.py:125-164) computed by K2 on the device; returns state.x."""
    _check_supported(state, params)
    ctx = device_context(state.system, params.precision, params.device)
    state._bind(ctx)
    state._upload(_INPUTS)
    ctx.initialize(_dparams(params))
    got = ctx.get_state(x=True, y=True)
    state._h["x"], state._h["y"] = got["x"], got["y"]
    state._stale_host.discard("x")
    state._stale_host.discard("y")
    return state._h["x"]


def _collision(ctx, system, params):
    key = (params.contact, params.n_col)
    if getattr(ctx, "_coll_key", None) != key:
        ctx.set_collision(system if params.contact is not None else None, params.contact, params.n_col)
        ctx._coll_key = key


def step(state, params, on_iteration=None):
    """Advance one step of size params.h on the GPU (solver.py:291-324)."""
    _check_supported(state, params)
    ctx = device_context(state.system, params.precision, params.device)
    _collision(ctx, state.system, params)
    state._bind(ctx)
    state._upload(_INPUTS)
    if on_iteration is None:
        try:
            ctx.step(_dparams(params), 1, state.step_index)
        except NonFiniteState:
            state._stale_host.update(("x", "y"))
            state._stale_dev.discard("x")
            raise
    else:
        ctx.step_begin(_dparams(params))
        for n in range(1, params.n_max + 1):
            for c in range(ctx.num_colors):
                ctx.step_color(c, n)
            ctx.step_iter_end(n)
            state._stale_host.update(("x", "y"))
            state._stale_dev.difference_update(("x", "y"))
            on_iteration(state, n)
            if "x" in state._stale_dev:
                state._upload(("x",))
        r = ctx.step_end(state.step_index, raise_nonfinite=False)
        if r.nonfinite:
            state._stale_host.update(("x", "y"))
            raise NonFiniteState("non-finite vertex position", step=state.step_index,
                                 iteration=r.iteration, vertex=int(r.vertex))
    state._stale_host.update(_FIELDS)
    state._stale_dev.clear()
    state.step_index += 1
    return state


def energy(state, params) -> float:
    """baselines.energy (baselines.py:42-44): G(x) = 1/(2h^2)|x - y|_M^2 + E(x)
    (_assembly.py:78-82) evaluated on the device.  Inside ``step(on_iteration=...)`` the
    iterate is already resident, so the per-iteration metric of harness.run_simulation
    (harness.py:664-678) costs no host transfer of x."""
    ctx = device_context(state.system, params.precision, params.device)
    state._bind(ctx)
    state._upload(("x", "y"))
    return ctx.energy(params.h)


def metrics(state, params):
    """(G, active contact count, max contact gap) at the iterate in one device reduction:
    the per-iteration columns of harness.run_simulation (harness.py:664-670)."""
    ctx = device_context(state.system, params.precision, params.device)
    state._bind(ctx)
    state._upload(("x", "y"))
    return ctx.metrics(params.h)


def max_penetration(state, params=None) -> float:
    """solver.py:327-332: the largest gap d = max(0, (x_b - x_a) . n) over the active contact
    set at state.x (0 without contacts), from the device contact set."""
    ctx = state._ctx
    if ctx is None:
        return 0.0
    state._upload(("x", "y"))
    return ctx.metrics(params.h if params is not None else 1.0)[2]


def color_pass(state, color_group, params, mode: int = 0) -> None:
    """One aux-buffer colour pass through the b200 backend (solver.py:191-201)."""
    from . import backend
    group = np.asarray(color_group, dtype=np.int64)
    backend.color_pass(state.system, state.carr, state.x, state.x_t, state.y, params.h, group,
                       mode, line_search=params.line_search, eps_det=params.eps_det,
                       precision=params.precision, device=params.device)


def local_solve(i: int, state, params, constraints=None):
    """Displacement of the single-vertex solve at i (solver.py:204-218), on the GPU."""
    sys_ = state.system
    if constraints is not None:
        if not hasattr(constraints, "kind"):
            constraints = compile_constraints(constraints, sys_.num_vertices)
        sys_ = replace(sys_, cons=constraints, _contexts={})
    from . import backend
    xc = np.array(state.x, dtype=np.float64)
    backend.color_pass(sys_, None, xc, state.x_t, state.y, params.h,
                       np.array([i], dtype=np.int64), 0, line_search=params.line_search,
                       eps_det=params.eps_det, precision=params.precision, device=params.device)
    return xc[i] - state.x[i]


def accelerate(state, omega: float, contact_set=None) -> np.ndarray:
    """Chebyshev blend x <- omega (x - x_pp) + x_pp on the host arrays
    (solver.py:221-232; inside ``step`` the same blend is K3 on the device)."""
    if omega == 1.0 or state._x_pp is None:
        return state.x
    cs = contact_set if contact_set is not None else state.contact_set
    x = state.x
    blended = omega * (x - state._x_pp) + state._x_pp
    if cs is not None and getattr(cs, "colliding_flag", np.zeros(0, bool)).any():
        blended[cs.colliding_flag] = x[cs.colliding_flag]
    x[...] = blended
    return x
