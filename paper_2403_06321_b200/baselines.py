"""Convergence instrumentation of the reference (pkg/src/vbdsim/baselines.py) on the device.

``descend`` records G per iteration for the sweep solvers on the frozen objective of one step
-- "vbd" (colour sweeps), "vbd-cheb" (colour sweeps + Chebyshev blend), "jacobi"
(``block_jacobi_step``: every vertex against the previous iterate) and "gd" (``gd_step``:
diagonally preconditioned gradient steps, kernel mode 1), the last two wrapped every 8
iterations by the global backtracking line search toward the last checkpoint
(baselines.py:139-189).  The whole trace is one C-ABI call (``vbd_descend``): sweeps, the G
reduction after every iteration and the line-search trials run on the GPU; only the line
search's accept test reads a scalar back.  ``wall_ms`` is device time (CUDA events) rather
than the reference's host clock.

Newton (``newton_step`` / ``minimize_newton`` / ``global_gradient_hessian``) assembles and
factorises the PSD-projected global Hessian with SciPy; it is a comparison baseline, not the
VBD hot path, and is not provided here (``NotImplementedError``, no CPU fallback).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import EmptyDescentRange
from .solver import color_pass, device_context

_LS_PERIOD = 8       # baselines.py:22
_MAX_HALVINGS = 16   # baselines.py:23
METHODS = ("vbd", "vbd-cheb", "jacobi", "gd")


@dataclass
class SolverTrace:
    """baselines.py:35-40."""

    method: str
    g: np.ndarray        # G at iterations 0..n
    wall_ms: np.ndarray  # cumulative device time, wall_ms[0] == 0
    x_final: np.ndarray


def energy(state, params) -> float:
    """baselines.py:42-44 (device reduction, ``solver.energy``)."""
    from .solver import energy as _energy
    return _energy(state, params)


def block_jacobi_step(state, params):
    """baselines.py:92-97: one simultaneous pass of block solves over every vertex."""
    color_pass(state, np.arange(state.system.num_vertices, dtype=np.int64), params, mode=0)
    return state


def gd_step(state, params):
    """baselines.py:100-104: one simultaneous pass of preconditioned gradient steps."""
    color_pass(state, np.arange(state.system.num_vertices, dtype=np.int64), params, mode=1)
    return state


def relative_loss(g_values, g_star: float) -> np.ndarray:
    """baselines.py:107-115: (G - G*) / (G_0 - G*); EmptyDescentRange without a descent range."""
    g = np.asarray(g_values, dtype=np.float64)
    denom = float(g[0]) - g_star
    if not denom > 0.0:
        raise EmptyDescentRange(f"G_0 - G* = {denom:.3e} leaves no descent range")
    return (g - g_star) / denom


def descend(state, params, method: str, n_iters: int) -> SolverTrace:
    """baselines.py:152-189 on the device: ``n_iters`` iterations of ``method`` from state.x
    against state.y, no detection updates.  state.x is left at the final iterate."""
    if method == "newton":
        raise NotImplementedError("newton is not provided by the b200 backend (global sparse "
                                  "factorisation baseline, not the VBD hot path)")
    if method not in METHODS:
        raise ValueError(f"unknown solver {method!r}")
    ctx = device_context(state.system, params.precision, params.device)
    state._bind(ctx)
    state._upload(("x_t", "x", "y"))  # x_t: the damping term of the block solve
    g, wall = ctx.descend(method, n_iters, params.h, rho=params.rho, eps_det=params.eps_det,
                          line_search=params.line_search)
    state._stale_host.add("x")
    return SolverTrace(method, g, wall, state.x.copy())


def newton_step(state, params):
    raise NotImplementedError("newton_step is not provided by the b200 backend")


def global_gradient_hessian(state, params, psd_project: bool = True):
    raise NotImplementedError("global_gradient_hessian is not provided by the b200 backend")


def minimize_newton(state, params, tol: float = 1e-10, max_iters: int = 200):
    raise NotImplementedError("minimize_newton is not provided by the b200 backend")
