"""The ``b200`` kernel backend: a drop-in for the reference's backend protocol.

pkg/src/vbdsim/_backend.py:13-32 selects a module exposing ``NAME`` and
``color_pass(system, carr, x, x_t, y, h, group, mode=0, line_search=False,
eps_det=1e-10, mu_c=0.0, eps_v=1e-2, n_threads=0)`` (_native.pyx:513-515).
This module has the same surface; ``color_pass`` runs K1 on the GPU with the
reference's auxiliary-buffer semantics (every group vertex reads the current x,
results are merged afterwards) and mutates ``x`` in place.  A non-empty contact
array (``carr``, detected by the caller) adds the contact penalty and friction
terms on the device.

Accepts the reference's own System objects as well as this package's.  No CPU
fallback: without a GPU or without libvbd_b200.so every call raises.
"""

import os

import numpy as np

from . import _lib

NAME = "b200"
DEFAULT_PRECISION = os.environ.get("VBD_B200_PRECISION", "fp64")


def max_threads():
    """Threads are a CPU notion; report the CUDA device count instead (>= 1 on a GPU box)."""
    return max(1, _lib.device_count())


def _has_contacts(carr):
    return carr is not None and getattr(carr, "count", 0)


def color_pass(system, carr, x, x_t, y, h, group, mode=0, line_search=False, eps_det=1e-10,
               mu_c=0.0, eps_v=1e-2, n_threads=0, precision=None, device=0):
    """One auxiliary-buffer colour pass over ``group`` on the GPU, updating x in place."""
    from .solver import _evict, device_context
    g = np.ascontiguousarray(group, dtype=np.int64).ravel()
    if len(g) == 0:
        return  # _native.pyx:520-521
    if x.dtype != np.float64 or not x.flags["C_CONTIGUOUS"]:
        raise TypeError("x must be C-contiguous float64")
    ctx = device_context(system, precision or DEFAULT_PRECISION, device)
    _evict(ctx)
    if _has_contacts(carr):  # penalty + friction terms of _native.pyx:351-399 on the device
        ctx.set_contacts(carr, mu_c, eps_v)
    elif getattr(ctx, "_contacts", None) is not None:
        ctx.set_contacts(None)
    ctx.color_pass(x, x_t, y, h, g, mode=mode, line_search=line_search, eps_det=eps_det)
