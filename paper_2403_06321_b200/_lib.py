"""ctypes binding of libvbd_b200.so (include/vbd_b200.h).

There is no CPU fallback: if the library is missing this module raises on import of
any compute entry point, and every call that needs a GPU fails loudly with the
library's own error message.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from .errors import VbdError

HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("VBD_B200_LIB", HERE / "libvbd_b200.so"))

VBD_OK = 0
VBD_ERR_ARG = -1
VBD_ERR_CUDA = -2
VBD_ERR_UNSUPPORTED = -3
VBD_ERR_NODEVICE = -5
VBD_ERR_INTERNAL = -6
PREC = {"fp32": 0, "fp64": 1}
INIT_MODES = {"prev_pos": 0, "inertia": 1, "inertia_accel": 2, "adaptive": 3}

P = ctypes.c_void_p
i64 = ctypes.c_int64
i32 = ctypes.c_int32
f64 = ctypes.c_double


class SystemDesc(ctypes.Structure):
    _fields_ = [("num_vertices", i64), ("num_tets", i64), ("tets", P), ("tet_w", P),
                ("tet_vol", P), ("tet_mu", P), ("tet_lam", P), ("tet_kd", P), ("masses", P),
                ("kind", P), ("t_off", P), ("t_id", P), ("t_slot", P), ("num_colors", i64),
                ("color_off", P), ("color_verts", P), ("rest_positions", P),
                ("num_springs", i64), ("springs", P), ("sp_l0", P), ("sp_k", P), ("sp_kd", P),
                ("sub_dim", P), ("sub_basis", P), ("sub_anchor", P), ("box_k", P),
                ("box_lo", P), ("box_hi", P)]


class BeamDesc(ctypes.Structure):
    _fields_ = [("nx", i64), ("ny", i64), ("nz", i64), ("spacing", f64), ("density", f64),
                ("origin", f64 * 3), ("mu", f64), ("lam", f64), ("kd", f64),
                ("fix_min_x", i32), ("fix_max_x", i32), ("jitter", f64)]


class StepParams(ctypes.Structure):
    _fields_ = [("h", f64), ("n_max", i32), ("init_mode", i32), ("rho", f64),
                ("eps_det", f64), ("a_ext", f64 * 3), ("line_search", i32), ("reserved", i32)]


class StepResult(ctypes.Structure):
    _fields_ = [("nonfinite", i32), ("step", i32), ("iteration", i32), ("reserved", i32),
                ("vertex", i64)]


class CtxInfo(ctypes.Structure):
    _fields_ = [("num_vertices", i64), ("num_solved", i64), ("num_ghost", i64),
                ("num_fixed", i64), ("num_tets", i64), ("num_entries", i64),
                ("num_colors", i64), ("color_count", i64 * 64), ("device_bytes", i64),
                ("precision", i32), ("inplace", i32), ("lanes_per_vertex", i32),
                ("num_materials", i32), ("layout", i32), ("entry_bytes", i32),
                ("num_entry_kinds", i64), ("tiles", i32), ("tile_nbr_cap", i32),
                ("tile_slots", i64), ("tile_nbr_refs", i64), ("tile_lanes", i32),
                ("tile_stages", i32), ("tile_ent_cap", i32), ("tile_smem_bytes", i32),
                ("resident", i32), ("resident_ctas", i32),
                ("contact_graph_steps", i64), ("contact_graph_fallbacks", i64),
                ("class_vertices", i64), ("class_tiles", i32), ("class_records", i32)]


# name -> (restype, argtypes); must match include/vbd_b200.h (checked by tests)
SIGNATURES = {
    "vbd_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "vbd_ctx_create": (ctypes.c_int, [ctypes.POINTER(SystemDesc), ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(P)]),
    "vbd_ctx_create_beams": (ctypes.c_int, [ctypes.POINTER(BeamDesc), i64, i64, i64,
                                            ctypes.c_int, ctypes.c_int, ctypes.POINTER(P)]),
    "vbd_ctx_destroy": (ctypes.c_int, [P]),
    "vbd_ctx_get_info": (ctypes.c_int, [P, ctypes.POINTER(CtxInfo)]),
    "vbd_set_stream": (ctypes.c_int, [P, P]),
    "vbd_get_stream": (ctypes.c_int, [P, ctypes.POINTER(P)]),
    "vbd_get_colors": (ctypes.c_int, [P, P]),
    "vbd_set_state": (ctypes.c_int, [P, P, P, P, P, P]),
    "vbd_get_state": (ctypes.c_int, [P, P, P, P, P, P]),
    "vbd_set_beam_velocities": (ctypes.c_int, [P, P]),
    "vbd_set_fixed_targets": (ctypes.c_int, [P, i64, P, P]),
    "vbd_step": (ctypes.c_int, [P, ctypes.POINTER(StepParams), i32, ctypes.POINTER(StepResult)]),
    "vbd_color_pass": (ctypes.c_int, [P, P, P, P, f64, P, i64, i32, i32, f64]),
    "vbd_initialize": (ctypes.c_int, [P, ctypes.POINTER(StepParams)]),
    "vbd_step_begin": (ctypes.c_int, [P, ctypes.POINTER(StepParams)]),
    "vbd_step_color": (ctypes.c_int, [P, i32, i32]),
    "vbd_step_iter_end": (ctypes.c_int, [P, i32]),
    "vbd_step_end": (ctypes.c_int, [P, ctypes.POINTER(StepResult)]),
    "vbd_halo_count": (ctypes.c_int, [P, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
    "vbd_halo_pack": (ctypes.c_int, [P, i32, i32, P]),
    "vbd_halo_unpack": (ctypes.c_int, [P, i32, i32, P]),
    "vbd_halo_ghost_blocks": (ctypes.c_int, [P, i32, P, P, P]),
    "vbd_halo_p2p_local": (ctypes.c_int, [P, ctypes.POINTER(P), ctypes.POINTER(P)]),
    "vbd_halo_p2p_export": (ctypes.c_int, [P, P, P]),
    "vbd_ipc_open": (ctypes.c_int, [ctypes.c_int, P, ctypes.POINTER(P)]),
    "vbd_ipc_close": (ctypes.c_int, [P]),
    "vbd_halo_p2p_connect": (ctypes.c_int, [P, i32, P, P, P, P]),
    "vbd_step_p2p_launch": (ctypes.c_int, [P, ctypes.POINTER(StepParams)]),
    "vbd_step_p2p_finish": (ctypes.c_int, [P, ctypes.POINTER(StepResult)]),
    "vbd_greedy_color": (ctypes.c_int, [i64, P, P, P, ctypes.c_int, P, ctypes.POINTER(i64)]),
    "vbd_resident_timeline": (ctypes.c_int, [P, ctypes.POINTER(i64), i64, ctypes.POINTER(i64)]),
    "vbd_profile_color_pass": (ctypes.c_int, [P, f64, i32, P]),
    "vbd_fma_peak": (ctypes.c_int, [i32, i32, i32, f64, P]),
    "vbd_energy": (ctypes.c_int, [P, f64, ctypes.POINTER(f64)]),
    "vbd_energy_metrics": (ctypes.c_int, [P, f64, ctypes.POINTER(f64), ctypes.POINTER(i64),
                                          ctypes.POINTER(f64)]),
    "vbd_descend": (ctypes.c_int, [P, i32, i32, f64, f64, f64, i32, P, P]),
    "vbd_set_contacts": (ctypes.c_int, [P, i64, P, P, P, P, P, P, P, P, P, f64, f64]),
    "vbd_set_collision": (ctypes.c_int, [P, i64, P, i64, P, f64, f64, f64, f64, f64, i32, f64, i32]),
    "vbd_detect_contacts": (ctypes.c_int, [P, i32, i64, ctypes.POINTER(i64), P, P, P, P]),
    "vbd_get_colliding": (ctypes.c_int, [P, P]),
    "vbd_last_error": (ctypes.c_char_p, []),
    "vbd_version": (ctypes.c_char_p, []),
}

_lib = None


def lib():
    """Load the native library (raises if it is missing -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C paper_2403_06321_b200/csrc` "
            "or __graft_entry__.build(); the B200 path has no CPU fallback")
    L = ctypes.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


class NativeError(VbdError):
    def __init__(self, code, message):
        super().__init__(f"[vbd_b200 {code}] {message}")
        self.code = code


def check(rc):
    if rc == VBD_OK:
        return
    msg = lib().vbd_last_error().decode(errors="replace")
    if rc == VBD_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == VBD_ERR_ARG:
        raise ValueError(msg)
    raise NativeError(rc, msg)


def ptr(a):
    return None if a is None else a.ctypes.data_as(P)


def f64c(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None and a.shape != shape:
        raise ValueError(f"expected shape {shape}, got {a.shape}")
    return a


def i64c(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def device_count():
    n = ctypes.c_int(0)
    check(lib().vbd_device_count(ctypes.byref(n)))
    return n.value
