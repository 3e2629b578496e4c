"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/vbd_b200.h declares with the ctypes signatures the host uses, and
fails loudly (no CPU fallback) when no GPU is present.  Host-only logic
(parameter validation, Chebyshev weights, procedural connectivity) is checked
against the oracle."""

import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "vbd_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vbd_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2403_06321_b200 import _lib
    L = _lib.lib()
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)
    assert _lib.lib().vbd_version().decode().startswith("vbd_b200")


def test_struct_layouts_match_header(tmp_path):
    """Every ctypes mirror has the size and field offsets the C compiler gives the header."""
    import ctypes
    import shutil
    import subprocess
    from paper_2403_06321_b200 import _lib
    mirrors = {"vbd_system_desc": _lib.SystemDesc, "vbd_beam_desc": _lib.BeamDesc,
               "vbd_step_params": _lib.StepParams, "vbd_step_result": _lib.StepResult,
               "vbd_ctx_info": _lib.CtxInfo}
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "vbd_b200.h"', "int main(void) {"]
    for cname, py in mirrors.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run([cc, "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = {}
    for ln in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n"):
        if ln:
            c, f, v = ln.split()
            got[(c, f)] = int(v)
    for cname, py in mirrors.items():
        assert got[(cname, "size")] == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2403_06321_b200 import _lib
    assert _lib.device_count() == 0
    import paper_2403_06321_b200 as V
    mesh = V.generate_beam(3, 2, 2, 0.1)
    with pytest.raises(Exception, match="no CUDA device"):
        V.build_system([V.Body(mesh, V.MaterialParams(1e5, 1e6))])
    with pytest.raises(Exception, match="no CUDA device"):
        V.DeviceContext.from_beams([V.Beam(3, 2, 2, 0.1, 1e5, 1e6)])


def test_host_mesh_matches_oracle(O):
    import paper_2403_06321_b200 as V
    for dims in ((2, 2, 2), (5, 3, 4), (9, 4, 4)):
        a = V.generate_beam(*dims, 0.05)
        b = O.generate_beam(*dims, 0.05)
        assert np.array_equal(a.tets, b.tets)
        assert np.array_equal(a.inv_rest_shape, b.inv_rest_shape)
        assert np.array_equal(a.masses, b.masses)
        assert np.array_equal(a.rest_volumes, b.rest_volumes)
    m = V.generate_beam(5, 3, 3, 0.1)
    adj = V.incidence(m)
    off, ids, slots = O.incidence_from_elements(m.tets, m.num_vertices)
    assert np.array_equal(adj.elem_offsets, off) and np.array_equal(adj.elem_ids, ids)
    assert np.array_equal(adj.elem_slots, slots)


def test_solver_params_validation():
    import paper_2403_06321_b200 as V
    for bad in (dict(h=0.0), dict(h=0.01, n_max=0), dict(h=0.01, rho=1.0),
                dict(h=0.01, n_col=0), dict(h=0.01, init_mode="warp"),
                dict(h=0.01, precision="fp16")):
        with pytest.raises(ValueError):
            V.SolverParams(**bad)


def test_chebyshev_matches_oracle(O):
    import paper_2403_06321_b200 as V
    for rho in (0.0, 0.5, 0.9, 0.95):
        for n in (1, 2, 3, 10, 60):
            assert V.chebyshev_omega(rho, n) == O.chebyshev_omega(rho, n)
    with pytest.raises(ValueError):
        V.chebyshev_omega(0.5, 0)


def test_backend_protocol_surface():
    import inspect
    from paper_2403_06321_b200 import backend
    assert backend.NAME == "b200"
    params = list(inspect.signature(backend.color_pass).parameters)
    # _native.pyx:513-515 order
    assert params[:13] == ["system", "carr", "x", "x_t", "y", "h", "group", "mode",
                           "line_search", "eps_det", "mu_c", "eps_v", "n_threads"]
