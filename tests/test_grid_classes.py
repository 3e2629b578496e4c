"""Grid-class templates of the K1T class tiles (csrc/vbd_grid_classes.cuh).

CPU checks: the committed header is what tools/gen_grid_classes.py derives from the mesh
generator (harness.py:42-76 restated in mesh.py); the device's pattern code (signs of E = W^-1
from cofactors of the slot-weight rows, vbd_build.cuh entry_code) equals the generator's (signs
of rest edges); and every interior vertex of a beam matches one class, boundary vertices none.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))

import gen_grid_classes as gen  # noqa: E402
from paper_2403_06321_b200 import mesh  # noqa: E402
from paper_2403_06321_b200.system import _slot_weight_rows  # noqa: E402


def test_header_matches_generator():
    text = (ROOT / "paper_2403_06321_b200" / "csrc" / "vbd_grid_classes.cuh").read_text()
    assert text == gen.emit(gen.classes())


def code_from_rows(W4, sl):
    """entry_code (vbd_build.cuh): cofactor signs of the other three slot rows."""
    w = np.array([W4[q] for q in range(4) if q != sl])
    cr = np.array([np.cross(w[(c + 1) % 3], w[(c + 2) % 3]) for c in range(3)])
    det = float(w[0] @ cr[0])
    tol = 1e-9 * np.abs(cr).max()
    code, p = 0, 1
    for v in cr.ravel():
        d = 1 if abs(v) <= tol else (2 if (v > 0) == (det > 0) else 0)
        code += d * p
        p *= 3
    return code


def slot_rows(m, t):
    """the system's tet_w rows of tet t (_system.py:139-144, restated in system.py)."""
    return _slot_weight_rows(m.inv_rest_shape[t:t + 1])[0]


def test_device_pattern_code_equals_generator_code():
    for jitter in (0.0, 0.2):
        m = mesh.generate_beam(5, 4, 4, 0.01)
        X = m.rest_positions.copy()
        if jitter:
            X = X + np.random.default_rng(1).uniform(-jitter, jitter, X.shape) * 0.01
            m = mesh.build_tet_mesh(X, m.tets, 1000.0)
            X = m.rest_positions
        for t, tet in enumerate(m.tets):
            W4 = slot_rows(m, t)
            for sl in range(4):
                others = [int(tet[q]) for q in range(4) if q != sl]
                assert code_from_rows(W4, sl) == gen.entry_code(X, int(tet[sl]), others)


def test_interior_vertices_match_a_class():
    cls = gen.classes()
    n = 7
    m = mesh.generate_beam(n, n - 1, n - 2, 0.02)
    X, T = m.rest_positions, m.tets
    inc = [[] for _ in range(len(X))]
    for t, tet in enumerate(T):
        for r in range(4):
            inc[tet[r]].append((t, r))
    ijk = np.round(X / 0.02).astype(int)
    dims = np.array([n, n - 1, n - 2])
    for v in range(len(X)):
        ents = sorted((gen.entry_code(X, v, [int(T[t][q]) for q in range(4) if q != r]),
                       [int(T[t][q]) for q in range(4) if q != r]) for t, r in inc[v])
        codes = tuple(c for c, _ in ents)
        match = None
        for k, (ccodes, nbr) in enumerate(cls):
            if codes != ccodes:
                continue
            loc = {}
            ok = all(loc.setdefault(nbr[q][r], o) == o for q, (_, oth) in enumerate(ents) for r, o in enumerate(oth))
            if ok:
                match = k
        interior = ijk[v].min() > 0 and (ijk[v] < dims - 1).all()
        assert (match is not None) == interior, (v, ijk[v])
