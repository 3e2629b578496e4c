"""The golden 'extras' scene (tests/golden/extras_scene.npz, written by the reference in
make_golden.extras_fixture): a beam, a spring cloth and a spring chain with fixed, subspace
and world-box constraints, rebuilt from the fixture's arrays with the oracle's builder."""

import numpy as np


def extras_system(O, g):
    m = O.generate_beam(7, 3, 3, 0.05)
    nb = m.num_vertices
    nc = len(g["cloth_parts"])
    sub = [(nb - 1, [[0.0], [0.0], [1.0]], m.rest_positions[-1]),
           (nb - 2, [[1.0, 0.0], [0.0, 1.0], [0.0, 0.0]], m.rest_positions[-2])]
    boxes = [(nb + v, (-1.0, -1.0, 0.185), (2.0, 2.0, 1.0), 1e4) for v in range(nc)]
    s = O.build_system_ex(
        [(m, (1e6, 1e7, 1e-6))],
        [(g["cloth_parts"], g["cloth_m"], g["cloth_idx"], g["cloth_l0"], g["cloth_k"], 1e-3),
         (g["chain_parts"], g["chain_m"], g["chain_idx"], g["chain_l0"], g["chain_k"], 5e-4)],
        fixed=[int(v) for v in g["fixed"]], subspace=sub, boxes=boxes)
    assert np.array_equal(s.color_of, g["color_of"])
    return m, s
