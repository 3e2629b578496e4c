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


class ContactCall:
    """ContactArrays look-alike (_system.py:86-96) of one recorded colour pass."""

    def __init__(self, g, k):
        for name in ("idx", "gamma", "refresh", "normal", "tangent", "k_c", "cv_off", "cv_cid",
                     "cv_slot"):
            setattr(self, name, g[f"call{k}_{name}"])
        self.count = len(self.idx)


def contact_system(O):
    """tests/golden/make_golden.contact_scene rebuilt with the oracle's builder."""
    import numpy as np
    n = 4
    light = O.generate_beam(n, n, n, 0.3 / (n - 1), density=10.0)
    heavy0 = O.generate_beam(n, n, n, 0.2 / (n - 1), density=2000.0)
    heavy = O.build_tet_mesh(heavy0.rest_positions + [0.05, 0.05, 0.3005], heavy0.tets, 2000.0)
    bottom = [i for i in range(light.num_vertices) if light.rest_positions[i, 2] < 1e-9]
    return O.build_system([(light, (1e6, 1e7, 0.0)), (heavy, (1e6, 1e7, 0.0))], bottom)
