import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O
import paper_2403_06321_b200 as V
G = (0.0, 0.0, -9.8); H = 1.0 / 60.0
m = O.generate_beam(13, 6, 6, 0.05)
fixed = np.flatnonzero(m.rest_positions[:, 0] < 1e-9)
s = O.build_system([(m, (1e6, 1e7, 1e-6))], fixed)
ctxs = {}
for mode in ("repl", "0"):
    os.environ["VBD_RESIDENT"] = mode
    c = V.DeviceContext.from_system(O.RefSystemView(s), precision="fp32")
    z = np.zeros((s.num_vertices, 3))
    c.set_state(x=s.rest_positions, x_t=s.rest_positions, v_t=z, v_prev=z)
    ctxs[mode] = c
for n_max in (1, 2):
  for step in range(3):
    st = {}
    for mode, c in ctxs.items():
        c.step(c.step_params(H, n_max, 0.0, 1e-10, "adaptive", G))
        st[mode] = c.get_state(x=True, x_t=True, v_t=True, v_prev=True, y=True)
    print("n_max", n_max, "after step", step + 1, {k: float(np.abs(st["repl"][k] - st["0"][k]).max()) for k in st["0"]})
    bad = np.flatnonzero(np.abs(st["repl"]["x"] - st["0"]["x"]).max(1) > 0)
    print("  bad vertices", bad[:10], "fixed?", np.isin(bad[:10], fixed), "colors", s.color_of[bad[:10]])
