"""Debug: step kernels vs each other on small scenes, per step (layouts x resident modes)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O
import paper_2403_06321_b200 as V

G = (0.0, 0.0, -9.8)
H = 1.0 / 60.0
VARS = {"explicit": dict(VBD_LAYOUT="explicit", VBD_TILES="1", VBD_RESIDENT="0", VBD_TILES_X="0"),
        "explicitX": dict(VBD_LAYOUT="explicit", VBD_TILES="1", VBD_RESIDENT="0", VBD_TILES_X="1"),
        "compact": dict(VBD_LAYOUT="auto", VBD_TILES="0", VBD_RESIDENT="0"),
        "k1t": dict(VBD_LAYOUT="auto", VBD_TILES="1", VBD_RESIDENT="0"),
        "repl": dict(VBD_LAYOUT="auto", VBD_TILES="1", VBD_RESIDENT="repl"),
        "glob": dict(VBD_LAYOUT="auto", VBD_TILES="1", VBD_RESIDENT="glob")}


def run(s, prec, var, nsteps, n_max, rho):
    for k, v in VARS[var].items():
        os.environ[k] = v
    ctx = V.DeviceContext.from_system(O.RefSystemView(s), precision=prec)
    z = np.zeros((s.num_vertices, 3))
    ctx.set_state(x=s.rest_positions, x_t=s.rest_positions, v_t=z, v_prev=z)
    p = ctx.step_params(H, n_max, rho, 1e-10, "adaptive", G)
    xs = []
    for _ in range(nsteps):
        ctx.step(p)
        xs.append(ctx.get_state(x=True)["x"])
    i = ctx._info()
    ctx.close()
    return xs, (i.layout, i.tiles > 0, i.resident)


for dims, mixed in (((13, 6, 6), False), ((41, 11, 11), False)):
    m = O.generate_beam(*dims, 0.05)
    fixed = np.flatnonzero(m.rest_positions[:, 0] < 1e-9)
    s = O.build_system([(m, (1e6, 1e7, 1e-6))], fixed)
    if mixed:
        pick = np.random.default_rng(3).random(len(s.tets)) < 0.5
        s.tet_mu = np.where(pick, 1e6, 3e6)
        s.tet_lam = np.where(pick, 1e7, 2e7)
        s.tet_kd = np.where(pick, 1e-6, 5e-6)
    for prec in ("fp32",):
        for rho in (0.0, 0.9):
            res = {v: run(s, prec, v, 3, 10, rho) for v in VARS}
            ref = res["explicit"][0]
            line = []
            for v, (xs, inf) in res.items():
                d = [float(np.abs(x - r).max()) for x, r in zip(xs, ref)]
                line.append(f"{v}{inf}:" + ",".join(f"{e:.1e}" for e in d))
            print(dims, "mixed" if mixed else "", prec, rho, " | ".join(line), flush=True)
