"""K1R GLOB on C2: step time vs n_max, normal and without the entry sweep (VBD_RES_DBG=2),
to size the grid barrier (CUDA events, n_steps=20 per launch batch)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_06321_b200.scenes import build, config

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
for mode, dbg in (("glob", "0"), ("glob", "2"), ("0", "0")):
    os.environ["VBD_RESIDENT"] = mode
    os.environ["VBD_RES_DBG"] = dbg
    cfg = config(name)
    ctx, _ = build(cfg, precision="fp32")
    stream = torch.cuda.ExternalStream(ctx.stream)
    out = []
    for n_max in (1, 5, 20, 50):
        p = ctx.step_params(cfg.h, n_max, 0.0, 1e-10, "adaptive", cfg.a_ext)
        try:
            ctx.step(p, n_steps=3)
        except Exception:
            pass
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        try:
            ctx.step(p, n_steps=20)
        except Exception:
            pass
        e1.record(stream)
        torch.cuda.synchronize()
        out.append((n_max, e0.elapsed_time(e1) / 20 * 1e3))
    ns, ts = np.array(out).T
    k, b = np.polyfit(ns, ts, 1)
    print(name, mode, "dbg", dbg, "resident", ctx._info().resident, " ".join(f"n_max={int(n)}:{t:.1f}us" for n, t in out),
          f"| slope {k / 4:.2f} us/pass, intercept {b:.1f} us", flush=True)
    ctx.close()
