"""K1R step time vs n_max on C1 (per-pass slope and fixed per-step cost), CUDA events."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_06321_b200.scenes import build, config

for mode, dbg in (("repl", "0"), ("repl", "1"), ("repl", "2"), ("0", "0")):
    os.environ["VBD_RESIDENT"] = mode
    os.environ["VBD_RES_DBG"] = dbg
    cfg = config("c1")
    ctx, _ = build(cfg, precision="fp32")
    stream = torch.cuda.ExternalStream(ctx.stream)
    out = []
    for n_max in (1, 2, 5, 10, 20, 40):
        p = ctx.step_params(cfg.h, n_max, 0.0, 1e-10, "adaptive", cfg.a_ext)
        for _ in range(5):
            ctx.step(p)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        ctx.step(p, n_steps=50)
        e1.record(stream)
        torch.cuda.synchronize()
        out.append((n_max, e0.elapsed_time(e1) / 50 * 1e3))
    ns, ts = np.array(out).T
    k, b = np.polyfit(ns, ts, 1)
    print(mode, "dbg", dbg, " ".join(f"n_max={int(n)}:{t:.1f}us" for n, t in out), f"| slope {k / 4:.2f} us/pass, intercept {b:.1f} us")
    ctx.close()
