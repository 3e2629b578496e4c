"""K1R pass timeline on C1 (VBD_RES_DBG=8: CTA 0's clock64 stamps per colour pass; results
unchanged): mean cycles of sweep / reduce+solve+push / barrier per pass."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["VBD_RES_DBG"] = "8"
from paper_2403_06321_b200 import _lib
from paper_2403_06321_b200.scenes import build, config

cfg = config(sys.argv[1] if len(sys.argv) > 1 else "c1")
ctx, _ = build(cfg, precision="fp32")
p = cfg.step_params()
ctx.step(p, n_steps=5)
npass = cfg.n_max * ctx.num_colors
buf = (ctypes.c_int64 * (5 * npass))()
n = ctypes.c_int64()
_lib.check(_lib.lib().vbd_resident_timeline(ctx._h, buf, 5 * npass, ctypes.byref(n)))
t = np.frombuffer(buf, dtype=np.int64).reshape(npass, 5).astype(np.float64)
sweep, post, bar = t[:, 1] - t[:, 0], t[:, 2] - t[:, 1], t[:, 3] - t[:, 2]
total = t[:, 3] - t[:, 0]
print(f"{cfg.name} K1R CTA 0, {npass} passes, cycles per pass (mean / median):")
for name, v in (("start -> last sweep end", sweep), ("-> last push end", post), ("-> barrier exit", bar),
                ("pass total", total), ("one group: sweep end -> push end", t[:, 4])):
    print(f"  {name:26s} {v.mean():8.0f} {np.median(v):8.0f}")
gaps = t[1:, 0] - t[:-1, 3]
print(f"  barrier exit -> next start  {gaps.mean():8.0f}")
