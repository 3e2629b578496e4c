import faulthandler, os, sys, time
faulthandler.dump_traceback_later(500, exit=True)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_06321_b200.scenes import build, config
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
t = time.time()
cfg = config("c5j", scale)
ctx, info = build(cfg, precision="fp32")
print("built", time.time() - t, "s", ctx.info.layout, ctx.info.num_entry_kinds, flush=True)
t = time.time()
ctx.step(cfg.step_params())
print("step", time.time() - t, flush=True)
print("k1", ctx.profile_color_pass(cfg.h, reps=2), flush=True)
