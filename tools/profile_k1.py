"""Small driver for ncu: build a BASELINE config on cuda:0, run one step, then a few
colour passes (the K1 launches ncu captures)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--precision", default="fp32")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()

from paper_2403_06321_b200.scenes import build, config  # noqa: E402

cfg = config(a.config, a.scale)
ctx, _ = build(cfg, precision=a.precision)
inf = ctx._info()
print("tiles", inf.tiles, "ent_cap", inf.tile_ent_cap, "nbr_cap", inf.tile_nbr_cap, "stages",
      inf.tile_stages, "smem/CTA", inf.tile_smem_bytes, "kinds", inf.num_entry_kinds)
ctx.step(cfg.step_params())
print("k1 ms per colour:", ctx.profile_color_pass(cfg.h, reps=a.reps))
