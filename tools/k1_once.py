"""Build one bench scene and run a few colour passes (for ncu captures of K1).

    python tools/k1_once.py c5 fp32 [--fma]
    ncu --metrics ... -k regex:k1_tiles --launch-skip 8 -c 1 python tools/k1_once.py c5 fp32

--fma runs the FMA-peak microbenchmark instead (vbd_fma_peak, fp32x2 and fp64).
"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
    from paper_2403_06321_b200 import _lib
    if "--fma" in sys.argv:
        for p, packed in ((0, 1), (0, 0), (1, 0)):
            out = ctypes.c_double()
            _lib.check(_lib.lib().vbd_fma_peak(0, p, packed, 0.5, ctypes.byref(out)))
            print(f"fma peak precision={p} packed={packed}: {out.value:.2f} TFLOP/s")
        return
    from paper_2403_06321_b200.scenes import build, config
    cfg = config(name)
    ctx, _ = build(cfg, precision=prec)
    ctx.step(cfg.step_params())
    i = ctx._info()
    print("tiles", i.tiles, "stages", i.tile_stages, "smem/CTA", i.tile_smem_bytes, "nbr_cap", i.tile_nbr_cap,
          "ent_cap", i.tile_ent_cap, "kinds", i.num_entry_kinds, "class_tiles", i.class_tiles,
          "class_vertices", i.class_vertices, "of", i.num_solved, "class_records", i.class_records)
    print("k1 ms per colour:", ctx.profile_color_pass(cfg.h, reps=2))
    ctx.close()


if __name__ == "__main__":
    main()
