"""Small-scene runs of every step kernel for compute-sanitizer (racecheck / memcheck / synccheck).

    compute-sanitizer --tool racecheck python tools/sanitize.py [case ...]

cases: k1t (K1T tiles, per-colour graph), k1t_class (K1T with grid-class tiles), k1r (K1R cluster-resident step), k1r_glob (grid-
resident), k1 (global-memory K1, compact), explicit (48-byte entries), slabs (3 slabs, host-
driven halo pack / unpack), p2p (3 slabs on 3 streams with the fused NVLink-style halo stores
and phase flags: needs concurrent kernels, so it cannot run under a sanitizer, which
serialises them), fp64 (K1T fp64 split stage)."""
import os
import sys
import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
G = (0.0, 0.0, -9.8)


def env(**kw):
    for k in ("VBD_RESIDENT", "VBD_TILES", "VBD_LAYOUT"):
        os.environ.pop(k, None)
    os.environ.update(kw)


def beam_case(V, prec="fp32", steps=2, rho=0.9):
    beam = V.Beam(13, 6, 6, 0.05, 1e6, 1e7, 1e-6, fix_min_x=True)
    ctx = V.DeviceContext.from_beams([beam], precision=prec)
    p = ctx.step_params(1 / 60, 4, rho, 1e-10, "adaptive", G)
    for _ in range(steps):
        ctx.step(p)
    x = ctx.get_state(x=True)["x"]
    assert np.isfinite(x).all()
    info = ctx._info()
    ctx.close()
    return info


def main():
    import paper_2403_06321_b200 as V
    cases = sys.argv[1:] or ["k1t", "k1r", "k1r_glob", "k1", "explicit", "fp64", "slabs"]
    for c in cases:
        if c == "k1t":
            env(VBD_RESIDENT="0")
            i = beam_case(V)
            assert i.tiles > 0 and i.resident == 0
        elif c == "k1t_class":  # grid-class tiles (one lane per vertex, neighbours in registers)
            env(VBD_RESIDENT="0", VBD_TILE_V="64", VBD_ENTRY_ORDER="code")
            beam = V.Beam(40, 10, 9, 0.02, 1e6, 1e7, 1e-6, fix_min_x=True)
            ctx = V.DeviceContext.from_beams([beam], precision="fp32")
            p = ctx.step_params(1 / 120, 4, 0.9, 1e-10, "adaptive", G)
            for _ in range(2):
                ctx.step(p)
            assert np.isfinite(ctx.get_state(x=True)["x"]).all()
            assert ctx._info().class_tiles > 0
            ctx.close()
            os.environ.pop("VBD_TILE_V", None)
            os.environ.pop("VBD_ENTRY_ORDER", None)
        elif c == "k1r":
            env(VBD_RESIDENT="repl")
            assert beam_case(V).resident == 1
        elif c == "k1r_glob":
            env(VBD_RESIDENT="glob")
            assert beam_case(V).resident == 2
        elif c == "k1":
            env(VBD_RESIDENT="0", VBD_TILES="0")
            assert beam_case(V).tiles == 0
        elif c == "explicit":
            env(VBD_RESIDENT="0", VBD_LAYOUT="explicit")
            assert beam_case(V).layout == 0
        elif c == "fp64":
            env(VBD_RESIDENT="0")
            assert beam_case(V, "fp64").tiles > 0
        elif c == "slabs":  # host-driven halo exchange (pack / unpack per colour) over 3 slabs
            env()
            from paper_2403_06321_b200.dist import SlabExchange
            beam = V.Beam(24, 7, 6, 0.02, 1e6, 1e7, 1e-6, fix_min_x=True)
            cuts = [0, 7, 15, beam.nx]
            slabs = [V.DeviceContext.from_beams([beam], precision="fp32", slab=(cuts[r], cuts[r + 1]))
                     for r in range(3)]
            ex = SlabExchange.local(slabs)
            p = slabs[0].step_params(1 / 120, 4, 0.9, 1e-10, "adaptive", G)
            for _ in range(2):
                ex.step(p)
            for s in slabs:
                assert np.isfinite(s.get_state(x=True)["x"]).all()
        elif c == "p2p":
            env()
            from paper_2403_06321_b200.dist import SlabP2P
            beam = V.Beam(24, 7, 6, 0.02, 1e6, 1e7, 1e-6, fix_min_x=True)
            cuts = [0, 7, 15, beam.nx]
            slabs = [V.DeviceContext.from_beams([beam], precision="fp32", slab=(cuts[r], cuts[r + 1]))
                     for r in range(3)]
            ex = SlabP2P.local(slabs)
            p = slabs[0].step_params(1 / 120, 4, 0.9, 1e-10, "adaptive", G)
            for _ in range(2):
                ex.step(p)
            for s in slabs:
                assert np.isfinite(s.get_state(x=True)["x"]).all()
        print("case", c, "ok", flush=True)


if __name__ == "__main__":
    main()
