"""Benchmark of the B200 VBD hot path (BASELINE.json metric: vertex-iterations/s and
ms/timestep at 1/2/4/8 B200 vs the CPU reference).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--precision fp32]
    python bench.py --impl reference ...      # the reference's own CPU kernel (oracle/_ref)

A "step" is one VBD time step (K2 init, n_max x (one colour pass per colour + Chebyshev),
K4 commit) of the whole scene; value = total vertex-iterations (N x n_max per step, all
ranks) / the max-over-ranks device time of the K timed steps.  The default workload is
BASELINE config 5 (single 364^3 tet block, 48.2M vertices / 239.2M tets, S=4 -> h=1/240,
n_max=40), which fits one B200; --config c4 is the 10,368-object scene.  Multi-GPU:
one process per GPU (torchrun), slabs with a per-colour NCCL halo exchange (c5) or object
shards with no data-path communication (c4).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "VBD vertex-iterations/sec and ms/timestep at 1/2/4/8 B200 vs CPU ref"
UNIT = "vertex-iterations/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 10; C1/C2/C3: enough for a >= 1 s timed region, "
                         "so the clock sampler sees it -- 10000 / 600 / 500)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5", "c5j"])
    ap.add_argument("--scale", type=float, default=1.0, help="shrink c4/c5 (tests only)")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--halo", default="p2p", choices=["p2p", "nccl"],
                    help="slab halo transport for N>1: fused peer-memory push or NCCL send/recv")
    ap.add_argument("--checksum", action="store_true",
                    help="add the sha256 of the owned positions after warm-up + timed steps "
                         "(rank order = vertex order) -- for the 1-rank vs N-rank bitwise test")
    ap.add_argument("--no-fp64-record", action="store_true",
                    help="skip the fp64 sub-record (the reference's precision) of the fp32 run")
    args = ap.parse_args()
    if args.steps is None:
        small = {"c1": 10000, "c2": 600, "c3": 500}
        args.steps = small.get(args.config, 10) if args.impl == "ours" else 10
    return args


# ----------------------------------------------------------------------------------------
# CPU reference (oracle/_ref: the reference's own compiled kernel; else the oracle port)

def _stock_reference():
    """The unmodified reference package (pip-installed into baseline/_ref), or None."""
    path = ROOT / "baseline" / "_ref"
    if not (path / "vbdsim").exists():
        return None
    if str(path) not in sys.path:
        sys.path.insert(0, str(path))
    try:
        import vbdsim
    except Exception:
        return None
    return vbdsim if vbdsim.backend_name() == "native" else None


def _sample_meshes(cfg_name, cfg, shrink=1.0):
    b = cfg.beams[0]
    if cfg_name == "c4":
        k = max(1, int(round(8 * shrink)))
        return [(b.nx, b.ny, b.nz, b.spacing)] * k, f"{k} of the 10,368 generate_cube(15,0.3) objects"
    if cfg_name in ("c5", "c5j"):
        n = max(8, int(round(31 * shrink ** (1 / 3))))
        return [(n, n, n, b.spacing)], (f"generate_beam({n},{n},{n},0.01) block (same material/h/n_max/BCs"
                                        + ("; regular rest shapes: the reference's per-tet cost does not "
                                           "depend on them)" if cfg_name == "c5j" else ")"))
    if cfg_name == "c3":
        n = max(8, int(round(300 * shrink)))
        return [(n, 4, 4, b.spacing)], f"generate_beam({n},4,4,0.01) (part of one C3 beam)"
    return [(bb.nx, bb.ny, bb.nz, bb.spacing) for bb in cfg.beams], "full scene"


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_reference_sample(cfg_name, budget_s=15.0, steps=None, warmup=1):
    """Time the reference on a bounded sample of the workload, on this box's host cores.

    Preferred: the UNMODIFIED reference package from baseline/_ref through its own public
    API (vbdsim.generate_beam / build_system / make_state / step, compiled native backend).
    Fallback: the reference's compiled kernel (oracle/_ref) driven by the oracle's step loop,
    else the oracle's C port.  The sample is a scaled-down scene of the same kind (same
    generator, material, h, n_max, rho, constraints); vertex-iterations/s is
    size-independent to first order.  The as-shipped kernel takes the GIL per tet inside its
    OpenMP loop, so 1 thread and all host threads are both timed (one step
    each) and the faster setting is used for the timed steps; both rates are reported.

    steps=None: as many steps as fit in budget_s (>= 3); else exactly `steps` timed steps
    after `warmup` untimed ones, on a sample shrunk so that they take about budget_s.
    """
    from paper_2403_06321_b200.scenes import config
    cfg = config(cfg_name)
    b = cfg.beams[0]
    shrink = 1.0
    if steps is not None and cfg_name in ("c3", "c4", "c5", "c5j"):
        # the 31^3 C5 sample takes ~1.8 s per step on one core
        shrink = min(1.0, budget_s / (1.8 * max(1, steps + warmup)))
    dims, sample = _sample_meshes(cfg_name, cfg, shrink)
    ncores = len(os.sched_getaffinity(0))
    vb = _stock_reference()
    if vb is not None:
        kind, how = "reference", "vbdsim.step (baseline/_ref, unmodified, native backend)"
        meshes = []
        for k, (nx, ny, nz, sp) in enumerate(dims):
            m = vb.generate_beam(nx, ny, nz, sp, density=b.density)
            meshes.append(vb.build_tet_mesh(m.rest_positions + np.array([0.0, 0.0, 2.0 * k]),
                                            m.tets, b.density))
        fixed, off = [], 0
        for m in meshes:
            if b.fix_min_x:
                fixed.extend((off + np.flatnonzero(m.rest_positions[:, 0] < 1e-9)).tolist())
            off += m.num_vertices
        s = vb.build_system([vb.Body(m, vb.MaterialParams(b.mu, b.lam, b.kd)) for m in meshes],
                            [vb.FixedConstraint(int(v)) for v in fixed])
        n_total, n_tets = s.num_vertices, len(s.tets)
        rest = s.rest_positions

        def make():
            return vb.make_state(s, x0=_x0(rest)) if cfg.random_init else vb.make_state(s)

        def one_step(st, threads):
            prm = vb.SolverParams(h=cfg.h, n_max=cfg.n_max, rho=cfg.rho, a_ext=cfg.a_ext,
                                  threads=threads)
            t0 = time.perf_counter()
            vb.step(st, prm)
            return time.perf_counter() - t0
    else:
        from oracle import oracle as O
        ref = O.ref_native()
        kind = "reference" if ref is not None else "port"
        how = "oracle step loop + " + ("oracle/_ref kernel" if ref is not None else "oracle C port")
        meshes = []
        for k, (nx, ny, nz, sp) in enumerate(dims):
            m = O.generate_beam(nx, ny, nz, sp, b.density)
            meshes.append(O.build_tet_mesh(m.rest_positions + np.array([0.0, 0.0, 2.0 * k]),
                                           m.tets, b.density))
        fixed, off = [], 0
        for m in meshes:
            if b.fix_min_x:
                fixed.extend((off + np.flatnonzero(m.rest_positions[:, 0] < 1e-9)).tolist())
            off += m.num_vertices
        s = O.build_system([(m, (b.mu, b.lam, b.kd)) for m in meshes], fixed)
        n_total, n_tets = s.num_vertices, len(s.tets)
        rest = s.rest_positions

        def make():
            return O.make_state(s, x0=_x0(rest)) if cfg.random_init else O.make_state(s)

        def one_step(st, threads):
            t0 = time.perf_counter()
            O.step(s, st, cfg.h, cfg.n_max, cfg.rho, cfg.a_ext, kernel=ref, n_threads=threads)
            return time.perf_counter() - t0

    vit = n_total * cfg.n_max
    probe = {}
    for threads in sorted({1, ncores}):
        probe[threads] = vit / one_step(make(), threads)
    threads = max(probe, key=probe.get)
    st = make()
    for _ in range(max(0, warmup)):
        one_step(st, threads)
    times = []
    t_start = time.perf_counter()
    if steps is not None:
        for _ in range(steps):
            times.append(one_step(st, threads))
    else:
        while len(times) < 3 or (time.perf_counter() - t_start < budget_s and len(times) < 20):
            times.append(one_step(st, threads))
            if time.perf_counter() - t_start > 2 * budget_s:
                break
    ms = 1e3 * statistics.mean(times)
    rate = vit / (ms / 1e3)
    return {"value": rate, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{sample}: {n_total} vertices, {n_tets} tets, n_max={cfg.n_max}; {how}; "
                      f"mean of {len(times)} steps after {warmup} warm-up, {ms:.1f} ms/step at "
                      f"{threads} thread(s)",
            "threads_probe": {f"{t}_threads": r for t, r in probe.items()},
            "host_threads": ncores, "cpu_model": cpu_model(),
            "sample_vertices": n_total, "sample_tets": n_tets, "sample_steps": len(times),
            "sample_warmup": warmup, "ms_per_step_sample": ms}


def _x0(rest):
    lo, hi = rest.min(0), rest.max(0)
    return np.random.default_rng(0).uniform(lo, hi, size=rest.shape)


# ----------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------------------

def algorithmic_bytes_per_iteration(info, precision):
    """SURVEY.md §8(d)'s algorithmic (compulsory-traffic) bytes of one iteration in the
    reference's data model: per vertex-iteration 4 (CSR offset) + 52 (x_i, x_t,i, y_i read,
    m_i, x_i write) + 52 d_v (3 neighbour ids + Dm^-1 + V per incident tet) + 12 (C - 1)
    (other-colour positions), i.e. B_iter = 92 N + 208 T for fp32 (C = 4) and 180 N + 368 T
    for fp64.  This is the `achieved` numerator of the roofline."""
    n, t, C = int(info.num_vertices), int(info.num_tets), int(info.num_colors)
    if precision == "fp32":
        return n * (4 + 52 + 12 * (C - 1)) + 4 * t * 52
    return n * (8 + 104 + 24 * (C - 1)) + 4 * t * 92


def layout_bytes_per_iteration(info, precision):
    """Compulsory DRAM bytes the kernels actually move per iteration in the layout in use
    (DESIGN.md §4): K1T tiles: 8 B per entry slot + 4 B per neighbour-list entry + 64 B per
    tile descriptor + x, x_t, y read and x written per solved vertex + one read of every
    other-colour position per colour pass; explicit / compact K1: entry_bytes per entry +
    8 B CSR offset + the same per-vertex terms."""
    r4 = 16 if precision == "fp32" else 32
    n_solved = int(info.num_solved)
    n_all = int(info.num_vertices)
    C = int(info.num_colors)
    other = sum(r4 * (n_all - int(info.color_count[c])) for c in range(min(C, 64)))
    if int(info.tiles):  # K1T; K1T-X (explicit layout) also streams 36 B of rows per slot
        rows = 36 * int(info.tile_slots) if int(info.layout) == 0 else 0
        return (8 * int(info.tile_slots) + rows + 4 * int(info.tile_nbr_refs) + 64 * int(info.tiles)
                + 4 * r4 * n_solved + other)
    return n_solved * (8 + 4 * r4) + int(info.num_entries) * int(info.entry_bytes) + other


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def fma_peak_tflops(device, precision, seconds=1.0):
    """Measured FMA-pipe peak of this GPU (vbd_fma_peak: independent FMA chains on every SM,
    packed fp32x2 FFMA2 for fp32, DFMA for fp64) run for `seconds` -- the denominator of the
    FP32 / FP64 roofline (MEASURED_PEAKS.json has no FP32 figure)."""
    import ctypes
    from paper_2403_06321_b200 import _lib
    out = ctypes.c_double(0.0)
    prec = 1 if precision == "fp64" else 0
    _lib.check(_lib.lib().vbd_fma_peak(int(device), prec, 1, float(seconds), ctypes.byref(out)))
    return out.value


def ncu_flops(cfg_name, precision, variant):
    """Executed floating-point operations of one K1 launch, from ncu SASS counters
    (profiles/k1_flops.json; FFMA / DFMA = 2, FFMA2 = 4, FADD2 / FMUL2 = 2)."""
    p = ROOT / "profiles" / "k1_flops.json"
    if not p.exists():
        return None
    return json.loads(p.read_text()).get(f"{cfg_name}_{precision}_{variant}")


def reference_model_flops_per_iteration(info):
    """~259 flops per (vertex, tet) entry in the reference's formulation
    (_native.pyx:181-198, 292-317) + ~75 per vertex (inertia, adjugate solve, update)."""
    return 75 * int(info.num_vertices) + 259 * 4 * int(info.num_tets)


def ncu_traffic(cfg_name, precision, variant):
    p = ROOT / "profiles" / "k1_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    return d.get(f"{cfg_name}_{precision}_{variant}")


def ncu_limiter(cfg_name, precision, variant):
    """The measured limiter of the colour pass from the committed ncu capture
    (profiles/k1_limiter.json): SOL percentages of the pipes that bound it."""
    p = ROOT / "profiles" / "k1_limiter.json"
    if not p.exists():
        return None
    return json.loads(p.read_text()).get(f"{cfg_name}_{precision}_{variant}")


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        args.gpus = world
    # one process per GPU; VBD_DIST_BACKEND=gloo (tests only) lets several ranks share a GPU
    backend = os.environ.get("VBD_DIST_BACKEND", "nccl")
    if world > 1 and backend == "nccl":   # communicator init lines (nranks) on stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    red_dev = "cuda" if backend == "nccl" else "cpu"
    if world > 1:  # first collective: every rank takes part (before any P2P batch)
        dist.all_reduce(torch.zeros(1, device=red_dev))
    from paper_2403_06321_b200.dist import SlabExchange
    from paper_2403_06321_b200.scenes import build, config

    cfg = config(args.config, args.scale)
    t_build = time.perf_counter()
    ctx, part = build(cfg, rank, world, args.precision, device=local)
    t_build = time.perf_counter() - t_build
    info = ctx.info
    p = cfg.step_params()
    exch = None
    if world > 1 and cfg.sharding == "slabs":
        if args.halo == "p2p":  # fused K1 push into the neighbour's ghosts over NVLink
            from paper_2403_06321_b200.dist import SlabP2P
            ok = 1.0
            try:
                exch = SlabP2P.distributed(ctx, rank, world, device=local)
            except Exception as e:  # e.g. no peer access between these GPUs
                print(f"rank {rank}: P2P halo setup failed ({e}); using the NCCL halo", file=sys.stderr)
                ok = 0.0
            flag = torch.tensor([ok], device=red_dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)  # every rank takes the same path
            if flag.item() < 1.0:
                args.halo = "nccl"
                ctx.p2p_disconnect()
                exch = SlabExchange.distributed(ctx, rank, world)
        else:                   # NCCL send/recv per colour
            exch = SlabExchange.distributed(ctx, rank, world)
    stream = torch.cuda.ExternalStream(ctx.stream) if ctx.stream else torch.cuda.current_stream()

    twist = None
    if cfg.twist_rev_s:  # C3: clamped ends driven kinematically, x_t rewritten every step
        from paper_2403_06321_b200.scenes import twist_targets
        rest = ctx.get_state(x=False, x_t=True)["x_t"]
        twist = {"rest": rest, "k": 0}

    def do_steps(k):
        if twist is not None:
            for _ in range(k):
                twist["k"] += 1
                idx, xyz = twist_targets(cfg, twist["rest"], twist["k"] * cfg.h)
                ctx.set_fixed_targets(idx, xyz)
                ctx.step(p)
        elif exch is None:
            ctx.step(p, n_steps=k)
        else:
            for _ in range(k):
                exch.step(p)

    clk = Clocks(local).__enter__()  # sampled from warm-up through the timed region
    do_steps(args.warmup)
    torch.cuda.synchronize()
    n_owned = int(info.num_solved + info.num_fixed) if exch is None else \
        (part[1] - part[0]) * cfg.beams[0].ny * cfg.beams[0].nz
    tot = torch.tensor([float(n_owned)], device=red_dev)
    if world > 1:
        dist.all_reduce(tot)
    n_total = int(tot.item())

    def timed(fn, strm=None):
        """CUDA-event time of fn() on the stream its kernels run on, max over ranks."""
        strm = stream if strm is None else strm
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(strm)
        fn()
        e1.record(strm)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        t = torch.tensor([ms], device=red_dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dist.barrier()
        return float(t.item())

    ms_total = timed(lambda: do_steps(args.steps))
    clk.__exit__(None, None, None)
    ms_step = ms_total / args.steps
    vit_per_step = n_total * cfg.n_max
    value = vit_per_step * args.steps / (ms_total / 1e3)
    checksum = state_checksum(ctx, cfg, part, exch, rank, world) if args.checksum else None

    # dominant kernel (K1) live timing on the same stream: average per-colour launch time
    # n_max sweeps in step order straight after the timed region: one step's worth of launches,
    # so the kernel runs at the same power-capped sustained clock as inside the step (a short
    # burst of 10 sweeps reads about 6 % faster on C5)
    k1_reps = max(10, cfg.n_max)
    k1_ms = ctx.profile_color_pass(cfg.h, reps=k1_reps)
    roof = roofline_record(cfg, info, args.precision, k1_ms, k1_reps, local)
    phases = 1 + cfg.n_max * (int(info.num_colors) + (1 if cfg.rho else 0)) + 1
    launches_per_step = phases
    resident = int(ctx._info().resident)  # decided at the first step (small scenes: K1R)
    if resident:
        launches_per_step = 1
        roof["step_kernel"] = ("k_step_resident (K1R, %s, %d CTAs): the whole step is one launch; the "
                               "k1 timing above is the per-colour K1T pass of the graph path"
                               % ("cluster replicas" if resident == 1 else "grid", int(ctx._info().resident_ctas)))
    if exch is not None and args.halo == "p2p":
        launches_per_step = 3 * phases + 1   # + phase wait / signal kernels, epoch advance
    elif exch is not None:
        launches_per_step += cfg.n_max * int(info.num_colors) * 4  # pack/unpack per side

    # end-to-end through the C ABI with host buffers: H2D of the step's inputs (x_t, v_t,
    # v_prev, (N,3) float64, pinned) + step + D2H of the result (x, v_t)
    n_loc = int(info.num_vertices)
    pin = lambda: torch.empty((n_loc, 3), dtype=torch.float64, pin_memory=True).numpy()
    hx, hxt, hv, hvp = pin(), pin(), pin(), pin()
    ctx.get_state(x=True, x_t=True, v_t=True, v_prev=True,
                  out={"x": hx, "x_t": hxt, "v_t": hv, "v_prev": hvp})

    bufs = {"x_t": hxt, "v_t": hv, "v_prev": hvp, "spare": hx}

    def e2e_steps(b=bufs):
        for _ in range(args.e2e_steps):
            ctx.set_state(x_t=b["x_t"], v_t=b["v_t"], v_prev=b["v_prev"])
            if twist is not None:
                twist["k"] += 1
                ctx.set_fixed_targets(*twist_targets(cfg, twist["rest"], twist["k"] * cfg.h))
            if exch is None:
                ctx.step(p)
            else:
                exch.step(p)
            # D2H of the result: x into the spare buffer, v_t into the retiring v_prev
            ctx.get_state(x=True, v_t=True, out={"x": b["spare"], "v_t": b["v_prev"]})
            # host-side commit as the reference's SimState does (x_t = x, v_prev = v_t),
            # by rotating buffers instead of copying them
            b["x_t"], b["spare"] = b["spare"], b["x_t"]
            b["v_t"], b["v_prev"] = b["v_prev"], b["v_t"]
    e2e_ms = timed(e2e_steps) / args.e2e_steps
    e2e_value = vit_per_step / (e2e_ms / 1e3)
    h2d = 3 * 24 * n_total
    d2h = 2 * 24 * n_total
    # the same loop through ordinary (pageable) numpy arrays -- what SimState hands the API
    pageable = {k: np.array(v) for k, v in bufs.items()}
    e2e_pageable_ms = timed(lambda: e2e_steps(pageable)) / args.e2e_steps
    del hx, hxt, hv, hvp, bufs, pageable

    # the reference's precision (fp64), timed in the same run on the same scene
    fp64 = None
    if (world == 1 and args.precision == "fp32" and not args.no_fp64_record
            and cfg.name in ("c4", "c5")):
        if exch is not None:
            exch = None
        ctx.close()
        ctx = None
        try:
            fp64 = fp64_record(cfg, local, timed)
        except Exception as e:  # pragma: no cover - reported, not fatal
            fp64 = {"error": str(e)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_sample(args.config, args.cpu_seconds)
            cpu.pop("ms_per_step_sample", None)
        except Exception as e:  # pragma: no cover - reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
                   "sample": f"failed: {e}"}

    clocks = clk.summary() if rank == 0 else None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if args.precision == "fp32" else "f64",
            "data": "synthetic (procedural generate_beam/cube scene built on the device)",
            "config": {
                "workload": f"{cfg.name}: {cfg.description}",
                "num_vertices": cfg.num_vertices, "num_tets": cfg.num_tets,
                "h": cfg.h, "n_max": cfg.n_max, "rho": cfg.rho, "substeps_S": round(1 / (cfg.h * 60)),
                "colors": int(info.num_colors),
                "parallelism": (f"{cfg.sharding}x{world}" + (f" ({args.halo} halo)" if cfg.sharding == "slabs" else "")
                                if world > 1 else "single GPU"),
                "dist_backend": backend if world > 1 else None,
                "layout": layout_name(info),
                "l2": ("inputs larger than L2: %.1f GB of layout bytes (slots, neighbour lists, "
                       "tile descriptors, per-vertex state) read per iteration per GPU, no flush"
                       % (roof["_layout_iter"] / 1e9)) if roof["_layout_iter"] > 4 * 126e6
                      else "scene fits in L2 (no flush)",
                "build_s": round(t_build, 2),
            },
            "roofline": {k: v for k, v in roof.items() if not k.startswith("_")},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                    "host_memory": "pinned (page-locked) numpy buffers",
                    "pageable": {"ms_per_step": e2e_pageable_ms,
                                 "value": vit_per_step / (e2e_pageable_ms / 1e3),
                                 "host_memory": "ordinary numpy arrays (pageable)"}},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
        }
        if fp64 is not None:
            line["fp64"] = fp64
        if checksum is not None:
            line["state_sha256"] = checksum
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if ctx is not None:
        ctx.close()


def state_checksum(ctx, cfg, part, exch, rank, world):
    """sha256 of the positions this run owns, concatenated in rank order (= original vertex
    order for slabs and object shards), after warm-up + timed steps."""
    import hashlib

    import torch.distributed as dist
    x = ctx.get_state(x=True)["x"]
    if exch is not None and cfg.sharding == "slabs":
        plane = cfg.beams[0].ny * cfg.beams[0].nz
        lo = max(part[0] - 1, 0)
        x = x[(part[0] - lo) * plane:(part[1] - lo) * plane]
    x = np.ascontiguousarray(x)
    if world > 1:
        allx = [None] * world
        dist.all_gather_object(allx, x)
        x = np.concatenate(allx)
    return hashlib.sha256(x.tobytes()).hexdigest() if rank == 0 else None


def layout_name(info):
    if int(info.tiles) and int(info.layout) == 0:
        return ("K1T-X tiles (irregular mesh, %d lanes/vertex, %d stages): 8 B entry slots + 36 B of "
                "slot-weight rows per slot streamed, constants derived per entry" % (info.tile_lanes, info.tile_stages))
    if int(info.tiles) and int(info.class_tiles):
        return ("K1T tiles (%d stages) with grid-class tiles: %d of %d solved vertices one lane per vertex, "
                "8 B neighbour-offset rows, neighbours in registers, %d class records; the rest 2 lanes/vertex, "
                "8 B entry slots + %d entry kinds"
                % (info.tile_stages, info.class_vertices, info.num_solved, info.class_records,
                   info.num_entry_kinds))
    if int(info.tiles):
        return ("K1T tiles (%d lanes/vertex, %d stages): 8 B entry slots + %d entry kinds"
                % (info.tile_lanes, info.tile_stages, info.num_entry_kinds))
    if info.layout == 1:
        return "compact: 16 B entries + %d entry kinds" % info.num_entry_kinds
    return "explicit: %d B entries" % info.entry_bytes


def roofline_record(cfg, info, precision, k1_ms, k1_reps, device):
    """The HBM roofline of the dominant kernel (K1, one colour pass per launch) and its FP32 /
    FP64 roofline.

    HBM: `achieved` = the compulsory bytes of the layout actually used (DESIGN.md §4:
    slots, neighbour lists, tile descriptors, own-vertex state, other-colour positions) per
    launch / the live CUDA-event launch time; `peak` = MEASURED_PEAKS.json hbm_gbs.  The
    SURVEY §8(d) figure (the reference's data model, Dm^-1 stored per entry) is reported
    separately as `reference_model` -- it exceeds the peak because the entry dictionary
    replaces those bytes losslessly.
    FP: executed flops per launch from ncu SASS counters (profiles/k1_flops.json) / the same
    launch time, against the FMA peak measured live (vbd_fma_peak) after the timed region."""
    bytes_iter = algorithmic_bytes_per_iteration(info, precision)
    layout_iter = layout_bytes_per_iteration(info, precision)
    ncol = max(1, int(info.num_colors))
    k1_iter_ms = float(np.sum(k1_ms))
    peak, peak_kind = load_peaks()
    layout_achieved = layout_iter / (k1_iter_ms / 1e3) / 1e9
    ref_achieved = bytes_iter / (k1_iter_ms / 1e3) / 1e9
    kname = "k1_tiles" if int(info.tiles) else "k1_color_pass"
    variant = ("classtiles" if int(info.class_tiles) else "tiles") if int(info.tiles) else (
        "compact" if int(info.layout) == 1 else "explicit")
    rec = {"bound": "hbm", "achieved": layout_achieved, "peak": peak, "unit": "GB/s",
           "frac": layout_achieved / peak,
           "traffic": ncu_traffic(cfg.name, precision, variant),
           "kernel": kname, "peak_source": peak_kind,
           "bytes_per_launch": layout_iter / ncol,
           "bytes_model": "layout bytes (DESIGN.md §4): 8 B per entry slot + 4 B per neighbour-list "
                          "entry + 64 B per tile + x, x_t, y read and x written per solved vertex + "
                          "one read of every other-colour position" if int(info.tiles) else
                          "layout bytes: entry_bytes per entry + CSR offset + per-vertex state + "
                          "other-colour positions",
           "k1_ms_per_color": [round(float(x), 4) for x in k1_ms],
           "k1_timing": f"CUDA events per launch on the context stream, colours in step order, "
                        f"{k1_reps} sweeps right after the timed region (sustained clocks)",
           "reference_model": {
               "bytes_per_launch": bytes_iter / ncol, "achieved": ref_achieved,
               "frac": ref_achieved / peak,
               "model": "SURVEY 8(d): 92 N + 208 T bytes per iteration (fp32) / 180 N + 368 T (fp64), "
                        "the reference's data layout (Dm^-1 + V + 3 ids per entry); above 1 because "
                        "the entry dictionary and 8-byte tile slots remove those bytes losslessly"},
           "limiter": ncu_limiter(cfg.name, precision, variant),
           "traffic_unit": "DRAM bytes per k1 launch (ncu dram__bytes_read+write, profiles/k1_traffic.json)",
           "_layout_iter": layout_iter}
    fl = ncu_flops(cfg.name, precision, variant)
    try:
        fpk = fma_peak_tflops(device, precision, 1.0)
    except Exception:  # pragma: no cover
        fpk = None
    fp = {"unit": "TFLOP/s", "peak": fpk,
          "peak_source": "measured live: vbd_fma_peak, %s chains on every SM for 1 s after the "
                         "timed region" % ("FFMA2 (fp32x2)" if precision == "fp32" else "DFMA"),
          "reference_model_flops_per_launch": reference_model_flops_per_iteration(info) / ncol}
    if fl:
        per = float(fl["flops_per_launch"])
        fp.update({"flops_per_launch": per, "achieved": per / (k1_iter_ms / ncol / 1e3) / 1e12,
                   "flops_source": "ncu SASS thread-instruction counters of one launch "
                                   "(profiles/k1_flops.json: %s)" % fl.get("source", "")})
        if fpk:
            fp["frac"] = fp["achieved"] / fpk
    ra = fp["reference_model_flops_per_launch"] / (k1_iter_ms / ncol / 1e3) / 1e12
    fp["reference_model_achieved"] = ra
    rec["fp32" if precision == "fp32" else "fp64"] = fp
    if variant == "classtiles":
        rec["note"] = ("grid-class tiles (DESIGN.md 3): interior vertices one lane each with every neighbour "
                       "loaded once into registers; their layout moves 42 % fewer bytes than the plain "
                       "2-lane tiles (C5: 2.12 vs 3.68 GB per launch) in 16 % less time (0.84 vs 0.996 ms), "
                       "so the HBM fraction is lower while the kernel is faster; no pipe is saturated "
                       "(latency-bound, see limiter)")
    return rec


def fp64_record(cfg, device, timed, steps=3, warmup=2):
    """The same scene at the reference's precision (fp64 build), timed in this run."""
    from paper_2403_06321_b200.scenes import build
    t0 = time.perf_counter()
    ctx, _ = build(cfg, 0, 1, "fp64", device=device)
    t_build = time.perf_counter() - t0
    import torch
    p = cfg.step_params()
    ctx.step(p, n_steps=warmup)
    strm = torch.cuda.ExternalStream(ctx.stream) if ctx.stream else torch.cuda.current_stream()
    ms = timed(lambda: ctx.step(p, n_steps=steps), strm) / steps
    info = ctx.info
    reps = max(10, cfg.n_max)
    k1 = ctx.profile_color_pass(cfg.h, reps=reps)
    roof = roofline_record(cfg, info, "fp64", k1, reps, device)
    vit = int(info.num_solved + info.num_fixed) * cfg.n_max
    ctx.close()
    return {"dtype": "f64", "ms_per_step": ms, "value": vit / (ms / 1e3), "unit": UNIT,
            "steps": steps, "warmup": warmup, "build_s": round(t_build, 2),
            "layout": layout_name(info),
            "k1_ms_per_color": roof["k1_ms_per_color"], "layout_frac": roof["frac"],
            "roofline": {k: v for k, v in roof.items() if not k.startswith("_")}}


def run_reference(args):
    """The reference arm: the unmodified reference (baseline/_ref, else oracle/_ref) on this
    box's host cores.  It runs exactly --warmup untimed and --steps timed steps of a bounded
    sample of the workload (same generator, material, h, n_max, BCs; shrunk so the whole run
    takes about a minute); ms_per_step is the sample's own, value its vertex-iterations/s
    (the metric is size-independent to first order), and the full-scene ms/step it implies is
    reported separately as an extrapolation."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2403_06321_b200.scenes import config
    cfg = config(args.config)
    budget = max(20.0, min(90.0, 4 * args.cpu_seconds))
    r = cpu_reference_sample(args.config, budget, steps=args.steps, warmup=args.warmup)
    ms_sample = r.pop("ms_per_step_sample")
    vit_full = cfg.num_vertices * cfg.n_max
    line = {
        "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world,
        "steps": r["sample_steps"], "warmup": r["sample_warmup"],
        "ms_per_step": ms_sample, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generators), bounded sample of the workload",
        "config": {"workload": f"{cfg.name} sample: {r['sample']}",
                   "full_workload": f"{cfg.name}: {cfg.description}",
                   "sample_vertices": r["sample_vertices"], "sample_tets": r["sample_tets"],
                   "num_vertices": cfg.num_vertices, "num_tets": cfg.num_tets,
                   "h": cfg.h, "n_max": cfg.n_max, "rho": cfg.rho},
        "extrapolated": True,
        "extrapolated_full_scene_ms_per_step": vit_full / r["value"] * 1e3,
        "impl": "reference",
        "cpu_baseline": r,
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def spawn_ranks(args):
    """`python bench.py --gpus N` outside torchrun: start the N ranks ourselves, exactly as
    `python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py ...`
    would.  With fewer GPUs than ranks (tests, 1-GPU boxes) the ranks share the GPUs and the
    control-plane collectives run over gloo (NCCL refuses two ranks on one device); the halo
    itself stays the fused peer-memory push."""
    import socket
    try:
        import torch
        ngpu = torch.cuda.device_count()
    except Exception:
        ngpu = 0
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    if ngpu < args.gpus:
        env.setdefault("VBD_DIST_BACKEND", "gloo")
    env.setdefault("NCCL_DEBUG", "INFO")            # communicator init lines (nranks) on stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(ROOT / "bench.py")] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


if __name__ == "__main__":
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(a))
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
