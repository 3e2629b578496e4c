"""Cross-process slab halo over cudaIpc peer memory (the multi-GPU transport), run as two
processes sharing one GPU: each process owns one slab context, maps its neighbour's position
and flag buffers with cudaIpcOpenMemHandle, and K1 pushes boundary vertices straight into the
neighbour's ghost block.  Positions must equal a single-context run bit for bit."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
BEAM = dict(nx=20, ny=6, nz=5, spacing=0.02, mu=1e6, lam=1e7, kd=1e-6, fix_min_x=True)
G = (0.0, 0.0, -9.8)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2403_06321_b200 as V
        from paper_2403_06321_b200.dist import SlabP2P, slab_cuts
        torch.cuda.set_device(0)
        beam = V.Beam(**BEAM)
        cuts = slab_cuts(beam.nx, world)
        ctx = V.DeviceContext.from_beams([beam], precision="fp32", slab=(cuts[rank], cuts[rank + 1]))
        ex = SlabP2P.distributed(ctx, rank, world, device=0)
        p = ctx.step_params(1 / 120, 5, 0.9, 1e-10, "adaptive", G)
        for k in range(3):
            ex.step(p, k)
        x = ctx.get_state(x=True)["x"]
        plane = beam.ny * beam.nz
        lo = max(cuts[rank] - 1, 0)
        own = x[(cuts[rank] - lo) * plane:(cuts[rank + 1] - lo) * plane]
        q.put((rank, cuts[rank] * plane, own))
        dist.barrier()
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, -1, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_process_ipc_slabs_bitwise():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import torch.multiprocessing as mp
    import paper_2403_06321_b200 as V
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _port()
    procs = [ctxm.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for r, off, x in got:
        assert off >= 0, x
    full = V.DeviceContext.from_beams([V.Beam(**BEAM)], precision="fp32")
    p = full.step_params(1 / 120, 5, 0.9, 1e-10, "adaptive", G)
    for _ in range(3):
        full.step(p)
    xf = full.get_state(x=True)["x"]
    for r, off, x in got:
        assert np.array_equal(x, xf[off:off + len(x)]), r
