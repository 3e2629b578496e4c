"""Multi-GPU execution.

* Many-object scenes shard by object (``object_shard``): each rank owns a
  contiguous range of bodies in its own DeviceContext; there is no data-path
  communication, and because the greedy colouring of disjoint bodies restricted
  to one body equals that body's own colouring, results are bitwise identical to
  one GPU.
* One large mesh is decomposed into x-slabs (``slab_cuts``); each rank holds its
  owned vertex planes plus one ghost plane per neighbour.  After every colour
  pass the boundary vertices of that colour are exchanged point-to-point
  (``SlabExchange``: NCCL send/recv through torch.distributed on the context's
  stream).  K2/K3/K4 are elementwise, so ghosts are advanced locally and only the
  per-colour halo travels; the result is bitwise identical to one GPU.

One process per GPU; ranks/world from torch.distributed (``torchrun``).
"""

from __future__ import annotations

import numpy as np


def slab_cuts(nx: int, world: int, fixed_lo: int = 0, fixed_hi: int = 0):
    """Owned vertex-plane ranges [cuts[r], cuts[r+1]) along x, balanced by SOLVED planes: the
    fixed_lo first / fixed_hi last planes (a clamped face: never solved, only copied by K2 /
    K4) ride on the first / last rank instead of counting as a plane of work."""
    if world < 1 or world > nx - fixed_lo - fixed_hi:
        raise ValueError("need 1 <= world <= solved planes")
    work = nx - fixed_lo - fixed_hi
    cuts = [fixed_lo + int(round(r * work / world)) for r in range(world + 1)]
    cuts[0], cuts[-1] = 0, nx
    return cuts


def object_shard(num_objects: int, rank: int, world: int):
    """Contiguous object range [lo, hi) of rank r (balanced by count)."""
    lo = num_objects * rank // world
    hi = num_objects * (rank + 1) // world
    return lo, hi


def _halo_dtype(ctx):
    import torch
    return torch.float64 if int(ctx.info.precision) == 1 else torch.float32


class SlabExchange:
    """Drives one step of a slab-decomposed scene with a per-colour halo exchange.

    ``ctxs`` are the DeviceContexts this process drives (one per rank normally;
    several when emulating ranks on one GPU with ``local``).  ``peers[i][side]``
    is the neighbour of ctxs[i] on side 0 (towards lower x) / 1 (higher x): either
    ("local", j) for another context in this process or ("rank", r) for a remote
    torch.distributed rank, or None.
    """

    def __init__(self, ctxs, peers, device=None):
        import contextlib

        import torch
        self.ctxs = list(ctxs)
        self.peers = peers
        self.torch = torch
        dev = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        if dev.type == "cuda":
            self.stream = torch.cuda.Stream(device=dev)
            for c in self.ctxs:
                c.set_stream(self.stream.cuda_stream)
            self._on_stream = lambda: torch.cuda.stream(self.stream)
        else:  # CPU contexts (host-logic tests with gloo)
            self.stream = None
            self._on_stream = contextlib.nullcontext
        ncol = max(c.num_colors for c in self.ctxs)
        self.ncol = ncol
        self.bufs = []
        for c in self.ctxs:
            per = {}
            for side in (0, 1):
                counts = [c.halo_count(side, k) for k in range(c.num_colors)]
                ns = max([a for a, _ in counts] + [0])
                nr = max([b for _, b in counts] + [0])
                dt = _halo_dtype(c)
                per[side] = (torch.empty((max(ns, 1), 4), dtype=dt, device=dev),
                             torch.empty((max(nr, 1), 4), dtype=dt, device=dev))
            self.bufs.append(per)

    @classmethod
    def local(cls, ctxs, device=None):
        """All slabs driven by this process on one device (ordered by x)."""
        peers = [{0: ("local", i - 1) if i > 0 else None,
                  1: ("local", i + 1) if i + 1 < len(ctxs) else None} for i in range(len(ctxs))]
        return cls(ctxs, peers, device)

    @classmethod
    def distributed(cls, ctx, rank, world, device=None):
        peers = [{0: ("rank", rank - 1) if rank > 0 else None,
                  1: ("rank", rank + 1) if rank + 1 < world else None}]
        return cls([ctx], peers, device)

    def _stage_host(self):
        import torch.distributed as dist
        return self.stream is not None and dist.get_backend() == "gloo"

    def _exchange(self, color):
        torch = self.torch
        import torch.distributed as dist
        ops, unpack = [], []
        # pack every outgoing side first (all on self.stream)
        for i, c in enumerate(self.ctxs):
            for side in (0, 1):
                peer = self.peers[i][side]
                if peer is None or color >= c.num_colors:
                    continue
                ns, nr = c.halo_count(side, color)
                sbuf, rbuf = self.bufs[i][side]
                if ns:
                    c.halo_pack(side, color, sbuf.data_ptr())
                kind, j = peer
                if kind == "local":
                    # the neighbour's receive side faces us: copy our send buffer into it
                    other_side = 1 - side
                    _, orb = self.bufs[j][other_side]
                    if ns:
                        with self._on_stream():
                            orb[:ns].copy_(sbuf[:ns])
                    unpack.append((j, other_side, ns))
                else:
                    if ns:
                        ops.append(dist.P2POp(dist.isend, sbuf[:ns], j))
                    if nr:
                        ops.append(dist.P2POp(dist.irecv, rbuf[:nr], j))
                    unpack.append((i, side, nr))
        if ops and self._stage_host():
            # gloo cannot send device tensors: stage through host memory (used only to run
            # several ranks on one GPU for testing; NCCL is the production transport)
            torch.cuda.current_stream().wait_stream(self.stream)
            self.stream.synchronize()
            host_ops, back = [], []
            for op in ops:
                h = op.tensor.cpu()
                host_ops.append(dist.P2POp(op.op, h, op.peer))
                if op.op is dist.irecv:
                    back.append((op.tensor, h))
            for r in dist.batch_isend_irecv(host_ops):
                r.wait()
            with self._on_stream():
                for dst, h in back:
                    dst.copy_(h)
        elif ops:
            with self._on_stream():
                for r in dist.batch_isend_irecv(ops):
                    r.wait()
        for i, side, n in unpack:
            if n:
                self.ctxs[i].halo_unpack(side, color, self.bufs[i][side][1].data_ptr())

    def step(self, params, step_index=0):
        n_max = int(params.n_max)
        for c in self.ctxs:
            c.step_begin(params)
        for n in range(1, n_max + 1):
            for color in range(self.ncol):
                for c in self.ctxs:
                    if color < c.num_colors:
                        c.step_color(color, n)
                self._exchange(color)
            for c in self.ctxs:
                c.step_iter_end(n)
        res = [c.step_end(step_index) for c in self.ctxs]
        return res


class SlabP2P:
    """Slab halo over peer memory, the B200-native transport.

    K1 stores every boundary vertex of the colour it just solved directly into the
    neighbour's ghost slot (NVLink stores through a cudaIpc mapping), and each phase of the
    step (K2, every colour pass, K3, K4) starts only after both neighbours finished the
    previous phase, signalled with release/acquire flags in peer memory.  A whole step is one
    CUDA graph per rank: no NCCL call and no host round trip per colour.
    """

    def __init__(self, ctxs):
        self.ctxs = list(ctxs)

    @classmethod
    def local(cls, ctxs):
        """Several slabs of one process (same device, separate streams): direct pointers."""
        ptrs = [c.p2p_local_ptrs() for c in ctxs]
        for i, c in enumerate(ctxs):
            if i > 0:
                b, n, _ = ctxs[i - 1].ghost_blocks(1)
                c.p2p_connect(0, ptrs[i - 1][0], ptrs[i - 1][1], b, n)
            if i + 1 < len(ctxs):
                b, n, _ = ctxs[i + 1].ghost_blocks(0)
                c.p2p_connect(1, ptrs[i + 1][0], ptrs[i + 1][1], b, n)
        return cls(ctxs)

    @classmethod
    def distributed(cls, ctx, rank, world, device):
        """One slab per process; peers mapped with cudaIpcOpenMemHandle (NVLink)."""
        import torch.distributed as dist
        pos_h, fl_h = ctx.p2p_export()
        mine = {"pos": pos_h, "flags": fl_h,
                "ghost0": [a.tolist() for a in ctx.ghost_blocks(0)[:2]],
                "ghost1": [a.tolist() for a in ctx.ghost_blocks(1)[:2]]}
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        opened = []
        for side, peer in ((0, rank - 1), (1, rank + 1)):
            if 0 <= peer < world:
                p = allv[peer]
                pos = ctx.ipc_open(device, p["pos"])
                fl = ctx.ipc_open(device, p["flags"])
                opened += [pos, fl]
                facing = p["ghost1"] if side == 0 else p["ghost0"]
                ctx.p2p_connect(side, pos, fl, facing[0], facing[1])
        dist.barrier()
        obj = cls([ctx])
        obj._opened = opened
        return obj

    def step(self, params, step_index=0):
        for c in self.ctxs:
            c.step_p2p_launch(params)
        return [c.step_p2p_finish(step_index) for c in self.ctxs]
