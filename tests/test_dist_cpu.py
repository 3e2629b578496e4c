"""Multi-rank host logic on CPU (gloo, world_size 2): the slab halo-exchange
orchestration of paper_2403_06321_b200.dist.SlabExchange, driven over real
torch.distributed point-to-point messages, with each rank's slab solved by the
oracle.  The sharded trajectory must equal the single-domain oracle trajectory
bit for bit (the same property the GPU test checks for the device contexts)."""

import os
import socket

import numpy as np
import pytest

NX, NY, NZ, SP = 14, 4, 5, 0.03
MAT = (1e6, 1e7, 1e-6)
G = (0.0, 0.0, -9.8)
H = 1.0 / 120.0


class OracleSlab:
    """CPU stand-in for a slab DeviceContext (same interface as SlabExchange uses)."""

    class _Info:
        precision = 1

    def __init__(self, O, lo, hi):
        self.O = O
        full = O.generate_beam(NX, NY, NZ, SP)
        fixed = np.flatnonzero(full.rest_positions[:, 0] < 1e-9)
        fs = O.build_system([(full, MAT)], fixed)  # global colouring
        plane = NY * NZ
        a0, a1 = max(lo - 1, 0), min(hi, NX - 1)
        self.vbase = a0 * plane
        n = (a1 - a0 + 1) * plane
        cells = (NY - 1) * (NZ - 1) * 5
        tsl = slice(a0 * cells, a1 * cells)
        tets = fs.tets[tsl] - self.vbase
        t_off, t_id, t_slot = O.incidence_from_elements(tets, n)
        vs = slice(self.vbase, self.vbase + n)
        self.sys = O.System(n, fs.masses[vs].copy(), fs.rest_positions[vs].copy(), tets,
                            fs.tet_w[tsl], fs.tet_vol[tsl], fs.tet_mu[tsl], fs.tet_lam[tsl],
                            fs.tet_kd[tsl], t_off, t_id, t_slot, fs.color_of[vs].copy(),
                            np.zeros(1, np.int64), np.zeros(0, np.int64), fs.kind[vs].copy())
        ax = a0 + np.arange(n) // plane
        owned = (ax >= lo) & (ax < hi)
        col = self.sys.color_of
        self.num_colors = int(fs.color_of.max()) + 1
        self.groups = [np.flatnonzero(owned & (col == c)) for c in range(self.num_colors)]
        self.owned = np.flatnonzero(owned)
        side_planes = {0: (lo, lo - 1, lo > 0), 1: (hi - 1, hi, hi < NX)}
        self.send, self.recv = {}, {}
        for side, (ps, pr, exists) in side_planes.items():
            for c in range(self.num_colors):
                s = np.flatnonzero((ax == ps) & (col == c)) if exists else np.zeros(0, np.int64)
                r = np.flatnonzero((ax == pr) & (col == c)) if exists else np.zeros(0, np.int64)
                self.send[side, c], self.recv[side, c] = s, r
        self.info = self._Info()
        self.st = O.make_state(self.sys)

    # --- interface used by SlabExchange ---
    def set_stream(self, handle):
        pass

    def halo_count(self, side, color):
        return len(self.send[side, color]), len(self.recv[side, color])

    @staticmethod
    def _view(ptr, n):
        import ctypes
        return np.ctypeslib.as_array((ctypes.c_double * (4 * n)).from_address(ptr)).reshape(n, 4)

    def halo_pack(self, side, color, ptr):
        ids = self.send[side, color]
        buf = self._view(ptr, len(ids))
        buf[:, :3] = self.st.x[ids]
        buf[:, 3] = 0.0

    def halo_unpack(self, side, color, ptr):
        ids = self.recv[side, color]
        self.st.x[ids] = self._view(ptr, len(ids))[:, :3]

    def step_begin(self, p):
        O, st = self.O, self.st
        self.p = p
        st.y = O.inertia_target(st.x_t, st.v_t, np.asarray(p.a_ext), p.h)
        O.initialize(self.sys, st, p.h, np.asarray(p.a_ext), "adaptive")
        st.x_prev1, st.x_pp = st.x.copy(), None

    def step_color(self, color, n):
        self.O.color_pass(self.sys, self.st.x, self.st.x_t, self.st.y, self.p.h, self.groups[color])

    def step_iter_end(self, n):
        st = self.st
        w = self.O.chebyshev_omega(self.p.rho, n)
        if w != 1.0 and st.x_pp is not None:
            st.x[...] = w * (st.x - st.x_pp) + st.x_pp
        st.x_pp, st.x_prev1 = st.x_prev1, st.x.copy()

    def step_end(self, step_index=0):
        st = self.st
        v = (st.x - st.x_t) / self.p.h
        st.v_prev, st.v_t, st.x_t = st.v_t, v, st.x.copy()


class _P:
    def __init__(self, h, n_max, rho, a_ext):
        self.h, self.n_max, self.rho, self.a_ext = h, n_max, rho, a_ext


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2403_06321_b200.dist import SlabExchange, slab_cuts
        cuts = slab_cuts(NX, world)
        ctx = OracleSlab(O, cuts[rank], cuts[rank + 1])
        ex = SlabExchange.distributed(ctx, rank, world, device="cpu")
        p = _P(H, 6, 0.9, G)
        for k in range(3):
            ex.step(p, k)
        q.put((rank, ctx.vbase + ctx.owned, ctx.st.x[ctx.owned]))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 3])
def test_slab_exchange_gloo_bitwise_equals_single_domain(O, world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = O.generate_beam(NX, NY, NZ, SP)
    fixed = np.flatnonzero(full.rest_positions[:, 0] < 1e-9)
    fs = O.build_system([(full, MAT)], fixed)
    st = O.make_state(fs)
    for _ in range(3):
        O.step(fs, st, H, 6, 0.9, G)
    seen = np.zeros(fs.num_vertices, bool)
    for rank, ids, x in got:
        assert np.array_equal(x, st.x[ids]), rank
        seen[ids] = True
    assert seen.all()


def test_partition_helpers():
    from paper_2403_06321_b200.dist import object_shard, slab_cuts
    assert slab_cuts(364, 8)[0] == 0 and slab_cuts(364, 8)[-1] == 364
    cuts = slab_cuts(364, 8)
    assert max(np.diff(cuts)) - min(np.diff(cuts)) <= 1
    spans = [object_shard(10368, r, 8) for r in range(8)]
    assert spans[0][0] == 0 and spans[-1][1] == 10368
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert {hi - lo for lo, hi in spans} == {1296}
    with pytest.raises(ValueError):
        slab_cuts(4, 5)
    # the fixed x = 0 face of C5 is not work: the other 363 planes are split evenly
    fc = slab_cuts(364, 8, 1, 0)
    assert fc[0] == 0 and fc[-1] == 364
    solved = np.diff(fc) - np.array([1] + [0] * 7)
    assert max(solved) - min(solved) <= 1 and solved.sum() == 363
