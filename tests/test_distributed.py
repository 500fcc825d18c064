"""Slab-decomposed multi-rank orchestration (distributed.py).

CPU: world_size-2 gloo process group running the real orchestration
(partitions, all-to-all split sizes, blocked receive tables, status
reductions) with a numpy restatement of the two device passes.
GPU: the same orchestration emulated in one process on one GPU (ranks run
sequentially, the all-to-all is a device concatenation), which exercises the
device kernels on the blocked layout; results must be bit-identical to the
single-GPU solve.
"""

import os
import socket

import numpy as np
import pytest

from oracle import bhcp_oracle as O
from paper_2107_06381_b200 import distributed as D
from paper_2107_06381_b200 import workloads


def test_partition_balanced_and_uneven():
    assert D.partition(10, 4) == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert D.partition(3, 8)[-1] == (3, 3)
    for total, parts in [(511, 2), (511, 8), (513, 8), (1023, 8), (255, 3)]:
        p = D.partition(total, parts)
        sizes = [b - a for a, b in p]
        assert sum(sizes) == total and max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("dim,m,n,world", [(2, 7, 9, 2), (2, 5, 6, 3), (3, 4, 5, 2), (2, 3, 4, 4)])
def test_layout_tables_address_every_line_once(dim, m, n, world):
    L = D.SlabLayout(dim, m, n, world)
    tb = D.TB
    for r in range(world):
        koff = L.block_tables(r)
        total = sum(L.recv_splits(r))
        seen = np.zeros(total, dtype=int)
        for t in range(L.levels(r)):
            for k1 in range(m):
                for rest in range(m ** (dim - 1)):
                    seen[koff[k1] + ((t // tb) * m ** (dim - 1) + rest) * tb + t % tb] += 1
        assert seen.sum() == L.levels(r) * m**dim
        assert total == 0 or seen.max() == 1
    assert sum(L.levels(r) for r in range(world)) == n
    assert all(c % tb == 0 or c == n for c, _ in L.lev)


@pytest.mark.parametrize("dim,m,n,world", [(2, 7, 9, 2), (2, 5, 30, 3), (3, 4, 17, 4)])
def test_peer_offsets_match_all_to_all_placement(dim, m, n, world):
    """Pass A stores of the peer transport land exactly where all_to_all_single
    would put each sender's chunk."""
    L = D.SlabLayout(dim, m, n, world)
    for q in range(world):
        recv = L.recv_splits(q)
        starts = np.concatenate([[0], np.cumsum(recv)[:-1]]).astype(int)
        for p in range(world):
            assert D.peer_offsets(L, p)[q] == starts[p]
            assert L.send_splits(p)[q] == recv[p]


def test_transport_names():
    with pytest.raises(ValueError):
        D.make_transport("shmem", D.SlabLayout(2, 5, 9, 2), 0, None)
    assert D.make_transport("nccl", D.SlabLayout(2, 5, 9, 2), 0, None) is None


def test_layout_rejects_1d():
    with pytest.raises(ValueError):
        D.SlabLayout(1, 255, 257, 2)


class NumpyOps:
    """numpy restatement of the device passes (test-only injection)."""

    def __init__(self, kind, alpha, w):
        self.args = (kind, alpha, w.dim, w.length, w.num_cells, w.horizon, w.num_steps, w.g_delta)
        self.dim, self.m = w.dim, w.num_cells - 1
        self.sums = (0.0, 0.0)

    def modes(self, layout, rank):
        """W_r blocked per destination level slab (bhcp_pint_modes layout)."""
        import torch
        kb, ke = layout.mode_range(rank)
        W, sre, sim = O.fused_pass_a(*self.args, kb, ke)   # (n, S) level-major
        self.sums = (sre, sim)
        tb, plane = D.TB, layout.plane
        nk1 = (ke - kb) // plane
        chunks = []
        for c, d in layout.lev:
            nt = (d - c + tb - 1) // tb
            blk = np.zeros((nk1, nt, plane, tb))
            for t in range(c, d):
                blk[:, (t - c) // tb, :, (t - c) % tb] = W[t].reshape(nk1, plane)
            chunks.append(blk.ravel())
        return torch.from_numpy(np.concatenate(chunks))

    def tables(self, layout, rank):
        return layout.block_tables(rank)

    def levels_blocked(self, recv, koff, L):
        import torch
        recv = recv.numpy()
        m, d, tb = self.m, self.dim, D.TB
        plane = m ** (d - 1)
        F = np.zeros((L, m**d))
        for t in range(L):
            for k1 in range(m):
                s = koff[k1] + (t // tb) * plane * tb + t % tb
                F[t, k1 * plane:(k1 + 1) * plane] = recv[s:s + plane * tb:tb]
        return torch.from_numpy(O.fused_pass_b(F, d, m))


def _worker(rank, world, port, kind, dim, cells, steps, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = workloads.make_small(dim, cells, steps, seed=11)
    layout = D.SlabLayout(dim, cells - 1, steps + 1, world)
    ops = NumpyOps(kind, 1e-2, w)
    comm = D.TorchComm(torch.device("cpu"))
    y, (c, d) = D.sharded_solve(ops, comm, layout, rank)
    sre, sim, bad = D.reduce_status(comm, ops.sums[0], ops.sums[1], -1)
    q.put((rank, c, d, y.numpy(), sre, sim, bad))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,dim,cells,steps", [("pint-mqbvm", 2, 8, 8), ("pint-qbvm", 2, 9, 6),
                                                   ("pint-mqbvm", 3, 5, 5)])
def test_gloo_world2_matches_oracle(kind, dim, cells, steps):
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, dim, cells, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    outs.sort(key=lambda o: o[0])
    y = np.concatenate([o[3] for o in outs], axis=0)
    assert outs[0][1] == 0 and outs[-1][2] == steps + 1
    w = workloads.make_small(dim, cells, steps, seed=11)
    ref = O.spectral_oracle(kind, 1e-2, dim, w.length, cells, w.horizon, steps, w.g_delta)
    assert np.linalg.norm(y - ref) / np.linalg.norm(ref) <= 1e-11
    # both ranks agree on the reduced residue accumulators and no singular column
    assert outs[0][4] == outs[1][4] and outs[0][5] == outs[1][5]
    assert outs[0][6] == -1 and outs[1][6] == -1
    assert np.sqrt(outs[0][5]) <= 1e-8 * np.sqrt(outs[0][4] + outs[0][5])


# ---------------------------------------------------------------- GPU emulation

def emulate_peer(system, world):
    """Peer transport emulated on one GPU: one receive buffer per rank; each
    rank's pass A stores straight into all of them (bhcp_pint_modes_to)."""
    import ctypes

    import torch

    import paper_2107_06381_b200 as B
    from paper_2107_06381_b200 import plans

    grid, tg = system.grid, system.timegrid
    layout = D.SlabLayout(grid.dim, grid.num_cells - 1, tg.n_levels, world)
    plan = B.PintPlan(grid, tg.n_levels, tg.tau, system.omega)
    ops = D.DeviceOps(plan, plans.to_device(system.data, torch.float64),
                      system.method.condition_divisor(tg.tau))
    recv = [torch.full((max(1, sum(layout.recv_splits(q))),), float("nan"), dtype=torch.float64, device="cuda")
            for q in range(world)]
    for p in range(world):
        offs = D.peer_offsets(layout, p)
        dst = (ctypes.c_void_p * world)(*[recv[q].data_ptr() + 8 * offs[q] for q in range(world)])
        ops.modes_to(layout, p, dst)
    ys = [ops.levels_blocked(recv[q], ops.tables(layout, q), layout.levels(q)).clone() for q in range(world)]
    return torch.cat(ys).cpu().numpy()


def emulate_peer_sym(system, world):
    """Symmetric pass A split over emulated ranks (bhcp_pint_modes_sym_to):
    every rank computes a share of the mirror-pair tiles and stores both modes
    into all receivers through their block tables."""
    import ctypes

    import torch

    import paper_2107_06381_b200 as B
    from paper_2107_06381_b200 import plans

    grid, tg = system.grid, system.timegrid
    layout = D.SlabLayout(grid.dim, grid.num_cells - 1, tg.n_levels, world)
    plan = B.PintPlan(grid, tg.n_levels, tg.tau, system.omega)
    ops = D.DeviceOps(plan, plans.to_device(system.data, torch.float64),
                      system.method.condition_divisor(tg.tau))
    if ops.sym_tiles() == 0:
        return None
    recv = [torch.full((max(1, sum(layout.recv_splits(q))),), float("nan"), dtype=torch.float64, device="cuda")
            for q in range(world)]
    bases = (ctypes.c_void_p * world)(*[recv[q].data_ptr() for q in range(world)])
    for p in range(world):
        ops.modes_sym_to(layout, p, bases)
    ys = [ops.levels_blocked(recv[q], ops.tables(layout, q), layout.levels(q)).clone() for q in range(world)]
    return torch.cat(ys).cpu().numpy()


def emulate(system, world):
    import torch

    import paper_2107_06381_b200 as B
    from paper_2107_06381_b200 import plans

    grid, tg = system.grid, system.timegrid
    layout = D.SlabLayout(grid.dim, grid.num_cells - 1, tg.n_levels, world)
    plan = B.PintPlan(grid, tg.n_levels, tg.tau, system.omega)
    ops = D.DeviceOps(plan, plans.to_device(system.data, torch.float64),
                      system.method.condition_divisor(tg.tau))
    Ws = [ops.modes(layout, r).clone() for r in range(world)]
    ys = []
    for q in range(world):
        chunks = []
        for r in range(world):
            off = sum(layout.send_splits(r)[:q])
            chunks.append(Ws[r][off:off + layout.send_splits(r)[q]])
        recv = torch.cat(chunks)
        koff = ops.tables(layout, q)
        ys.append(ops.levels_blocked(recv, koff, layout.levels(q)).clone())
    return torch.cat(ys).cpu().numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("dim,cells,steps,world", [(2, 16, 12, 2), (2, 20, 9, 3), (3, 8, 6, 2), (3, 9, 7, 4),
                                                   (2, 12, 256, 2), (3, 7, 256, 3), (2, 10, 1024, 2),
                                                   (2, 20, 512, 3), (2, 6, 4096, 2), (3, 6, 1024, 2),
                                                   (2, 512, 512, 8), (2, 1024, 19, 3)])
def test_emulated_ranks_bitwise_equal_single_gpu(dim, cells, steps, world):
    """(2, 1024, 19, 3): the c3 grid, whose receivers run the level-group kernel
    (k_dst_lvl4) on their level slabs (3 ranks: 8 + 8 + 4 levels)."""
    import paper_2107_06381_b200 as B

    w = workloads.make_small(dim, cells, steps, seed=3) if cells != 512 else workloads.make("c2")
    grid = B.build_grid(dim, w.length, cells)
    tg = B.TimeGrid(w.horizon, steps)
    system = B.assemble(B.MethodKind.PINT_MQBVM, 1e-2, grid, tg, w.g_delta)
    single = B.solve_pint(system).trajectory
    multi = emulate(system, world)
    assert np.array_equal(single, multi)
    assert np.array_equal(single, emulate_peer(system, world))
    sym = emulate_peer_sym(system, world)
    if sym is not None:
        assert np.array_equal(single, sym)
