"""The c5 regularisation sweep: host orchestration (CPU, gloo world 2) and the
device sweep against the closed-form oracle's error-vs-alpha curve (B200).

Bar (BASELINE c5 / north star): e_h = l2_error(y[0], z0) of every (kind, alpha)
agrees with the oracle's to 3 significant digits (relative 5e-4 here).
"""

import os
import socket

import numpy as np
import pytest

from oracle import bhcp_oracle as O
from paper_2107_06381_b200 import sweep, workloads


def fake_solve(kind, alpha):
    # deterministic stand-in for a device solve: (e_h, ms)
    return (1.0 if kind == "pint-qbvm" else 2.0) * np.log10(alpha) ** 2, 0.5


def test_assign_covers_every_pair_once():
    for n in (1, 5, 128):
        for world in (1, 2, 3, 8):
            got = sorted(i for r in range(world) for i in sweep.assign(n, r, world))
            assert got == list(range(n))
    with pytest.raises(ValueError):
        sweep.assign(4, 2, 2)


def test_run_pairs_world1_order_and_curve():
    alphas = list(np.logspace(-6, -1, 7))
    pairs = [(k, a) for k in ("pint-qbvm", "pint-mqbvm") for a in alphas]
    res = sweep.run_pairs(pairs, fake_solve)
    assert [(p.kind, p.alpha) for p in res.points] == [(k, float(a)) for k, a in pairs]
    a, e = res.curve("pint-mqbvm")
    assert np.allclose(a, alphas) and np.allclose(e, 2.0 * np.log10(alphas) ** 2)
    assert res.best("pint-qbvm").alpha == pytest.approx(1e-1)


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    alphas = list(np.logspace(-6, -1, 9))
    pairs = [(k, a) for k in ("pint-qbvm", "pint-mqbvm") for a in alphas]
    res = sweep.run_pairs(pairs, fake_solve, rank, world)
    q.put((rank, [(p.kind, p.alpha, p.e_h, p.rank) for p in res.points], res.wall_s))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_gathers_all_pairs():
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=120) for _ in range(2)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank holds the full 18-point curve, in pair order, computed half by each rank
    assert outs[0][1] == outs[1][1]
    pts = outs[0][1]
    assert len(pts) == 18
    assert sorted({r for *_, r in pts}) == [0, 1]
    assert [p[3] for p in pts] == [i % 2 for i in range(18)]
    assert outs[0][2] == outs[1][2]   # wall time: max over ranks


@pytest.mark.gpu
@pytest.mark.parametrize("config,idx", [("small", None), ("c5", [0, 21, 42, 63])])
def test_device_sweep_matches_oracle_curve(config, idx):
    import paper_2107_06381_b200 as B

    if config == "small":
        w = workloads.make_small(1, 64, 64, seed=9, length=np.pi, horizon=1.0, delta=1e-3)
        alphas = list(np.logspace(-6, -1, 16))
        kinds = ("pint-qbvm", "pint-mqbvm")
    else:
        w = workloads.make("c5")
        alphas = [w.alphas[i] for i in idx]
        kinds = w.kinds
    grid = B.build_grid(w.dim, w.length, w.num_cells)
    tg = B.TimeGrid(w.horizon, w.num_steps)
    res = sweep.alpha_sweep(grid, tg, w.g_delta, w.z0, kinds, alphas)
    assert len(res.points) == len(kinds) * len(alphas)
    for p in res.points:
        ref = O.spectral_oracle(p.kind, p.alpha, w.dim, w.length, w.num_cells, w.horizon, w.num_steps,
                                w.g_delta, levels=np.array([0]))
        e_ref = workloads.l2_error(ref[0], w.z0, grid.h, w.dim)
        assert abs(p.e_h - e_ref) <= 5e-4 * e_ref, (p.kind, p.alpha, p.e_h, e_ref)
        assert p.ms > 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("cells,steps,nalpha", [(64, 4096, 18), (48, 64, 3)])
def test_batched_solves_bitwise_equal_single(cells, steps, nalpha):
    """bhcp_pint_solve_batch (pint.PintBatch): every trajectory bitwise the single
    fused solve of its (kind, alpha); residue norms per solve. n = 4097 runs the
    batched prime-factor pass A (36 solves: two launches of <= 32 pairs), n = 65
    the per-pair fallback."""
    import torch

    import paper_2107_06381_b200 as B
    from paper_2107_06381_b200 import pint

    w = workloads.make_small(1, cells, steps, seed=4, length=np.pi, horizon=1.0, delta=1e-3)
    grid = B.build_grid(1, w.length, w.num_cells)
    tg = B.TimeGrid(w.horizon, w.num_steps)
    alphas = list(np.logspace(-6, -1, nalpha))
    systems = [B.assemble(B.MethodKind(k), a, grid, tg, w.g_delta) for k in ("pint-qbvm", "pint-mqbvm") for a in alphas]
    plans_ = [pint.PintPlan(grid, tg.n_levels, tg.tau, s.omega) for s in systems]
    divs = [s.method.condition_divisor(tg.tau) for s in systems]
    g = torch.from_numpy(w.g_delta).cuda()
    batch = pint.PintBatch(plans_)
    yb = batch.solve_device(g, divs).cpu().numpy()
    for i, (p, d) in enumerate(zip(plans_, divs)):
        y1 = p.solve_device(g, d).cpu().numpy()
        st1 = p.check_status()
        stb = batch.check(i)
        assert np.array_equal(yb[i], y1), f"solve {i}"
        assert abs(stb.residue - st1.residue) <= 1e-9 * st1.residue + 1e-300
        assert abs(stb.norm - st1.norm) <= 1e-12 * st1.norm
