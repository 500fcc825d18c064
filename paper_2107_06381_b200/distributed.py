"""Slab-decomposed multi-GPU solve (one process per GPU, NCCL over NVLink).

The fused dataflow of pint.py has two halves with different natural
partitions:

  pass A  (bhcp_pint_modes)   independent per spatial mode k, all time levels
  pass B  (bhcp_pint_levels)  independent per time level t, all spatial modes

so the P ranks split the outermost mode axis k1 into slabs for pass A, then
exchange W with ONE all-to-all (the space<->time transpose of SURVEY 5, but
on real float64 W: 8 B per DOF instead of 16 B for complex S2), and split the
time levels into slabs for pass B. The inverse DST reads the all-to-all
receive buffer in place through a per-k1 address table (no unpack pass).
The residue norms are summed and the first singular column is min-reduced
across ranks, so every rank raises the same error as the 1-GPU solve.
Neither N_t nor M-1 needs to be divisible by P: slabs are uneven with
explicit split sizes.

``ops`` (the per-rank compute) and ``comm`` (the collectives) are injected:
the product path uses ``DeviceOps`` + ``TorchComm`` (NCCL); the CPU tests run
the same orchestration with a numpy restatement of the two passes over gloo.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List, Tuple

import numpy as np


TB = 8  # levels per W tile (fastk::kTBL)


def partition(total: int, parts: int) -> List[Tuple[int, int]]:
    """Balanced contiguous split of range(total) into `parts` (sizes differ by <= 1)."""
    base, extra = divmod(total, parts)
    out, start = [], 0
    for r in range(parts):
        size = base + (1 if r < extra else 0)
        out.append((start, start + size))
        start += size
    return out


@dataclass
class SlabLayout:
    dim: int
    m: int           # interior points per axis
    n: int           # time levels
    world: int

    def __post_init__(self):
        if self.dim < 2:
            raise ValueError("slab decomposition needs dim >= 2 (1D runs stay on one GPU)")
        self.k1 = partition(self.m, self.world)
        # level slabs start at multiples of 8: W is stored in tiles of 8
        # levels and the level pass packs levels (2u, 2u+1) into one complex
        # FFT, so no tile or pair straddles two ranks and every rank count
        # gives the single-GPU result bit for bit
        tiles = partition((self.n + TB - 1) // TB, self.world)
        self.lev = [(min(TB * a, self.n), min(TB * b, self.n)) for a, b in tiles]
        self.plane = self.m ** (self.dim - 1)   # modes per k1 value

    @property
    def n_space(self) -> int:
        return self.m ** self.dim

    def mode_range(self, r: int) -> Tuple[int, int]:
        a, b = self.k1[r]
        return a * self.plane, b * self.plane

    def slab_modes(self, r: int) -> int:
        a, b = self.k1[r]
        return (b - a) * self.plane

    def levels(self, r: int) -> int:
        c, d = self.lev[r]
        return d - c

    def tiles(self, r: int) -> int:
        return (self.levels(r) + TB - 1) // TB

    def send_splits(self, r: int) -> List[int]:
        """Rank r sends the blocked chunk of level slab q of its W_r to rank q."""
        return [self.tiles(q) * TB * self.slab_modes(r) for q in range(self.world)]

    def recv_splits(self, r: int) -> List[int]:
        return [self.tiles(r) * TB * self.slab_modes(p) for p in range(self.world)]

    def slab_bounds(self) -> np.ndarray:
        """Level-slab boundaries (the W chunking of bhcp_pint_modes)."""
        return np.array([c for c, _ in self.lev] + [self.n], dtype=np.int64)

    def block_tables(self, r: int) -> np.ndarray:
        """koff of bhcp_pint_levels_blocked for receiver r: the receive buffer
        holds, for every sender p, its blocked chunk (S_p modes x NT_r tiles of
        8 levels); mode (k1, rest) of local level t is at
        koff[k1] + ((t // 8) * plane + rest) * 8 + t % 8."""
        nt = self.tiles(r)
        koff = np.empty(self.m, dtype=np.int64)
        offset = 0
        recv = self.recv_splits(r)
        for p in range(self.world):
            a, b = self.k1[p]
            for k1 in range(a, b):
                koff[k1] = offset + (k1 - a) * nt * self.plane * TB
            offset += recv[p]
        return koff


# ---------------------------------------------------------------- orchestration

def sharded_solve(ops, comm, layout: SlabLayout, rank: int, events=None):
    """Run one slab-decomposed solve on this rank; returns (y_local, (c, d)).

    ops.modes(layout, rank)            -> W_r, blocked per destination slab (flat)
    ops.levels_blocked(recv, koff, L)  -> y (L, n_space)
    comm.all_to_all(send, send_splits, recv_splits) -> recv buffer (flat)
    """
    if events:
        events[0].record()
    W = ops.modes(layout, rank)
    if events:
        events[1].record()
    recv = comm.all_to_all(W.reshape(-1), layout.send_splits(rank), layout.recv_splits(rank))
    if events:
        events[2].record()
    koff = ops.tables(layout, rank)
    y = ops.levels_blocked(recv, koff, layout.levels(rank))
    if events:
        events[3].record()
    return y, layout.lev[rank]


def peer_offsets(layout: SlabLayout, rank: int) -> List[int]:
    """Element offset of `rank`'s chunk inside every destination q's receive
    buffer -- exactly where all_to_all_single places it (senders in rank order)."""
    return [int(sum(layout.recv_splits(q)[:rank])) for q in range(layout.world)]


def sharded_solve_peer(ops, transport, layout: SlabLayout, rank: int, events=None):
    """The same solve with pass A storing straight into the receivers' buffers
    over NVLink peer memory: no separate all-to-all, the transfer overlaps
    pass A's compute store by store. When the time length has a symmetric
    pass-A kernel, the ranks split its mirror-pair tile list evenly
    (bhcp_pint_modes_sym_to: half the FFT work of a k1-slab split, each pair
    stored into both owners through the receivers' block tables); otherwise
    each rank runs its k1 slab (bhcp_pint_modes_to). Two device barriers:
    receivers are done with the previous solve's buffer; all stores landed."""
    transport.barrier()
    if events:
        events[0].record()
    if ops.sym_tiles() > 0:
        ops.modes_sym_to(layout, rank, transport.bases)
    else:
        ops.modes_to(layout, rank, transport.dst)
    if events:
        events[1].record()
    transport.barrier()
    if events:
        events[2].record()
    koff = ops.tables(layout, rank)
    y = ops.levels_blocked(transport.recv, koff, layout.levels(rank))
    if events:
        events[3].record()
    return y, layout.lev[rank]


class PeerTransport:
    """Receive buffers in symmetric memory (torch.distributed._symmetric_memory,
    CUDA peer mappings over NVLink / NVSwitch): rank p's pass A writes its
    chunk for rank q at q's buffer + peer_offsets(p)[q]."""

    def __init__(self, layout: SlabLayout, rank: int, device, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        group = group or dist.group.WORLD
        try:
            symm_mem.enable_symm_mem_for_group(group.group_name)
        except Exception:  # newer torch enables it on rendezvous
            pass
        size = max(int(sum(layout.recv_splits(q))) for q in range(layout.world))
        self.buf = symm_mem.empty(max(size, 1), dtype=torch.float64, device=device)
        self.hdl = symm_mem.rendezvous(self.buf, group)
        ptrs = list(self.hdl.buffer_ptrs)
        offs = peer_offsets(layout, rank)
        self.dst = (ctypes.c_void_p * layout.world)(*[int(ptrs[q]) + 8 * offs[q] for q in range(layout.world)])
        self.bases = (ctypes.c_void_p * layout.world)(*[int(p) for p in ptrs[: layout.world]])
        self.recv = self.buf[: int(sum(layout.recv_splits(rank)))]

    def barrier(self):
        self.hdl.barrier()


def make_transport(kind: str, layout: SlabLayout, rank: int, device):
    """'peer' (NVLink stores from pass A), 'nccl' (all_to_all_single), or
    'auto' = peer when symmetric memory can be set up, else nccl."""
    if kind not in ("auto", "peer", "nccl"):
        raise ValueError(f"unknown transport {kind!r}")
    if kind == "nccl":
        return None
    try:
        return PeerTransport(layout, rank, device)
    except Exception as e:
        if kind == "peer":
            raise
        # not silent: the sharded bench line reports the transport it used, and the
        # reason the peer (symmetric-memory) path was not available is logged here
        import warnings

        warnings.warn(f"rank {rank}: peer transport unavailable ({type(e).__name__}: {e}); "
                      "falling back to the NCCL all-to-all (set BHCP_TRANSPORT=nccl to select it explicitly)",
                      RuntimeWarning, stacklevel=2)
        return None


def reduce_status(comm, sre: float, sim: float, bad: int) -> Tuple[float, float, int]:
    """Sum the residue accumulators and min-reduce the first singular column."""
    s = comm.all_reduce_sum([sre, sim])
    b = comm.all_reduce_min(bad if bad >= 0 else np.iinfo(np.int64).max)
    return s[0], s[1], (-1 if b == np.iinfo(np.int64).max else int(b))


class TorchComm:
    """torch.distributed collectives (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, device=None):
        import torch
        import torch.distributed as dist

        self.dist = dist
        self.torch = torch
        self.device = device

    def all_to_all(self, send, send_splits, recv_splits):
        torch = self.torch
        recv = torch.empty(int(sum(recv_splits)), dtype=send.dtype, device=send.device)
        self.dist.all_to_all_single(recv, send.contiguous(), output_split_sizes=list(recv_splits),
                                    input_split_sizes=list(send_splits))
        return recv

    def all_reduce_sum(self, values):
        t = self.torch.tensor(values, dtype=self.torch.float64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return t.cpu().tolist()

    def all_reduce_min(self, value):
        t = self.torch.tensor([value], dtype=self.torch.int64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN)
        return int(t.item())

    def all_reduce_max(self, value: float) -> float:
        t = self.torch.tensor([value], dtype=self.torch.float64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())


class DeviceOps:
    """Per-rank device compute through libbhcp_b200.so."""

    def __init__(self, plan, g_dev, divisor: float):
        import torch

        from . import _lib, plans

        self.torch = torch
        self._lib = _lib
        self.plans = plans
        self.plan = plan
        self.lib = _lib.lib()
        self.n = plan.n
        self.nx = plan.grid.n_interior
        dev = g_dev.device
        self.status = plans.status_block()
        self.ghat = torch.empty(self.nx, dtype=torch.float64, device=dev)
        self.g = g_dev
        self.divisor = divisor
        self._tables = {}
        self._W = None
        self._y = None
        self._sync = None   # level-group kernel scratch (bhcp_pint_levels_sync_bytes)

    def prepare(self):
        """status reset + ghat = DST(g) / (divisor * n) (replicated on every rank)."""
        p = self.plans
        self._lib.check(self.lib.bhcp_status_reset(p.ptr(self.status), p.stream_handle()), "reset")
        self._lib.check(self.lib.bhcp_pint_ghat(self.plan.sp.handle, p.ptr(self.g), 1.0 / (self.divisor * self.n),
                                                p.ptr(self.ghat), p.stream_handle()), "ghat")

    def modes(self, layout: SlabLayout, rank: int):
        torch, p = self.torch, self.plans
        kb, ke = layout.mode_range(rank)
        S = ke - kb
        size = sum(layout.tiles(q) for q in range(layout.world)) * TB * S
        if self._W is None or self._W.numel() != size:
            self._W = torch.empty(size, dtype=torch.float64, device=self.g.device)
        bounds = layout.slab_bounds()
        self.prepare()
        self._lib.check(self.lib.bhcp_pint_modes(self.plan.sp.handle, self.plan.tp.handle, p.ptr(self.ghat), kb, ke,
                                                 p.ptr(self._W), layout.world,
                                                 bounds.ctypes.data_as(ctypes.c_void_p), p.ptr(self.status),
                                                 p.stream_handle()), "modes")
        return self._W

    def modes_to(self, layout: SlabLayout, rank: int, dst):
        """Pass A with slab q stored at dst[q] (ctypes array of device pointers,
        local or peer-mapped)."""
        p = self.plans
        kb, ke = layout.mode_range(rank)
        bounds = layout.slab_bounds()
        self.prepare()
        self._lib.check(self.lib.bhcp_pint_modes_to(self.plan.sp.handle, self.plan.tp.handle, p.ptr(self.ghat), kb, ke,
                                                    ctypes.cast(dst, ctypes.c_void_p), layout.world,
                                                    bounds.ctypes.data_as(ctypes.c_void_p), p.ptr(self.status),
                                                    p.stream_handle()), "modes_to")

    def sym_tiles(self) -> int:
        """Length of the symmetric pass-A tile list for this plan (0: none)."""
        if not hasattr(self, "_sym_tiles"):
            self._sym_tiles = int(self.lib.bhcp_pint_sym_tiles(self.plan.sp.handle, self.plan.tp.handle))
        return self._sym_tiles

    def sym_range(self, rank: int, world: int):
        total = self.sym_tiles()
        return total * rank // world, total * (rank + 1) // world

    def modes_sym_to(self, layout: SlabLayout, rank: int, bases):
        """Symmetric pass A over this rank's share of the tile list, both
        mirrors stored into every receiver q at bases[q] + block_tables(q)."""
        p = self.plans
        tb, te = self.sym_range(rank, layout.world)
        koffs = [self.tables(layout, q) for q in range(layout.world)]
        karr = (ctypes.c_void_p * layout.world)(*[k.data_ptr() for k in koffs])
        bounds = layout.slab_bounds()
        self.prepare()
        self._lib.check(self.lib.bhcp_pint_modes_sym_to(self.plan.sp.handle, self.plan.tp.handle, p.ptr(self.ghat),
                                                        tb, te, ctypes.cast(bases, ctypes.c_void_p),
                                                        ctypes.cast(karr, ctypes.c_void_p), layout.world,
                                                        bounds.ctypes.data_as(ctypes.c_void_p), p.ptr(self.status),
                                                        p.stream_handle()), "modes_sym_to")

    def tables(self, layout: SlabLayout, rank: int):
        key = (layout.world, rank)
        if key not in self._tables:
            koff = layout.block_tables(rank)
            # the TMA level passes view the receive buffer with one k1 stride
            # (bhcp_pint_levels_blocked); the slab layouts always produce it
            stride = layout.tiles(rank) * layout.plane * TB
            if not np.array_equal(koff, np.arange(layout.m, dtype=np.int64) * stride):
                raise ValueError("receive-buffer block table is not uniform")
            self._tables[key] = self.torch.from_numpy(koff).to(self.g.device)
        return self._tables[key]

    def levels_blocked(self, recv, koff, L: int):
        torch, p = self.torch, self.plans
        if self._y is None or self._y.shape != (L, self.nx):
            self._y = torch.empty((L, self.nx), dtype=torch.float64, device=self.g.device)
        if L > 0:
            # tables() verified koff is the uniform stride: the receive buffer is a
            # single-slab W of this rank's L levels, so the level-group kernel
            # (k_dst_lvl4, 2D m + 1 = 1024) or the TMA passes (koff NULL) run on it
            nsync = int(self.lib.bhcp_pint_levels_sync_bytes(self.plan.sp.handle, L))
            if nsync:
                if self._sync is None or self._sync.numel() < nsync:
                    self._sync = torch.empty(nsync, dtype=torch.uint8, device=self.g.device)
                self._lib.check(self.lib.bhcp_pint_levels_fused(self.plan.sp.handle, p.ptr(recv), p.ptr(self._y), L,
                                                                p.ptr(self._sync), p.stream_handle()),
                                "levels_fused")
            else:
                self._lib.check(self.lib.bhcp_pint_levels_blocked(self.plan.sp.handle, p.ptr(recv), None,
                                                                  p.ptr(self._y), L, p.stream_handle()),
                                "levels_blocked")
        return self._y

    def local_status(self):
        """(sum Re^2, sum Im^2, first singular column) of this rank (synchronises)."""
        st = self._lib.Status()
        self._lib.check(self.lib.bhcp_read_status(self.plans.ptr(self.status), 1.0, ctypes.byref(st),
                                                  self.plans.stream_handle()), "read_status")
        return st.norm ** 2 - st.residue ** 2, st.residue ** 2, int(st.bad_column)


def check_global_status(comm, ops, shifts, tol: float = 1e-8):
    """Apply the reference's decision rules on the all-reduced status."""
    from .circulant import ImaginaryResidueError
    from .space import SingularShiftError, singular_message

    sre, sim, bad = ops.local_status()
    sre, sim, bad = reduce_status(comm, sre, sim, bad)
    if bad >= 0:
        raise SingularShiftError(f"column {bad}: {singular_message(complex(shifts[bad]))}")
    norm, residue = float(np.sqrt(sre + sim)), float(np.sqrt(sim))
    if residue > tol * max(norm, np.finfo(float).tiny):
        raise ImaginaryResidueError(f"imaginary residue {residue:.3e} exceeds {tol:.1e} of the result norm {norm:.3e}")
    return norm, residue


def solve_pint_sharded(system, comm=None, transport: str = "auto"):
    """Drop-in style entry point under torch.distributed: every rank calls it
    with the same system; returns (local level slab y (L_r, n_space) on this
    rank's GPU, (level_begin, level_end)). ``transport``: 'peer' (pass A
    stores into the receivers over NVLink), 'nccl' (all_to_all_single) or
    'auto'. Both give the single-GPU result bit for bit."""
    import torch
    import torch.distributed as dist

    from . import plans
    from .methods import condition_divisor
    from .pint import _check_kind, pint_plan

    _check_kind(system)
    world, rank = dist.get_world_size(), dist.get_rank()
    comm = comm or TorchComm(torch.device("cuda", torch.cuda.current_device()))
    grid, tg = system.grid, system.timegrid
    layout = SlabLayout(grid.dim, grid.num_cells - 1, tg.n_levels, world)
    plan = pint_plan(grid, tg, system.omega)
    divisor = condition_divisor(system.method.kind, system.method.alpha, tg.tau)
    ops = DeviceOps(plan, plans.to_device(system.data, torch.float64), divisor)
    peer = make_transport(transport, layout, rank, torch.device("cuda", torch.cuda.current_device()))
    if peer is not None:
        y, lev = sharded_solve_peer(ops, peer, layout, rank)
    else:
        y, lev = sharded_solve(ops, comm, layout, rank)
    check_global_status(comm, ops, plan.shifts)
    return y, lev


# ---------------------------------------------------------------- bench (N > 1)

# NVLink 5 per GPU and direction: 770 GB/s measured peer copy on this pool's
# B200s, 900 GB/s nominal (/opt/skills/guides/B200_PROFILING.md, NVLink
# references); the fraction is reported against the measured figure
NVLINK_MEASURED_GBPS = 770.0
NVLINK_NOMINAL_GBPS = 900.0


def _nvlink_stats(nbytes: float, ms: float, transport: str) -> dict:
    """Bytes each rank sends to its peers and the rate over the phase that
    carries them (the all-to-all, or pass A itself for peer stores)."""
    gbps = nbytes / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
    return {"bytes_per_rank": nbytes, "carried_by": "pass A stores" if transport == "peer" else "all_to_all",
            "transport": transport, "achieved_GBps": gbps, "peak_GBps": NVLINK_MEASURED_GBPS,
            "peak_source": "measured peer copy per direction (B200_PROFILING.md); nominal 900",
            "frac": gbps / NVLINK_MEASURED_GBPS, "frac_nominal": gbps / NVLINK_NOMINAL_GBPS}


def bench_sharded(args, w, system, rank, world, dev, ClockSampler, peaks, metric, unit, config_of):
    import torch
    import torch.distributed as dist

    from . import plans
    from .pint import PintPlan

    grid, tg = system.grid, system.timegrid
    layout = SlabLayout(grid.dim, grid.num_cells - 1, tg.n_levels, world)
    plan = PintPlan(grid, tg.n_levels, tg.tau, system.omega)
    divisor = system.method.condition_divisor(tg.tau)
    ops = DeviceOps(plan, torch.from_numpy(w.g_delta).to(dev), divisor)
    comm = TorchComm(dev)
    import os
    peer = make_transport(os.environ.get("BHCP_TRANSPORT", "auto"), layout, rank, dev)
    transport = "peer" if peer is not None else "nccl"

    def solve(events=None):
        if peer is not None:
            return sharded_solve_peer(ops, peer, layout, rank, events=events)
        return sharded_solve(ops, comm, layout, rank, events=events)

    sampler = ClockSampler(dev.index)
    sampler.start()
    for _ in range(args.warmup):
        solve()
    torch.cuda.synchronize()
    check_global_status(comm, ops, plan.shifts)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    t0.record()
    for k in range(args.steps):
        solve(events=evs[k])
    t1.record()
    torch.cuda.synchronize()
    dist.barrier()
    clocks = sampler.stop()
    check_global_status(comm, ops, plan.shifts)
    local_ms = t0.elapsed_time(t1)
    ms = comm.all_reduce_max(local_ms) / args.steps
    ph = np.zeros(3)
    for k in range(args.steps):
        for p in range(3):
            ph[p] += evs[k][p].elapsed_time(evs[k][p + 1])
    ph /= args.steps
    a2a_bytes = 8.0 * sum(s for q, s in enumerate(layout.send_splits(rank)) if q != rank)
    value = w.dof / (ms * 1e-3)
    hbm, kind = peaks()
    # e2e: pinned host g -> device, sharded solve, this rank's level slab -> pinned host
    g_host = torch.from_numpy(w.g_delta).pin_memory()
    c0, c1 = layout.lev[rank]
    y_host = torch.empty((c1 - c0, w.n_space), dtype=torch.float64).pin_memory()
    g_dev = ops.g

    def e2e_step():
        g_dev.copy_(g_host, non_blocking=True)
        y, _ = solve()
        y_host.copy_(y, non_blocking=True)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    dist.barrier()
    a0 = torch.cuda.Event(enable_timing=True)
    a1 = torch.cuda.Event(enable_timing=True)
    e2e_steps = max(3, min(args.steps, 10))
    a0.record()
    for _ in range(e2e_steps):
        e2e_step()
    a1.record()
    torch.cuda.synchronize()
    e2e_ms = comm.all_reduce_max(a0.elapsed_time(a1)) / e2e_steps
    check_global_status(comm, ops, plan.shifts)
    # dominant per-rank phase vs HBM: pass A writes 8 B per local DOF, pass B moves 32 B per local DOF
    local_dof_a = layout.slab_modes(rank) * layout.n
    local_dof_b = layout.levels(rank) * layout.n_space
    alg = [8.0 * local_dof_a, 0.0, 32.0 * local_dof_b]
    dom = 0 if ph[0] >= ph[2] else 2
    achieved = alg[dom] / (ph[dom] * 1e-3) / 1e9
    modes_kernel = {257: "k_modes_rader", 513: "k_modes_fast", 1025: "k_modes_gt", 4097: "k_modes_pf"}.get(
        tg.n_levels, "k_modes")
    level_kernels = {256: "k_dst_wax + k_dst_blk3", 512: "k_dst_wax2 + k_dst_blk3",
                     1024: "k_dst_lvl4"}.get(grid.num_cells, "level passes")
    # the same per-kernel breakdown as the N = 1 line (rank 0's phases, algorithmic bytes of its slab)
    kernels = [
        {"kernel": f"{modes_kernel} (pass A, this rank's modes, W stores" +
                   (" into the owners over NVLink)" if peer is not None else ")"),
         "ms": ph[0], "alg_bytes": alg[0], "achieved_GBps": alg[0] / (ph[0] * 1e-3) / 1e9 if ph[0] > 0 else 0.0},
        {"kernel": "rank barrier" if peer is not None else "NCCL all_to_all", "ms": ph[1], "alg_bytes": a2a_bytes,
         "achieved_GBps": a2a_bytes / (ph[1] * 1e-3) / 1e9 if ph[1] > 0 else 0.0},
        {"kernel": f"{level_kernels} (level passes of this rank's level slab)", "ms": ph[2], "alg_bytes": alg[2],
         "achieved_GBps": alg[2] / (ph[2] * 1e-3) / 1e9 if ph[2] > 0 else 0.0},
    ]
    for k in kernels:
        k["hbm_frac"] = k["achieved_GBps"] / hbm
    launches = 1 + (grid.dim + 1) + 1 + grid.dim  # status reset, ghat (dim passes + scale), modes, level passes
    if rank != 0:
        return None
    return {
        "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json config construction)",
        "config": config_of(args.config, w, system.method.kind.value, system.method.alpha),
        "transport": transport,
        "parallelism": (f"pass A over 1/P of the mirror-pair tiles (or a k1 slab) storing into the "
                        f"level-slab owners over NVLink peer memory -> level slabs, P={world}")
                       if peer is not None else
                       f"mode slabs -> NCCL all-to-all -> level slabs, P={world}",
        "roofline": {"bound": "hbm", "kernel": kernels[dom]["kernel"],
                     "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm, "traffic": None,
                     "peak_source": kind},
        "phases_ms_rank0": {"pass_a_modes": ph[0], ("rank_barrier" if peer is not None else "all_to_all"): ph[1],
                            "pass_b_levels": ph[2]},
        "kernels": kernels,
        "nvlink": _nvlink_stats(a2a_bytes, ph[0] if peer is not None else ph[1], transport),
        "e2e": {"value": w.dof / (e2e_ms * 1e-3), "unit": unit, "h2d_bytes_per_step": 8 * w.n_space,
                "d2h_bytes_per_step": 8 * (c1 - c0) * w.n_space, "ms_per_step": e2e_ms},
        "gpu_launches": launches * args.steps,
        "clocks": clocks,
    }
