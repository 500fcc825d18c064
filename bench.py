"""Benchmark of the PinT QBVM/MQBVM all-at-once solve on B200.

Contract (see the task statement): ``python bench.py --gpus N --steps K
--warmup W`` prints ONE JSON line on rank 0. A "step" is one complete solve
of BASELINE.json config 3 -- the largest config that fits one GPU (2D
pint-qbvm, 1023^2 interior, N = 1024 steps, 1,072,692,225 space-time DOFs) --
with the data g already resident in HBM; the metric is space-time DOFs/s over
all ranks. ``--config c1|c2|c4|c5`` runs the others.

* value      -- K solves timed with CUDA events on the launching stream,
                barrier + synchronize on both sides, max over ranks.
* e2e        -- the same solve through the C-ABI call with HOST buffers:
                pinned g -> device, bhcp_pint_solve, full trajectory -> pinned
                host, every step inside the timed region (the trajectory copy of
                step k overlaps step k+1 on a second stream).
* roofline   -- dominant kernel of the step: algorithmic bytes (or, for the
                FP64-bound pass A, algorithmic flops) / its average CUDA-event
                duration vs the measured HBM copy bandwidth (FP64 FMA peak);
                roofline_hbm / kernels give every kernel's HBM fraction.
* cpu_baseline -- the reference 3-step algorithm (oracle port, bit-identical
                to the reference on the golden vectors) on a bounded sample of
                the same workload (a fraction f of every per-unit operation,
                extrapolated as elapsed / f), 1 host core = the reference's
                default workers=None, rank 0 at N=1.
* ``--impl reference`` times that CPU path with all host threads instead.

N > 1: slab decomposition (mode slabs -> NCCL all-to-all -> level slabs),
strong scaling of the one problem over the ranks.
"""

from __future__ import annotations

import argparse
import ctypes
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

CONFIG_NAME = "c3"
# fraction of every per-unit operation in the CPU samples: about 10-30 s of
# one host core (cpu_baseline) and about 1-3 s of all host threads per
# --impl reference step
CPU_FRACTION = {"c1": 1.0, "c2": 1.0, "c3": 0.05, "c4": 0.01, "c5": 1.0}
REF_FRACTION = {"c1": 1.0, "c2": 0.1, "c3": 0.03, "c4": 0.005, "c5": 0.5}
METRIC = "space-time DOFs/s of QBVM/MQBVM all-at-once solve; % of HBM roofline"
UNIT = "DOF/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default=CONFIG_NAME)
    p.add_argument("--cpu-fraction", type=float, default=None,
                   help="fraction of every per-unit operation in the CPU-baseline sample (default per config)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--quick", action="store_true", help="device timing only (no e2e / unfused / CPU legs)")
    return p.parse_args()


def peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def describe(name, w, kind, alpha) -> str:
    return f"{name}: {w.dim}D {kind}, {w.num_cells - 1}^{w.dim} interior x {w.n_levels} levels, alpha={alpha:g}"


def config_of(name, w, kind, alpha) -> dict:
    """The `config` object of both arms' lines (identical, so the driver can pair them)."""
    return {"workload": describe(name, w, kind, alpha), "dof_per_solve": w.dof,
            "l2": f"working set (W + y = {2 * 8 * w.dof / 1e9:.2f} GB) larger than the 126 MB L2; no flush"}


def fp64_peak():
    """Dense FP64 FMA throughput measured on a B200 of this pool by tools/probe_fp64.cu
    (profiles/fp64_peak.json), else the 37 TFLOP/s datasheet figure."""
    f = ROOT / "profiles" / "fp64_peak.json"
    if f.exists():
        d = json.loads(f.read_text())
        return float(d["dfma_tflops"]), "measured (tools/probe_fp64.cu)"
    return 37.0, "datasheet"


def modes_alg_flops(dim: int, m: int, n: int) -> float:
    """Algorithmic FP64 flops of pass A: per time FFT of length n the textbook
    5 n log2 n, plus 7 flops per point for the shift generator 1/(s_j + mu); per
    stored mode 8 flops per level (Re(gamma^-1 X) * ghat and the two residue
    norms). 2D/3D: one FFT serves a mirror pair of modes (k1 <-> k2)."""
    import math
    modes = m ** dim
    ffts = modes if dim == 1 else (m * (m + 1) // 2) * (m ** (dim - 2))
    return ffts * (5.0 * n * math.log2(n) + 7.0 * n) + modes * 8.0 * n


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the GPU is loaded."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_sample(w, kind, alpha, fraction, workers):
    from oracle import bhcp_oracle as O

    dof, secs = O.solve_pint_sample(kind, alpha, w.dim, w.length, w.num_cells, w.horizon, w.num_steps,
                                    w.g_delta, fraction, workers=workers)
    return dof, secs


def reference_package_check(w, kind, alpha, cores, levels=33):
    """The UNMODIFIED reference package (pip-installed into baseline/_ref, test data
    only) on this config's spatial grid with a reduced number of time levels, next
    to the oracle port on exactly the same reduced problem: pins the port's timing
    (and its trajectory) to the reference's own solve_pint (pint.py:69-110) on the
    box the bench runs on. None when the package is not there."""
    ref_root = ROOT / "baseline" / "_ref"
    if not (ref_root / "bhcp").is_dir():
        return None
    import time

    import numpy as np

    sys.path.insert(0, str(ref_root))
    try:
        from bhcp.circulant import TimeGrid
        from bhcp.methods import MethodKind, assemble
        from bhcp.pint import solve_pint
        from bhcp.space import build_grid
    except Exception as e:  # noqa: BLE001 -- reported, not fatal
        return {"unavailable": f"{type(e).__name__}: {e}"}
    finally:
        sys.path.pop(0)
    from oracle import bhcp_oracle as O

    if w.dim > 2:
        return {"unavailable": "the reference rejects dim 3 (space.py:42-43)"}
    steps = min(levels - 1, w.num_steps)
    horizon = w.horizon * steps / w.num_steps   # the same tau as the full config
    grid = build_grid(w.dim, w.length, w.num_cells)
    tg = TimeGrid(horizon, steps)
    system = assemble(MethodKind(kind), alpha, grid, tg, w.g_delta)
    dof = (steps + 1) * w.g_delta.shape[0]
    out = {"levels": steps + 1, "dof": dof, "note": "same spatial grid and tau, reduced time levels"}
    try:
        for label, workers in (("workers_none", None), ("workers_all", cores)):
            t0 = time.perf_counter()
            res = solve_pint(system, workers=workers)
            out[label] = {"seconds": time.perf_counter() - t0, "DOF_s": dof / (time.perf_counter() - t0),
                          "workers": workers}
        traj = np.asarray(res.trajectory)
    except Exception as e:  # noqa: BLE001 -- e.g. ImaginaryResidueError at this size
        out["unavailable"] = f"{type(e).__name__}: {e}"
        return out
    d1, s1 = O.solve_pint_sample(kind, alpha, w.dim, w.length, w.num_cells, horizon, steps, w.g_delta, 1.0,
                                 workers=None)
    dn, sn = O.solve_pint_sample(kind, alpha, w.dim, w.length, w.num_cells, horizon, steps, w.g_delta, 1.0,
                                 workers=cores)
    out["port_workers_none"] = {"seconds": s1, "DOF_s": d1 / s1}
    out["port_workers_all"] = {"seconds": sn, "DOF_s": dn / sn, "workers": cores}
    orc, _ = O.solve_pint(kind, alpha, w.dim, w.length, w.num_cells, horizon, steps, w.g_delta)
    out["port_vs_reference_rel_l2"] = float(np.linalg.norm(orc - traj) / np.linalg.norm(traj))
    return out


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU algorithm (oracle port) on host cores."""
    if rank != 0:
        return
    from paper_2107_06381_b200 import workloads

    w = workloads.make(args.config)
    kind, alpha = w.kinds[0], w.alphas[0]
    cores = os.cpu_count() or 1
    frac = args.cpu_fraction if args.cpu_fraction is not None else REF_FRACTION.get(args.config, 0.05)
    for _ in range(args.warmup):
        cpu_sample(w, kind, alpha, frac / 4, cores)
    total_dof, total_s = 0.0, 0.0
    for _ in range(args.steps):
        dof, s = cpu_sample(w, kind, alpha, frac, cores)
        total_dof += dof
        total_s += s
    value = total_dof / total_s
    pkg = reference_package_check(w, kind, alpha, cores)
    sample = (f"{args.config}: per step, fraction {frac} of every per-unit op of the reference 3-step solve "
              f"(time FFTs of {frac:.1%} of the spatial rows, shifted solves incl. the singular-shift scan of "
              f"{frac:.1%} of the levels on a {cores}-thread pool, back transform + residue + transposed copy of "
              f"{frac:.1%} of the rows); DOF/s = {frac} * DOF / elapsed (every op is linear in rows/levels)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_s / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json config construction)",
        "config": config_of(args.config, w, kind, alpha),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if pkg is not None:
        line["reference_package"] = pkg
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    # BHCP_FORCE_SHARDED=1 runs the slab-decomposed NCCL path even on one rank
    # (exercises the multi-GPU code on a single-GPU box: all-to-all to itself)
    sharded = world > 1 or os.environ.get("BHCP_FORCE_SHARDED") == "1"
    if sharded:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2107_06381_b200 import _lib, plans, workloads
    from paper_2107_06381_b200 import distributed as D
    import paper_2107_06381_b200 as B

    w = workloads.make(args.config)
    kind, alpha = w.kinds[0], w.alphas[0]
    grid = B.build_grid(w.dim, w.length, w.num_cells)
    tg = B.TimeGrid(w.horizon, w.num_steps)
    system = B.assemble(B.MethodKind(kind), alpha, grid, tg, w.g_delta)
    divisor = system.method.condition_divisor(tg.tau)
    dev = torch.device("cuda", local)
    g_dev = torch.from_numpy(w.g_delta).to(dev)
    stream = torch.cuda.current_stream()
    lib = _lib.lib()
    nx, n = w.n_space, w.n_levels

    if not sharded:
        plan = B.PintPlan(grid, n, tg.tau, system.omega)
        y = torch.empty((n, nx), dtype=torch.float64, device=dev)
        ws = plan.workspace()
        wsp = ws.data_ptr()
        status = ctypes.c_void_p(wsp)
        ghat = ctypes.c_void_p(wsp + 256)
        W = ctypes.c_void_p(wsp + 256 + ((8 * nx + 255) // 256) * 256)
        sh = plans.stream_handle()
        sp, tp = plan.sp.handle, plan.tp.handle
        ev = None
        wax = bool(lib.bhcp_pint_w_passes_supported(sp))
        # the one-kernel level-group pass (k_dst_lvl4: 2D, m + 1 = 1024)
        lvl_sync = int(lib.bhcp_pint_levels_sync_bytes(sp, n))
        sync_buf = torch.zeros(max(lvl_sync, 8) // 4 + 1, dtype=torch.int32, device=dev)

        def step(record=None):
            # phases: [0] ghat, [1] k_modes, [2 + a] DST axis pass a
            if record:
                record[0].record()
            _lib.check(lib.bhcp_status_reset(status, sh), "reset")
            _lib.check(lib.bhcp_pint_ghat(sp, plans.ptr(g_dev), 1.0 / (divisor * n), ghat, sh), "ghat")
            if record:
                record[1].record()
            _lib.check(lib.bhcp_pint_modes(sp, tp, ghat, 0, nx, W, 0, None, status, sh), "modes")
            if record:
                record[2].record()
            # the solve's own pass order (bhcp_pint_levels): strided axes in place
            # on W (k_dst_wax), then the last axis W -> y (k_dst_blk2)
            if lvl_sync:
                _lib.check(lib.bhcp_pint_levels_fused(sp, W, plans.ptr(y), n, plans.ptr(sync_buf), sh), "levels")
                if record:
                    record[3].record()
            elif wax:
                for a in range(w.dim - 1):
                    _lib.check(lib.bhcp_pint_w_pass(sp, W, n, a, sh), "w pass")
                    if record:
                        record[3 + a].record()
                _lib.check(lib.bhcp_pint_level_pass(sp, W, None, plans.ptr(y), n, 0, sh), "level pass")
                if record:
                    record[2 + w.dim].record()
            else:
                for a in range(w.dim):
                    _lib.check(lib.bhcp_pint_level_pass(sp, W, None, plans.ptr(y), n, a, sh), "level pass")
                    if record:
                        record[3 + a].record()

        # kernels in the graph of bhcp_pint_solve: reset, ghat passes, modes, level
        # passes (the level-group pass is one kernel after a memset node)
        launches_per_step = 1 + w.dim + 1 + (1 if lvl_sync else w.dim)
        sampler = ClockSampler(local)
        sampler.start()
        time.sleep(0.5)  # let nvidia-smi start sampling before the GPU is loaded
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        plan.check_status()
        nph = 4 if lvl_sync else 3 + w.dim
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nph)] for _ in range(args.steps)]
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        # timed region: K replays of the captured step (one CUDA graph = the 7 kernels)
        graph = plan.capture(g_dev, divisor, y)
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()
        t0.record()
        for k in range(args.steps):
            graph.replay()
        t1.record()
        torch.cuda.synchronize()
        plan.check_status()
        total_ms = t0.elapsed_time(t1)
        # per-phase CUDA events come from a second, eager pass over the same K steps
        for k in range(args.steps):
            step(evs[k])
        torch.cuda.synchronize()
        clocks = sampler.stop()
        plan.check_status()
        phase_ms = np.zeros(nph - 1)
        for k in range(args.steps):
            for p in range(nph - 1):
                phase_ms[p] += evs[k][p].elapsed_time(evs[k][p + 1])
        phase_ms /= args.steps
        modes_kernel = {257: "k_modes_rader", 513: "k_modes_fast", 1025: "k_modes_gt", 4097: "k_modes_pf"}.get(n, "k_modes")
        names = ["ghat (DST of g)", f"{modes_kernel} (shifts + time FFT + Gamma^-1 + Re)"]
        if lvl_sync:
            names += ["k_dst_lvl4 level phase (both axes, W -> y, L2-resident level tiles)"]
        elif wax:
            names += [("k_dst_wax2" if w.num_cells == 512 else "k_dst_wax") +
                      f" W pass (spatial axis {a}, in place, TMA)" for a in range(w.dim - 1)]
            names += ["k_dst_blk3 level pass (axis -1, W -> y)"]
        else:
            names += [(("k_dst_blk4" if w.num_cells == 1024 else "k_dst_blk2") if a == 0 else "k_dst_cols3") +
                      f" level pass {a} (axis -{a + 1})" for a in range(w.dim)]
        dom = int(np.argmax(phase_ms))
        # algorithmic bytes per launch of each kernel
        dof = w.dof
        alg_bytes = [16.0 * nx, 8.0 * dof + 8.0 * nx] + [16.0 * dof] * (nph - 3)
        hbm, peak_kind = peaks()
        # DRAM bytes per launch of each kernel from the committed ncu --set full capture
        tfile = ROOT / "profiles" / f"ncu_traffic_{args.config}.json"
        tmap = json.loads(tfile.read_text()) if tfile.exists() else {}

        def traffic_of(name):
            short = name.split()[0]
            for key, val in tmap.items():
                if key.split("::")[-1].split("<")[0] == short:
                    return val
            return None

        kernels = []
        for i, nm in enumerate(names):
            gbs = alg_bytes[i] / (phase_ms[i] * 1e-3) / 1e9
            kernels.append({"kernel": nm, "ms": float(phase_ms[i]), "alg_bytes": alg_bytes[i],
                            "achieved_GBps": gbs, "hbm_frac": gbs / hbm, "traffic": traffic_of(nm)})
        # the dominant HBM-bound kernel (the level passes); pass A is FP64-bound
        mem_idx = [i for i in range(2, len(names))]
        mdom = max(mem_idx, key=lambda i: phase_ms[i])
        roof_hbm = {"bound": "hbm", "kernel": names[mdom], "achieved": kernels[mdom]["achieved_GBps"], "peak": hbm,
                    "unit": "GB/s", "frac": kernels[mdom]["hbm_frac"], "traffic": kernels[mdom]["traffic"],
                    "peak_source": peak_kind, "alg_bytes_per_launch": alg_bytes[mdom]}
        if lvl_sync and w.num_cells == 1024:
            roof_hbm["note"] = ("k_dst_lvl4 moves its 16 B/DOF of compulsory traffic (read W, write y) at well under "
                                "the HBM peak: it is bound by the LSU / shared-memory pipe of its consumer warps (six "
                                "conflict-free 16 KB passes per 1024-point line pair, the prefix-sum shuffles and the "
                                "global stores: ~75% busy; FP64 pipe 38%; removing every butterfly saves 0.4 of 8.8 ms "
                                "-- DESIGN.md 3.3, profiles/r02_c3_summary.md), not by HBM or FP64")
        # pass A against the measured FP64 peak (reported whichever kernel dominates)
        fpk, fpk_kind = fp64_peak()
        flops = modes_alg_flops(w.dim, w.num_cells - 1, n)
        tf = flops / (phase_ms[1] * 1e-3) / 1e12
        roof_fp64 = {"bound": "fp64", "kernel": names[1], "achieved": tf, "peak": fpk, "unit": "TFLOP/s",
                     "frac": tf / fpk, "traffic": kernels[1]["traffic"], "peak_source": fpk_kind,
                     "alg_flops_per_launch": flops,
                     "hbm": {"achieved": kernels[1]["achieved_GBps"], "frac": kernels[1]["hbm_frac"],
                             "alg_bytes_per_launch": alg_bytes[1]}}
        if dom == 1:
            roofline = dict(roof_fp64, note="pass A is the dominant kernel and is FP64-bound (one n-point time FFT "
                                            "per mirror pair of modes, 8 B/DOF written); roofline_hbm is the "
                                            "dominant HBM-bound kernel")
        else:
            roofline = roof_hbm
        ms_per_step = total_ms / args.steps
        value = dof / (ms_per_step * 1e-3)
        # the pipe that actually bounds both c3 kernels: L1 data-pipe (LSU) wavefronts
        # -- shared-memory loads/stores, shuffles, global stores -- counted per launch
        # by ncu (profiles/ncu_lsu_c3.json; fixed for a workload) over the live kernel
        # time, against one wavefront per clock per SM at the sampled SM clock
        roof_lsu = None
        lsu_file = ROOT / "profiles" / "ncu_lsu_c3.json"
        if args.config == "c3" and lsu_file.exists() and clocks.get("sm_mhz"):
            cnt = json.loads(lsu_file.read_text())
            peak_wf = 148 * clocks["sm_mhz"] * 1e6
            roof_lsu = {"bound": "lsu", "unit": "G wavefronts/s", "peak": peak_wf / 1e9,
                        "peak_source": "1 wavefront / clk / SM x 148 SMs x the SM clock sampled under load",
                        "kernels": []}
            for key, idx in (("fastk::k_modes_gt", 1), ("lvl::k_dst_lvl4", 2)):
                if key in cnt and idx < len(names):
                    wf = cnt[key]["lsu_data_wavefronts"]
                    ach = wf / (phase_ms[idx] * 1e-3)
                    roof_lsu["kernels"].append({"kernel": names[idx], "wavefronts_per_launch": wf,
                                                "achieved": ach / 1e9, "frac": ach / peak_wf})
            roof_lsu["note"] = ("both kernels issue their shared-memory passes in bursts (every warp reaches the same "
                                "FFT stage together), so the average sits below 1 while the bursts saturate the pipe; "
                                "see DESIGN.md 3.3 for the ablation runs")

        if args.quick:
            print(json.dumps({"config": args.config, "ms_per_step": ms_per_step, "value": value,
                              "phases_ms": {nm: float(t) for nm, t in zip(names, phase_ms)}}), flush=True)
            return
        # ---- e2e through the C-ABI with host buffers. Every step: pinned g -> device
        # (compute stream), bhcp_pint_solve, full trajectory -> pinned host on a copy
        # stream. Two trajectory buffers let step k's device->host copy overlap step
        # k+1's H2D + solve; the timed region ends when the last copy has landed.
        g_host = torch.from_numpy(w.g_delta).pin_memory()
        # one pinned host trajectory (the copies serialise on copy_stream anyway)
        y_host = torch.empty((n, nx), dtype=torch.float64).pin_memory()
        y_hosts = [y_host, y_host]
        ys = [y, torch.empty_like(y)]
        g_e2e = torch.empty_like(g_dev)
        wsb = plan.ws_bytes
        copy_stream = torch.cuda.Stream()
        solved = [torch.cuda.Event() for _ in range(2)]
        copied = [None, None]

        def e2e_step(k):
            b = k % 2
            if copied[b] is not None:
                stream.wait_event(copied[b])           # y buffer b's previous copy has read it
            g_e2e.copy_(g_host, non_blocking=True)
            _lib.check(lib.bhcp_pint_solve(sp, tp, plans.ptr(g_e2e), divisor, plans.ptr(ys[b]), ctypes.c_void_p(wsp),
                                           wsb, sh), "solve")
            solved[b].record(stream)
            with torch.cuda.stream(copy_stream):
                copy_stream.wait_event(solved[b])
                y_hosts[b].copy_(ys[b], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy_stream)
                copied[b] = ev

        e2e_steps = max(3, min(args.steps, 10))
        for k in range(2):
            e2e_step(k)
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for k in range(e2e_steps):
            e2e_step(k)
        stream.wait_stream(copy_stream)
        a1.record(stream)
        torch.cuda.synchronize()
        plan.check_status()
        e2e_ms = a0.elapsed_time(a1) / e2e_steps
        e2e_value = dof / (e2e_ms * 1e-3)

        # ---- unfused literal 3-step dataflow for comparison (same kernels family;
        # two complex (n, nx) intermediates: skipped above 2e9 DOF)
        del y_hosts, y_host
        unfused_ms = None
        if dof <= 2e9:
            yu, wsu = plan.solve_unfused_device(g_dev, divisor)
            torch.cuda.synchronize()
            u0 = torch.cuda.Event(enable_timing=True)
            u1 = torch.cuda.Event(enable_timing=True)
            u0.record()
            for _ in range(3):
                plan.solve_unfused_device(g_dev, divisor, out=yu)
            u1.record()
            torch.cuda.synchronize()
            unfused_ms = u0.elapsed_time(u1) / 3
            del yu, wsu

        cpu = None
        if not args.no_cpu_baseline:
            frac = args.cpu_fraction if args.cpu_fraction is not None else CPU_FRACTION.get(args.config, 0.05)
            dof_s, secs = cpu_sample(w, kind, alpha, frac, None)
            cpu = {"value": dof_s / secs, "unit": UNIT, "cores": 1, "kind": "port",
                   "sample": f"{args.config}, fraction {frac} of every per-unit op of the reference 3-step solve "
                             f"(time FFTs of {frac:.1%} of the spatial rows, shifted solves incl. the singular-shift "
                             f"scan of {frac:.1%} of the levels, back transform + residue + transposed copy of "
                             f"{frac:.1%} of the rows) in {secs:.1f} s on one thread (the reference default "
                             f"workers=None); value = {frac} * DOF / elapsed, i.e. extrapolated linearly to the "
                             f"full solve ({secs / frac:.0f} s)",
                   "fraction": frac, "elapsed_s": secs, "extrapolated_full_solve_s": secs / frac}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json config construction)",
            "config": config_of(args.config, w, kind, alpha),
            "timing": f"K replays of the CUDA graph of one step ({launches_per_step} kernels); phases_ms from an eager "
                      "pass of the same K steps with CUDA events",
            "roofline": roofline,
            "roofline_hbm": roof_hbm,
            "roofline_fp64": roof_fp64,
            "roofline_lsu": roof_lsu,
            "kernels": kernels,
            "phases_ms": {nm: float(t) for nm, t in zip(names, phase_ms)},
            "pipeline_72B_per_dof": {"achieved_GBps": 72.0 * dof / (ms_per_step * 1e-3) / 1e9,
                                     "frac": 72.0 * dof / (ms_per_step * 1e-3) / 1e9 / hbm,
                                     "note": "SURVEY 8(d) 3-step algorithmic bytes; >1 means fused dataflow"},
            "unfused_3step_ms": unfused_ms,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * nx, "d2h_bytes_per_step": 8 * n * nx,
                    "ms_per_step": e2e_ms},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
        return

    # ---------------- N > 1: slab-decomposed solve
    line = D.bench_sharded(args, w, system, rank, world, dev, ClockSampler, peaks, METRIC, UNIT, config_of)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
