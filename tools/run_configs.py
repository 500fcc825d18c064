"""Time the fused device solve on every BASELINE config and check sampled
levels against the closed-form oracle; with --cpu also time the reference
3-step algorithm (oracle port) on a bounded sample of each config on the
host cores (usage: python tools/run_configs.py [--cpu] [c1 c3 ...])."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2107_06381_b200 as B
from oracle import bhcp_oracle as O
from paper_2107_06381_b200 import workloads

import os
cpu = "--cpu" in sys.argv
names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["c1", "c2", "c3", "c4", "c5"]
# sample fractions: every per-unit op of the 3-step solve on this share of rows / columns (about 5-20 s each)
CPU_FRACTION = {"c1": 1.0, "c2": 0.3, "c3": 0.03, "c4": 0.01, "c5": 0.2}
CPU_THREADS = os.cpu_count() or 1
out = {}
for name in names:
    t0 = time.time()
    w = workloads.make(name)
    gen_s = time.time() - t0
    grid = B.build_grid(w.dim, w.length, w.num_cells)
    tg = B.TimeGrid(w.horizon, w.num_steps)
    alphas = [w.alphas[0]] if name != "c5" else [w.alphas[0], w.alphas[32], w.alphas[-1]]
    res = {}
    for kind in w.kinds:
        for alpha in alphas:
            system = B.assemble(B.MethodKind(kind), alpha, grid, tg, w.g_delta)
            plan = B.PintPlan(grid, tg.n_levels, tg.tau, system.omega)
            g = torch.from_numpy(w.g_delta).cuda()
            div = system.method.condition_divisor(tg.tau)
            y = plan.solve_device(g, div)
            torch.cuda.synchronize()
            plan.check_status()
            reps = 3 if w.dof > 1e9 else 10
            graph = plan.capture(g, div, y)   # timed as CUDA-graph replays of the step
            graph.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                graph.replay()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            plan.check_status()
            levels = np.unique(np.linspace(0, w.num_steps, 5).astype(int))
            ref = O.spectral_oracle(kind, alpha, w.dim, w.length, w.num_cells, w.horizon, w.num_steps, w.g_delta,
                                    levels=levels)
            yl = y[torch.from_numpy(levels).cuda()].cpu().numpy()
            err = float(np.linalg.norm(yl - ref) / np.linalg.norm(ref))
            tol = O.parity_tolerance(tg.n_levels, system.omega)
            eh = workloads.l2_error(yl[0], w.z0, grid.h, w.dim)
            eh_ref = workloads.l2_error(ref[0], w.z0, grid.h, w.dim)
            res[f"{kind} alpha={alpha:.3g}"] = {"ms": ms, "GDOF_s": w.dof / ms / 1e6, "rel_l2_sampled_levels": err,
                                               "tol": tol, "ok": bool(err <= tol), "e_h": eh, "e_h_oracle": eh_ref}
            del y, plan, graph
            torch.cuda.empty_cache()
    out[name] = {"dof": w.dof, "gen_s": gen_s, "results": res}
    if name == "c5":
        # the full error-vs-alpha curve: 64 alpha x 2 kinds, every e_h against the oracle's
        from paper_2107_06381_b200 import sweep
        sw = sweep.alpha_sweep(grid, tg, w.g_delta, w.z0, w.kinds, w.alphas)
        dev = []
        for p in sw.points:
            ref0 = O.spectral_oracle(p.kind, p.alpha, w.dim, w.length, w.num_cells, w.horizon, w.num_steps,
                                     w.g_delta, levels=np.array([0]))
            e_ref = workloads.l2_error(ref0[0], w.z0, grid.h, w.dim)
            dev.append(abs(p.e_h - e_ref) / e_ref)
        out[name]["sweep"] = {
            "solves": len(sw.points), "wall_s": sw.wall_s, "device_ms_total": sum(p.ms for p in sw.points),
            "max_rel_dev_e_h": max(dev), "ok_3_sig_digits": bool(max(dev) <= 5e-4),
            "best": {k: {"alpha": sw.best(k).alpha, "e_h": sw.best(k).e_h} for k in w.kinds},
            "curve": {k: [[float(a), float(e)] for a, e in zip(*sw.curve(k))] for k in w.kinds}}
    if cpu:
        kind, alpha = w.kinds[0], w.alphas[0]
        dof_eq, secs = O.solve_pint_sample(kind, alpha, w.dim, w.length, w.num_cells, w.horizon, w.num_steps,
                                           w.g_delta, CPU_FRACTION[name], workers=CPU_THREADS)
        gpu_best = min(r["ms"] for r in res.values())
        out[name]["cpu_reference"] = {"DOF_s": dof_eq / secs, "threads": CPU_THREADS, "fraction": CPU_FRACTION[name],
                                      "seconds": secs, "kind": "port",
                                      "gpu_speedup": (w.dof / (gpu_best * 1e-3)) / (dof_eq / secs)}
    print(name, json.dumps(out[name]), flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/configs.json").write_text(json.dumps(out, indent=1))
