"""The NCCL slab path end to end on one GPU (world size 1 under torchrun:
the all-to-all is a self-exchange): solve_pint_sharded equals solve_pint bit
for bit and the sharded bench line is well formed."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r'''
import sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, "{root}")
import paper_2107_06381_b200 as B
from paper_2107_06381_b200 import workloads
from paper_2107_06381_b200.distributed import solve_pint_sharded
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
w = workloads.make_small(2, 40, 30, seed=5)
grid = B.build_grid(2, w.length, 40)
system = B.assemble(B.MethodKind.PINT_QBVM, 1e-3, grid, B.TimeGrid(w.horizon, 30), w.g_delta)
ref = B.solve_pint(system).trajectory
for transport in ("nccl", "peer"):
    y, (c, d) = solve_pint_sharded(system, transport=transport)
    assert (c, d) == (0, 31)
    assert np.array_equal(y.cpu().numpy(), ref), f"sharded ({{transport}}) != single"
    print("SHARDED_OK", transport)
dist.destroy_process_group()
'''


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def torchrun(args, env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port())] + args
    return subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                          env={**os.environ, **(env or {})})


def test_solve_pint_sharded_world1_nccl(tmp_path):
    script = tmp_path / "sharded.py"
    script.write_text(SCRIPT.format(root=ROOT))
    r = torchrun([str(script)])
    assert r.returncode == 0, r.stderr[-2000:]
    assert "SHARDED_OK nccl" in r.stdout and "SHARDED_OK peer" in r.stdout


@pytest.mark.parametrize("transport", ["nccl", "peer"])
def test_bench_sharded_line_world1(transport):
    r = torchrun(["bench.py", "--gpus", "1", "--steps", "3", "--warmup", "1"],
                 env={"BHCP_FORCE_SHARDED": "1", "BHCP_TRANSPORT": transport})
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "ms_per_step", "e2e", "gpu_launches", "clocks", "roofline"):
        assert key in line
    assert line["value"] > 0
    assert line["transport"] == transport
