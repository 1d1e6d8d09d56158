"""The driver's N > 1 launch of bench.py (torchrun, one rank per GPU, NCCL) on a one-GPU box:
ST_BENCH_SHARED_GPU=1 puts both ranks on cuda:0 as distinct NCCL hosts. Checks the path
end to end — the NCCL parity leg against the oracle (trace exact, W / loss / ΔW gates),
the 1F1B session over NCCL, barrier + max-over-ranks timing and the JSON line — not speed."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_torchrun_two_ranks_nccl_parity_leg():
    env = dict(os.environ, ST_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--workload", "deep_mlp", "--steps", "4", "--warmup", "3", "--no-cpu", "--no-e2e"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 4 and d["value"] > 0
    assert d["config"]["stages"] == 2 and "shared_gpu_validation" in d["config"]
    leg = d["nccl_parity"]
    assert leg["trace_bit_exact"] and leg["pass"], leg
    assert leg["w_rel_l2"] <= 1e-4 and leg["loss_rel_l2"] <= 1e-4
