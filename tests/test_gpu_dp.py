"""Data-parallel comparator on the GPU (-m gpu): two replica
processes share cuda:0 (gloo all-reduce of the G arena; NCCL needs one GPU per rank),
each trains on its half of every mini-batch through the library's verbs; the result must
equal the oracle's 1-stage run on the whole batch (reading D23): W and the averaged loss
within 1e-4 rel-L2."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synthdata as sd
from tests.gpu_helpers import layers_of, oracle_run, rel_l2

pytestmark = pytest.mark.gpu

MODEL = dict(widths=[784, 128, 96, 10])
M, B, LR = 12, 32, 0.05


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    import torch.distributed as dist

    import paper_1809_02839_b200 as st
    from paper_1809_02839_b200.dp import DataParallelStage
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    model = sd.mlp(MODEL["widths"], cuts=[])
    w0, X, Y = sd.parity_inputs(model, M, B, seed=11)
    half = B // world
    dev = torch.device("cuda", 0)
    r = DataParallelStage(layers_of(model), half, LR, 0.9, gemm=st.ST_GEMM_FP32X3, device=0, max_minibatches=M)
    r.set_params(w0[0])
    xs = torch.from_numpy(np.ascontiguousarray(X[:, rank * half:(rank + 1) * half])).to(dev)
    ys = torch.from_numpy(np.ascontiguousarray(Y[:, rank * half:(rank + 1) * half])).to(dev)
    losses = r.run(xs, ys, want_losses=True)
    W, V, ver = r.get_params()
    np.savez(os.path.join(outdir, f"r{rank}.npz"), W=W, losses=losses, ver=ver)
    r.close()
    dist.destroy_process_group()


def test_data_parallel_two_replicas_equal_global_batch():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        r0, r1 = np.load(os.path.join(d, "r0.npz")), np.load(os.path.join(d, "r1.npz"))
    model = sd.mlp(MODEL["widths"], cuts=[])
    w0, X, Y = sd.parity_inputs(model, M, B, seed=11)
    ref = oracle_run(model, w0, X, Y, LR)
    assert int(r0["ver"]) == int(r1["ver"]) == M
    np.testing.assert_array_equal(r0["W"], r1["W"])  # replicas stay identical
    assert rel_l2(r0["W"], ref.W[0]) <= 1e-4
    assert rel_l2(0.5 * (r0["losses"] + r1["losses"]), ref.losses) <= 1e-4
    assert rel_l2(ref.W[0], np.concatenate(sd.widen(w0))) > 1e-4
