"""Hybrid data × pipeline parallelism ("we combine pipeline
with data parallelism and adopt data parallelism in the first stage to mitigate the
imbalance between pipeline stages").

A replicated stage splits each mini-batch by rows across its replicas, which sum their
gradients before the identical K-B update (reading D25) — so the hybrid pipeline
computes what the unreplicated one computes: the oracle's plain SpecTrain run is the
reference (trace bit-exact per replica, W and loss within 1e-4). Co-located replicas
(LOCAL transport, in-place reduce across the replica contexts) and one process per
replica (NCCL transport, flattened stage-major ranks, ncclAllReduce over the replica
communicator; on one GPU through NCCL_HOSTID like tests/test_gpu_nccl.py).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synthdata as sd
from tests.gpu_helpers import layers_of, oracle_run, rel_l2

pytestmark = pytest.mark.gpu


def _hybrid_local(model, reps, B, lr, M):
    import paper_1809_02839_b200 as st
    ctxs = []
    for k in range(model.num_stages):
        for r in range(reps[k]):
            ctxs.append(st.Stage(layers_of(model), model.cuts, k, B, lr, 0.9, transport=st.ST_TRANSPORT_LOCAL,
                                 device=0, max_minibatches=M, seq_len=model.seq_len, replicas=reps, replica=r))
    st.connect_local(ctxs)
    return ctxs


def _check(model, reps, ctxs, w0, X, Y, lr):
    import paper_1809_02839_b200 as st
    for s in ctxs:
        s.set_params(w0[s.k])
    dev = torch.device("cuda", 0)
    xs = torch.from_numpy(np.ascontiguousarray(X, np.float32)).to(dev)
    ys = torch.from_numpy(np.ascontiguousarray(Y, np.int32)).to(dev)
    losses = st.run_group(ctxs, X.shape[0], xs, ys, want_losses=True)
    ref = oracle_run(model, w0, X, Y, lr)
    Ws = {}
    for s in ctxs:
        assert s.trace() == [e.as_tuple() for e in ref.trace[s.k]], f"trace mismatch at stage {s.k} replica {s.replica}"
        W = s.get_params()[0]
        if s.k in Ws:  # replicas stay bit-identical (same summed gradient, same update)
            assert np.array_equal(W, Ws[s.k]), f"replicas of stage {s.k} diverged"
        Ws[s.k] = W
    W = np.concatenate([Ws[k] for k in range(model.num_stages)])
    rw = rel_l2(W, np.concatenate(ref.W))
    rl = rel_l2(losses, ref.losses)
    assert rw <= 1e-4 and rl <= 1e-4, (rw, rl)
    return rw, rl


@pytest.mark.parametrize("reps", [[2, 1, 1], [1, 2, 1], [4, 1, 1], [2, 1, 2, 1]], ids=str)
def test_hybrid_local_matches_oracle(reps):
    model = sd.mlp([784, 256, 192, 128, 10], cuts=[1, 2, 3] if len(reps) == 4 else [1, 3])
    M, B, lr = 10, 32, 0.05
    w0, X, Y = sd.parity_inputs(model, M, B, seed=1)
    ctxs = _hybrid_local(model, reps, B, lr, M)
    try:
        _check(model, reps, ctxs, w0, X, Y, lr)
    finally:
        for s in ctxs:
            s.close()


def test_hybrid_vgg_first_stage_replicated():
    """The paper's case: the conv front of a VGG is the bottleneck stage."""
    model = sd.vgg(cfg=(32, "M", 32, "M"), fc=(64,), classes=10, hw=8, cuts=[3, 5])
    reps = [2, 1, 1]
    M, B, lr = 6, 16, 0.02
    w0, X, Y = sd.parity_inputs(model, M, B, seed=3)
    ctxs = _hybrid_local(model, reps, B, lr, M)
    try:
        _check(model, reps, ctxs, w0, X, Y, lr)
    finally:
        for s in ctxs:
            s.close()


# ---------------------------------------------------------------- NCCL: one process per replica
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, reps, M, B, lr, out_dir):
    os.environ["NCCL_HOSTID"] = f"spectrain-hybrid-host-{rank}"  # distinct "hosts" on one GPU
    os.environ["NCCL_SOCKET_IFNAME"] = "lo"
    os.environ["NCCL_IB_DISABLE"] = "1"
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1809_02839_b200 as st
    model = sd.mlp([784, 256, 128, 10], cuts=[1, 2])
    w0, X, Y = sd.parity_inputs(model, M, B, seed=0)
    base = np.cumsum([0] + list(reps))
    k = int(np.searchsorted(base, rank, side="right") - 1)
    r = rank - int(base[k])
    obj = [st.nccl_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    torch.cuda.set_device(0)
    s = st.Stage(layers_of(model), model.cuts, k, B, lr, 0.9, transport=st.ST_TRANSPORT_NCCL, device=0,
                 max_minibatches=M, nccl_id=obj[0], replicas=reps, replica=r)
    s.set_params(w0[k])
    dev = torch.device("cuda", 0)
    xs = torch.from_numpy(np.ascontiguousarray(X, np.float32)).to(dev)
    ys = torch.from_numpy(np.ascontiguousarray(Y, np.int32)).to(dev)
    losses = s.run(M, xs if s.is_first else None, ys if s.is_last else None, want_losses=s.is_last)
    s.sync()
    np.save(os.path.join(out_dir, f"W{rank}.npy"), s.get_params()[0])
    np.save(os.path.join(out_dir, f"trace{rank}.npy"), np.array(s.trace(), np.int64))
    np.save(os.path.join(out_dir, f"ks{rank}.npy"), np.array([k, r]))
    if losses is not None:
        np.save(os.path.join(out_dir, "losses.npy"), losses)
    s.close()
    dist.destroy_process_group()


def test_hybrid_nccl_processes_match_oracle(tmp_path):
    reps = [2, 1, 1]
    world = sum(reps)
    M, B, lr = 10, 32, 0.05
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, reps, M, B, lr, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    hung = []
    for p in procs:
        p.join(600)
        if p.is_alive():
            hung.append(p.pid)
            p.kill()
            p.join(10)
    assert not hung, f"process(es) {hung} hung (killed)"
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    model = sd.mlp([784, 256, 128, 10], cuts=[1, 2])
    w0, X, Y = sd.parity_inputs(model, M, B, seed=0)
    ref = oracle_run(model, w0, X, Y, lr)
    Ws = {}
    for rank in range(world):
        k, r = [int(v) for v in np.load(tmp_path / f"ks{rank}.npy")]
        tr = [tuple(int(v) for v in row) for row in np.load(tmp_path / f"trace{rank}.npy")]
        assert tr == [e.as_tuple() for e in ref.trace[k]], f"trace mismatch at stage {k} replica {r}"
        W = np.load(tmp_path / f"W{rank}.npy")
        if k in Ws:
            assert np.array_equal(W, Ws[k])
        Ws[k] = W
    W = np.concatenate([Ws[k] for k in range(3)])
    assert rel_l2(W, np.concatenate(ref.W)) <= 1e-4
    assert rel_l2(np.load(tmp_path / "losses.npy"), ref.losses) <= 1e-4
