"""The NCCL transport executed for real: N processes, one
stage each, ST_TRANSPORT_NCCL, two communicators, comm streams — on ONE GPU.

NCCL refuses two ranks of a communicator on the same device ("Duplicate GPU"),
unless they look like different hosts: each rank gets its own NCCL_HOSTID, so the
ranks talk through NCCL's socket transport over loopback (GPU → host → socket). The
data path is slower than NVLink but the library code is the one a multi-GPU run
executes: the same communicators, comm streams, events, plan order and async-error
handling. Results must match the oracle exactly like the LOCAL-transport tests."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synthdata as sd
from tests.gpu_helpers import layers_of, oracle_run, rel_l2

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _nccl_env(rank: int):
    os.environ["NCCL_HOSTID"] = f"spectrain-test-host-{rank}"  # distinct "hosts" on one GPU
    os.environ["NCCL_SOCKET_IFNAME"] = "lo"
    os.environ["NCCL_IB_DISABLE"] = "1"
    os.environ.setdefault("NCCL_DEBUG", "WARN")


def _worker(rank, world, port, model_name, M, B, lr, out_dir, fail_rank, timeout_s):
    import faulthandler
    # diagnostics only: a stuck stage prints its Python stack (the parent kills it)
    faulthandler.dump_traceback_later(timeout_s + 60 if fail_rank >= 0 else 500, exit=False)
    _nccl_env(rank)
    os.environ["ST_COMM_TIMEOUT_S"] = str(timeout_s)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1809_02839_b200 as st
        model = _model(model_name, world)
        w0, X, Y = sd.parity_inputs(model, M, B, seed=0)
        obj = [st.nccl_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        torch.cuda.set_device(0)
        s = st.Stage(layers_of(model), model.cuts, rank, B, lr, 0.9, transport=st.ST_TRANSPORT_NCCL, device=0,
                     max_minibatches=M, nccl_id=obj[0])
        if os.environ.get("ST_TEST_GRAPH") == "1":
            s.set_graph_mode(True)  # the session (NCCL calls included) as one captured CUDA graph
        s.set_params(w0[rank])
        dev = torch.device("cuda", 0)
        xs = torch.from_numpy(np.ascontiguousarray(X, np.float32)).to(dev)
        ys = torch.from_numpy(np.ascontiguousarray(Y, np.int32)).to(dev)
        if fail_rank >= 0:
            # session 1 on both ranks (the communicators connect), then the peer hangs:
            # it stays alive but never posts another transfer
            s.run(2, xs if s.is_first else None, ys if s.is_last else None, want_losses=False)
            s.sync()
            if rank == fail_rank:
                import time
                time.sleep(3 * timeout_s)
                os._exit(0)
        try:
            losses = s.run(M, xs if s.is_first else None, ys if s.is_last else None, want_losses=s.is_last)
            W, V, ver = s.get_params()
            np.save(os.path.join(out_dir, f"W{rank}.npy"), W)
            np.save(os.path.join(out_dir, f"V{rank}.npy"), V)
            np.save(os.path.join(out_dir, f"trace{rank}.npy"), np.array(s.trace(), np.int64))
            if losses is not None:
                np.save(os.path.join(out_dir, "losses.npy"), losses)
            np.save(os.path.join(out_dir, f"status{rank}.npy"), np.array([0]))
        except st.SpecTrainError as e:
            np.save(os.path.join(out_dir, f"status{rank}.npy"), np.array([e.status]))
            with open(os.path.join(out_dir, f"err{rank}.txt"), "w") as f:
                f.write(str(e))
            os._exit(0)  # the communicators were aborted: skip the collective teardown
        s.close()
    finally:
        dist.destroy_process_group()


def _model(name, N):
    if name == "mlp":
        return sd.mlp([784, 256, 256, 10], cuts=[1] if N == 2 else sd.even_cuts(3, N))
    return sd.config_deep_mlp(N)


def _spawn(world, model_name, M, B, lr, tmp_path, fail_rank=-1, timeout_s=600):
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, model_name, M, B, lr, str(tmp_path), fail_rank,
                                                 timeout_s)) for r in range(world)]
    for p in procs:
        p.start()
    hung = []
    for p in procs:
        p.join(max(120, 4 * timeout_s) if fail_rank >= 0 else 600)
        if p.is_alive():
            hung.append(p.pid)
            p.kill()
            p.join(10)
    assert not hung, f"stage process(es) {hung} hung (killed)"
    return [p.exitcode for p in procs]


@pytest.mark.parametrize("world,model_name,M,B,lr", [(2, "mlp", 20, 32, 0.05), (3, "deep", 12, 64, 0.02)])
def test_nccl_pipeline_matches_oracle(tmp_path, world, model_name, M, B, lr):
    codes = _spawn(world, model_name, M, B, lr, tmp_path)
    assert all(c == 0 for c in codes), codes
    model = _model(model_name, world)
    w0, X, Y = sd.parity_inputs(model, M, B, seed=0)
    ref = oracle_run(model, w0, X, Y, lr)
    for k in range(world):
        assert int(np.load(tmp_path / f"status{k}.npy")[0]) == 0
        trace = [tuple(int(v) for v in e) for e in np.load(tmp_path / f"trace{k}.npy")]
        assert trace == [e.as_tuple() for e in ref.trace[k]], f"trace mismatch at stage {k}"
    W = np.concatenate([np.load(tmp_path / f"W{k}.npy") for k in range(world)])
    rw = rel_l2(W, np.concatenate(ref.W))
    rl = rel_l2(np.load(tmp_path / "losses.npy"), ref.losses)
    dw = rel_l2(W - np.concatenate(w0), np.concatenate(ref.W) - np.concatenate(sd.widen(w0)))
    assert rw <= 1e-4 and rl <= 1e-4 and dw <= 1e-3, (rw, rl, dw)


def test_nccl_hung_peer_surfaces_as_st_err_nccl(tmp_path):
    # after one good session stage 1 hangs (alive, silent); stage 0 must not hang with
    # it: its wait for the gradient times out, both communicators are aborted and
    # ST_ERR_NCCL (5) comes back
    codes = _spawn(2, "mlp", 4, 32, 0.05, tmp_path, fail_rank=1, timeout_s=10)
    assert codes == [0, 0], codes
    assert int(np.load(tmp_path / "status0.npy")[0]) == 5
    assert "hung or gone" in (tmp_path / "err0.txt").read_text()


def test_nccl_pipeline_graph_mode_matches_oracle(tmp_path, monkeypatch):
    """The NCCL pipeline with graph sessions: every stage captures its session — kernels,
    events and the ncclSend / ncclRecv on both comm streams — into one CUDA graph."""
    monkeypatch.setenv("ST_TEST_GRAPH", "1")
    world, model_name, M, B, lr = 2, "mlp", 20, 32, 0.05
    codes = _spawn(world, model_name, M, B, lr, tmp_path)
    assert all(c == 0 for c in codes), codes
    model = _model(model_name, world)
    w0, X, Y = sd.parity_inputs(model, M, B, seed=0)
    ref = oracle_run(model, w0, X, Y, lr)
    for k in range(world):
        tr = [tuple(int(v) for v in row) for row in np.load(tmp_path / f"trace{k}.npy")]
        assert tr == [e.as_tuple() for e in ref.trace[k]]
    W = np.concatenate([np.load(tmp_path / f"W{k}.npy") for k in range(world)])
    assert rel_l2(W, np.concatenate(ref.W)) <= 1e-4
    assert rel_l2(np.load(tmp_path / "losses.npy"), ref.losses) <= 1e-4
