"""The P2P transport: inter-stage transfer fused into the
producing kernels over peer memory — the last forward GEMM of stage k writes stage
k+1's stash slot, the layer-0 dX GEMM of stage k+1 writes stage k's gradient ring,
flags in the waiter's memory hand the buffers over (paper_1809_02839_b200/csrc/p2p.cu).

On the one GPU of this box the stages run as separate processes (torch.multiprocessing,
gloo only to exchange the descriptors) whose buffers are opened with CUDA IPC — the
code path a one-stage-per-GPU run takes over NVLink / NVSwitch. Results must match the
oracle like every other transport (trace bit-exact, W and loss within 1e-4) and the
LOCAL transport bit for bit (same kernels, same order).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synthdata as sd
from tests.gpu_helpers import build_pipeline, layers_of, oracle_run, rel_l2

pytestmark = pytest.mark.gpu


def test_p2p_refuses_same_process_same_gpu():
    """Stage contexts of ONE process on one GPU share its hardware work queues (streams
    are multiplexed onto a few channels): a spinning wait kernel could sit ahead of the
    very kernels it waits for. st_p2p_connect refuses that arrangement; P2P stages that
    share a GPU run as separate processes (below)."""
    import paper_1809_02839_b200 as st
    model = sd.mlp([784, 256, 256, 10], cuts=[1])
    stages = [st.Stage(layers_of(model), model.cuts, k, 32, 0.05, 0.9, transport=st.ST_TRANSPORT_P2P, device=0,
                       max_minibatches=4) for k in range(2)]
    try:
        with pytest.raises(st.SpecTrainError, match="separate"):
            st.connect_p2p_local(stages)
    finally:
        for s in stages:
            s.close()


# ---------------------------------------------------------------- one process per stage (CUDA IPC)
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _model(name, N):
    if name == "mlp":
        return sd.mlp([784, 256, 256, 10], cuts=[1] if N == 2 else sd.even_cuts(3, N))
    if name == "ragged":
        return sd.mlp([100, 72, 200, 40, 10], cuts=[1, 2, 3])
    if name == "lstm":
        return sd.lstm_lm(vocab=48, hidden=32, layers=2, cuts=[1, 3], seq_len=4)
    return sd.config_deep_mlp(N)


def _inputs(model, M, B, seed=0):
    """Seeded parity inputs: images for the MLPs, tokens for the LM (as tests/test_gpu_lstm.py)."""
    if model.layers[0].kind == sd.EMBED:
        w0 = sd.to_f32_params(sd.glorot_params(model, seed))
        X, Y = sd.tokens(model.layers[0].n_in, M, B, model.seq_len, seed + 1)
        return w0, X, Y
    return sd.parity_inputs(model, M, B, seed=seed)


def _worker(rank, world, port, model_name, M, B, lr, out_dir, hang_rank, timeout_s, sessions=1):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["ST_COMM_TIMEOUT_S"] = str(timeout_s)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1809_02839_b200 as st
    model = _model(model_name, world)
    w0, X, Y = _inputs(model, M, B)
    torch.cuda.set_device(0)
    s = st.Stage(layers_of(model), model.cuts, rank, B, lr, 0.9, transport=st.ST_TRANSPORT_P2P, device=0,
                 max_minibatches=M, seq_len=model.seq_len)
    st.connect_p2p(s)  # descriptors all-gathered over gloo, peers opened with CUDA IPC
    if os.environ.get("P2P_DEBUG"):
        import struct
        d = st.p2p_export(s)
        print(f"rank {rank} desc", struct.unpack_from("<IIiiiiqqqiiqqq", d), "X", X.dtype, X.shape, X.min(), X.max(),
              flush=True)
    s.set_params(w0[rank])
    dev = torch.device("cuda", 0)
    xs = torch.from_numpy(np.ascontiguousarray(X, np.int32 if X.dtype.kind in "iu" else np.float32)).to(dev)
    ys = torch.from_numpy(np.ascontiguousarray(Y, np.int32)).to(dev)
    dist.barrier()
    try:
        if hang_rank >= 0:
            # session 1 on every rank (every kernel gets loaded: with CUDA's lazy module
            # loading the first launch of a kernel waits for the device, which a spin-wait
            # on a dead peer would block before any timeout applies), then the peer hangs
            s.run(2, xs[:2] if s.is_first else None, ys[:2] if s.is_last else None, want_losses=False)
            s.sync()
            dist.barrier()
            if rank == hang_rank:
                import time
                time.sleep(3 * timeout_s)  # alive, never runs again: its peers' wait kernels spin
                os._exit(0)
        cuts_ = [M] if sessions == 1 else [M // 2, M]  # session boundaries (mini-batch counts)
        parts, lo = [], 0
        for hi in cuts_:
            part = s.run(hi - lo, xs[lo:hi] if s.is_first else None, ys[lo:hi] if s.is_last else None,
                         want_losses=s.is_last)
            parts.append(part)
            lo = hi
        losses = np.concatenate(parts) if s.is_last else None
        s.sync()
        W, V, ver = s.get_params()
        np.save(os.path.join(out_dir, f"W{rank}.npy"), W)
        np.save(os.path.join(out_dir, f"trace{rank}.npy"), np.array(s.trace(), np.int64))
        if losses is not None:
            np.save(os.path.join(out_dir, "losses.npy"), losses)
        np.save(os.path.join(out_dir, f"status{rank}.npy"), np.array([0]))
    except st.SpecTrainError as e:
        np.save(os.path.join(out_dir, f"status{rank}.npy"), np.array([e.status]))
        with open(os.path.join(out_dir, f"err{rank}.txt"), "w") as f:
            f.write(str(e))
        os._exit(0)
    dist.barrier()  # peers may still read this rank's buffers until every rank is done
    s.close()
    dist.destroy_process_group()


def _spawn(world, model_name, M, B, lr, tmp_path, hang_rank=-1, timeout_s=600, sessions=1):
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, model_name, M, B, lr, str(tmp_path), hang_rank,
                                                 timeout_s, sessions)) for r in range(world)]
    for p in procs:
        p.start()
    hung = []
    for p in procs:
        p.join(max(120, 4 * timeout_s) if hang_rank >= 0 else 600)
        if p.is_alive():
            hung.append(p.pid)
            p.kill()
            p.join(10)
    assert not hung, f"stage process(es) {hung} hung (killed)"
    return [p.exitcode for p in procs]


@pytest.mark.parametrize("world,model_name,M,B,lr", [(2, "mlp", 20, 32, 0.05), (3, "deep", 12, 64, 0.02),
                                                     (4, "ragged", 9, 24, 0.05), (3, "lstm", 6, 8, 0.1)],
                         ids=["mlp2", "deep3", "ragged4", "lstm3"])
def test_p2p_ipc_processes_match_oracle(tmp_path, world, model_name, M, B, lr):
    codes = _spawn(world, model_name, M, B, lr, tmp_path)
    assert all(c == 0 for c in codes), codes
    model = _model(model_name, world)
    w0, X, Y = _inputs(model, M, B)
    ref = oracle_run(model, w0, X, Y, lr)
    for k in range(world):
        assert int(np.load(tmp_path / f"status{k}.npy")[0]) == 0
        tr = [tuple(int(v) for v in row) for row in np.load(tmp_path / f"trace{k}.npy")]
        assert tr == [e.as_tuple() for e in ref.trace[k]], f"trace mismatch at stage {k}"
    W = np.concatenate([np.load(tmp_path / f"W{k}.npy") for k in range(world)])
    losses = np.load(tmp_path / "losses.npy")
    assert rel_l2(W, np.concatenate(ref.W)) <= 1e-4
    assert rel_l2(losses, ref.losses) <= 1e-4


def test_p2p_two_sessions_bitwise_equal_local(tmp_path):
    """Sessions restart the mini-batch numbering; the flags keep increasing (base =
    backwards done before the session). Two sessions through P2P processes equal the
    same two sessions through the LOCAL transport (this process) bit for bit."""
    import paper_1809_02839_b200 as st
    world, M, B, lr = 3, 12, 32, 0.02
    codes = _spawn(world, "deep", M, B, lr, tmp_path, sessions=2)
    assert all(c == 0 for c in codes), codes
    model = _model("deep", world)
    w0, X, Y = sd.parity_inputs(model, M, B, seed=0)
    stages = build_pipeline(model, B, lr)
    try:
        for s, w in zip(stages, w0):
            s.set_params(w)
        dev = torch.device("cuda", 0)
        xs = torch.from_numpy(np.ascontiguousarray(X, np.float32)).to(dev)
        ys = torch.from_numpy(np.ascontiguousarray(Y, np.int32)).to(dev)
        l1 = st.run_group(stages, M // 2, xs[:M // 2], ys[:M // 2])
        l2 = st.run_group(stages, M - M // 2, xs[M // 2:], ys[M // 2:])
        Wl = [s.get_params()[0] for s in stages]
    finally:
        for s in stages:
            s.close()
    assert np.array_equal(np.load(tmp_path / "losses.npy"), np.concatenate([l1, l2]))
    for k in range(world):
        assert np.array_equal(np.load(tmp_path / f"W{k}.npy"), Wl[k]), f"stage {k}"


def test_p2p_hung_peer_releases_waiters(tmp_path):
    """A stage whose peer never runs: its wait kernels spin until the engine's wait
    loop times out (ST_COMM_TIMEOUT_S), which raises the host-mapped abort word —
    the run returns ST_ERR_STATE instead of hanging."""
    import paper_1809_02839_b200 as st
    codes = _spawn(2, "mlp", 6, 32, 0.05, tmp_path, hang_rank=1, timeout_s=5)
    assert all(c == 0 for c in codes), codes
    assert int(np.load(tmp_path / "status0.npy")[0]) == 3  # ST_ERR_STATE
    assert "hung" in (tmp_path / "err0.txt").read_text()
