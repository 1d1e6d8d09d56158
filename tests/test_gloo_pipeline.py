"""Multi-process check of the N>1 communication path on CPU (gloo, -m "not gpu").

Each rank plays one pipeline stage. The task order and the communication plan come
from the native library (`st_program` / `st_comm_plan` — the same host code the CUDA
engine executes); the stage arithmetic comes from the oracle. As in the engine
(engine.cpp issue_op), each direction has its own process group (communicator) and
its own comm thread (stream) that executes that direction's ops in plan order with
real blocking point-to-point transfers (gloo); sends wait until the compute thread
produced the message, the compute thread waits for received messages. The result
must equal the single-process oracle run bit for bit, and no rank may block forever."""
import os
import socket
import threading

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synthdata as sd
from oracle import spectrain_oracle as O

SEND_FWD, RECV_FWD, SEND_BWD, RECV_BWD = 0, 1, 2, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _stage_worker(rank, world, port, widths, M, B, eta, gamma, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1809_02839_b200 as st
        N, k = world, rank
        model = sd.mlp(widths, cuts=sd.even_cuts(len(widths) - 1, N))
        w0 = sd.glorot_params(model, 7)
        X, Y = sd.images_and_labels(widths[0], widths[-1], M, B, seed=8)
        layers = model.stage_layers(k)
        events = st.program(N, k, M)
        prog = [(e[2], e[3]) for e in events]
        assert prog == O.stage_program(N, k, M)
        plan = st.comm_plan(N, k, M)
        groups = [dist.new_group(list(range(world))), dist.new_group(list(range(world)))]  # activations, gradients
        W = np.array(w0[k], dtype=np.float64)
        V = np.zeros_like(W)
        d_in = layers[0].n_in
        d_out = layers[-1].n_out
        # message boxes between the compute thread and the two comm threads
        produced = {}  # (kind, mb) -> threading.Event set by compute when the send buffer is ready
        outbox = {}
        arrived = {}   # (kind, mb) -> threading.Event set by a comm thread when a receive landed
        inbox = {}
        errors = []
        for _, ops in plan:
            for kind, mb in ops:
                (produced if kind in (SEND_FWD, SEND_BWD) else arrived)[(kind, mb)] = threading.Event()

        def comm_thread(direction):
            try:
                g = groups[direction]
                for _, ops in plan:
                    for kind, mb in ops:
                        if (kind in (SEND_FWD, RECV_FWD)) != (direction == 0):
                            continue
                        if kind in (SEND_FWD, SEND_BWD):
                            assert produced[(kind, mb)].wait(60), ("send never produced", kind, mb)
                            dist.send(torch.from_numpy(outbox.pop((kind, mb))), k + 1 if kind == SEND_FWD else k - 1,
                                      group=g)
                        else:
                            t = torch.empty(B, d_in if kind == RECV_FWD else d_out, dtype=torch.float64)
                            dist.recv(t, k - 1 if kind == RECV_FWD else k + 1, group=g)
                            inbox[(kind, mb)] = t.numpy()
                            arrived[(kind, mb)].set()
            except Exception as e:  # surfaced by the main thread
                errors.append(e)

        threads = [threading.Thread(target=comm_thread, args=(d,), daemon=True) for d in (0, 1)]
        for t in threads:
            t.start()
        losses, stash, dlog = {}, {}, {}
        version = 0
        for n, (d, i) in enumerate(prog):
            s = O.version_difference(k, N, d)
            assert events[n][4] == version and events[n][5] == s
            W_hat = O.predict(W, V, s, eta)
            if d == O.FWD:
                if k > 0:
                    assert arrived[(RECV_FWD, i)].wait(60), ("activation never arrived", i)
                a = X[i] if k == 0 else inbox.pop((RECV_FWD, i))
                out, stash[i] = O.stage_forward(layers, W_hat, a)
                if k == N - 1:
                    losses[i], dlog[i] = O.loss_and_grad("softmax_ce", out, Y[i])
                else:
                    outbox[(SEND_FWD, i)] = np.ascontiguousarray(out)
                    produced[(SEND_FWD, i)].set()
            else:
                if k < N - 1:
                    assert arrived[(RECV_BWD, i)].wait(60), ("gradient never arrived", i)
                dA = dlog.pop(i) if k == N - 1 else inbox.pop((RECV_BWD, i))
                g, dA_in = O.stage_backward(layers, W_hat, stash.pop(i), dA, need_dA_in=k > 0)
                if k > 0:
                    outbox[(SEND_BWD, i)] = np.ascontiguousarray(dA_in)
                    produced[(SEND_BWD, i)].set()
                V = O.update_smoothed(V, g, gamma)
                W = W - eta * V
                version += 1
        for t in threads:
            t.join(60)
            assert not t.is_alive(), "comm thread hung"
        assert not errors, errors
        assert not outbox and not inbox
        ref = O.run(model, w0, X, Y, eta, gamma)
        np.testing.assert_array_equal(W, ref.W[k])
        np.testing.assert_array_equal(V, ref.V[k])
        if k == N - 1:
            np.testing.assert_array_equal(np.array([losses[i] for i in range(M)]), ref.losses)
        open(os.path.join(result_dir, f"ok{rank}"), "w").write("ok")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,M", [(2, 7), (2, 1), (3, 5), (4, 6)])
def test_gloo_pipeline_matches_oracle(tmp_path, world, M):
    widths = [20, 16, 12, 8, 5]
    port = _free_port()
    mp.spawn(_stage_worker, args=(world, port, widths, M, 4, 0.05, 0.9, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert (tmp_path / f"ok{r}").exists()
