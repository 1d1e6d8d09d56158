"""Hybrid data × pipeline parallelism on CPU, multi-process
(gloo, -m "not gpu"): the protocol the engine implements for `st_config.replicas`
(engine.cpp move / transport.cpp), with the oracle's arithmetic.

Ranks are stage-major contexts: rank(k, r) = Σ_{j<k} replicas[j] + r. Every context runs
the library's 1F1B program (`st_program`) and comm plan (`st_comm_plan`) of its stage.
A replicated stage computes its row slice [r·B/R, (r+1)·B/R) of every mini-batch; a
message between a replicated stage and its (unreplicated) neighbour becomes one
transfer per replica, row slice r to / from replica r; the replicas SUM their gradients
(all-reduce over the stage's replica group, reading D25) before the identical update.
Each direction's transfers run on their own comm thread in plan order (blocking gloo
send / recv), as in tests/test_gloo_pipeline.py. The result must equal the unreplicated
single-process oracle run (to fp64 rounding: the gradient sums over row slices in a
different order) on every replica, and no rank may block forever."""
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


def _worker(rank, world, port, reps, widths, M, B, eta, gamma, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1809_02839_b200 as st
        N = len(reps)
        base = np.concatenate([[0], np.cumsum(reps)]).astype(int)
        k = int(np.searchsorted(base, rank, side="right") - 1)
        r = rank - int(base[k])
        R = reps[k]
        model = sd.mlp(widths, cuts=sd.even_cuts(len(widths) - 1, N))
        w0 = sd.glorot_params(model, 7)
        X, Y = sd.images_and_labels(widths[0], widths[-1], M, B, seed=8)
        layers = model.stage_layers(k)
        events = st.program(N, k, M)
        prog = [(e[2], e[3]) for e in events]
        plan = st.comm_plan(N, k, M)
        groups = [dist.new_group(list(range(world))), dist.new_group(list(range(world)))]
        rep_groups = {s: dist.new_group([int(base[s]) + j for j in range(reps[s])]) for s in range(N) if reps[s] > 1}
        rows = slice(r * B // R, (r + 1) * B // R)  # this context's rows (all of them if unreplicated)
        W = np.array(w0[k], dtype=np.float64)
        V = np.zeros_like(W)
        d_in, d_out = layers[0].n_in, layers[-1].n_out
        produced, outbox, arrived, inbox, errors = {}, {}, {}, {}, []
        for _, ops in plan:
            for kind, mb in ops:
                (produced if kind in (SEND_FWD, SEND_BWD) else arrived)[(kind, mb)] = threading.Event()

        def peers(kind):
            """(rank, row slice of the message) per transfer of one message of `kind`."""
            ps = k + 1 if kind in (SEND_FWD, RECV_BWD) else k - 1
            if reps[ps] > 1:  # the neighbour is replicated: one slice per replica
                n = reps[ps]
                return [(int(base[ps]) + j, slice(j * B // n, (j + 1) * B // n)) for j in range(n)]
            return [(int(base[ps]), slice(0, B // R))]  # one transfer of this context's rows

        def comm_thread(direction):
            try:
                g = groups[direction]
                for _, ops in plan:
                    for kind, mb in ops:
                        if (kind in (SEND_FWD, RECV_FWD)) != (direction == 0):
                            continue
                        if kind in (SEND_FWD, SEND_BWD):
                            assert produced[(kind, mb)].wait(60), ("send never produced", kind, mb)
                            msg = outbox.pop((kind, mb))
                            for peer, sl in peers(kind):
                                dist.send(torch.from_numpy(np.ascontiguousarray(msg[sl])), peer, group=g)
                        else:
                            width = d_in if kind == RECV_FWD else d_out
                            buf = np.empty((B // R, width))
                            for peer, sl in peers(kind):
                                t = torch.empty(sl.stop - sl.start, width, dtype=torch.float64)
                                dist.recv(t, peer, group=g)
                                buf[sl] = t.numpy()
                            inbox[(kind, mb)] = buf
                            arrived[(kind, mb)].set()
            except Exception as e:  # surfaced by the main thread
                errors.append(e)

        threads = [threading.Thread(target=comm_thread, args=(d,), daemon=True) for d in (0, 1)]
        for t in threads:
            t.start()
        losses, stash, dlog = {}, {}, {}
        for d, i in prog:
            s = O.version_difference(k, N, d)
            W_hat = O.predict(W, V, s, eta)
            if d == O.FWD:
                if k > 0:
                    assert arrived[(RECV_FWD, i)].wait(60), ("activation never arrived", i)
                a = X[i][rows] if k == 0 else inbox.pop((RECV_FWD, i))
                out, stash[i] = O.stage_forward(layers, W_hat, a)
                if k == N - 1:
                    losses[i], dlog[i] = O.loss_and_grad("softmax_ce", out, Y[i])
                else:
                    outbox[(SEND_FWD, i)] = out
                    produced[(SEND_FWD, i)].set()
            else:
                if k < N - 1:
                    assert arrived[(RECV_BWD, i)].wait(60), ("gradient never arrived", i)
                dA = dlog.pop(i) if k == N - 1 else inbox.pop((RECV_BWD, i))
                g, dA_in = O.stage_backward(layers, W_hat, stash.pop(i), dA, need_dA_in=k > 0)
                if k > 0:
                    outbox[(SEND_BWD, i)] = dA_in
                    produced[(SEND_BWD, i)].set()
                if R > 1:  # D25: the replicas' row-slice gradients sum to the stage's gradient
                    tg = torch.from_numpy(g)
                    dist.all_reduce(tg, op=dist.ReduceOp.SUM, group=rep_groups[k])
                    g = tg.numpy()
                V = O.update_smoothed(V, g, gamma)
                W = W - eta * V
        for t in threads:
            t.join(60)
            assert not t.is_alive(), "comm thread hung"
        assert not errors, errors
        assert not outbox and not inbox
        ref = O.run(model, w0, X, Y, eta, gamma)
        np.testing.assert_allclose(W, ref.W[k], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(V, ref.V[k], rtol=1e-10, atol=1e-15)
        if k == N - 1:
            np.testing.assert_allclose(np.array([losses[i] for i in range(M)]), ref.losses, rtol=1e-12)
        open(os.path.join(result_dir, f"ok{rank}"), "w").write("ok")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("reps,M", [([2, 1], 6), ([2, 1, 1], 5), ([1, 2, 1], 5), ([2, 1, 2, 1], 6)], ids=str)
def test_gloo_hybrid_matches_oracle(tmp_path, reps, M):
    widths = [20, 16, 12, 8, 5]
    world = sum(reps)
    port = _free_port()
    mp.spawn(_worker, args=(world, port, reps, widths, M, 8, 0.05, 0.9, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert (tmp_path / f"ok{r}").exists()
