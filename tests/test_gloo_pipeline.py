"""Multi-process check of the N>1 communication path on CPU (gloo, -m "not gpu").

Each rank plays one pipeline stage. The task order and the grouped send/recv
sequence come from the native library (`st_program` / `st_comm_plan` — the same
host code the CUDA engine executes); the stage arithmetic comes from the oracle;
messages travel through real torch.distributed point-to-point ops (gloo), every
group's ops posted together and then waited on. The result must equal the
single-process oracle run bit for bit, and no rank may block forever."""
import os
import socket

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
        W = np.array(w0[k], dtype=np.float64)
        V = np.zeros_like(W)
        act_in, grad_in, out_act, out_grad, stash, dlog = {}, {}, {}, {}, {}, {}
        losses = {}
        d_in = layers[0].n_in
        d_out = layers[-1].n_out
        gi = 0

        def run_groups(upto):
            nonlocal gi
            while gi < len(plan) and plan[gi][0] <= upto:
                reqs, bufs = [], []
                for kind, mb in plan[gi][1]:
                    if kind == SEND_FWD:
                        reqs.append(dist.isend(torch.from_numpy(out_act.pop(mb)), k + 1))
                    elif kind == SEND_BWD:
                        reqs.append(dist.isend(torch.from_numpy(out_grad.pop(mb)), k - 1))
                    elif kind == RECV_FWD:
                        t = torch.empty(B, d_in, dtype=torch.float64)
                        reqs.append(dist.irecv(t, k - 1))
                        bufs.append((act_in, mb, t))
                    else:
                        t = torch.empty(B, d_out, dtype=torch.float64)
                        reqs.append(dist.irecv(t, k + 1))
                        bufs.append((grad_in, mb, t))
                for r in reqs:
                    r.wait()
                for d, mb, t in bufs:
                    d[mb] = t.numpy()
                gi += 1

        version = 0
        for n, (d, i) in enumerate(prog):
            run_groups(n)  # receives this task needs (and sends of the previous task)
            s = O.version_difference(k, N, d)
            assert events[n][4] == version and events[n][5] == s
            W_hat = O.predict(W, V, s, eta)
            if d == O.FWD:
                a = X[i] if k == 0 else act_in.pop(i)
                out, stash[i] = O.stage_forward(layers, W_hat, a)
                if k == N - 1:
                    losses[i], dlog[i] = O.loss_and_grad("softmax_ce", out, Y[i])
                else:
                    out_act[i] = np.ascontiguousarray(out)
            else:
                dA = dlog.pop(i) if k == N - 1 else grad_in.pop(i)
                g, dA_in = O.stage_backward(layers, W_hat, stash.pop(i), dA, need_dA_in=k > 0)
                if k > 0:
                    out_grad[i] = np.ascontiguousarray(dA_in)
                V = O.update_smoothed(V, g, gamma)
                W = W - eta * V
                version += 1
        run_groups(len(prog))
        assert gi == len(plan) and not out_act and not out_grad
        ref = O.run(model, w0, X, Y, eta, gamma)
        np.testing.assert_array_equal(W, ref.W[k])
        np.testing.assert_array_equal(V, ref.V[k])
        if k == N - 1:
            np.testing.assert_array_equal(np.array([losses[i] for i in range(M)]), ref.losses)
        open(os.path.join(result_dir, f"ok{rank}"), "w").write("ok")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,M", [(2, 7), (2, 1), (3, 5)])
def test_gloo_pipeline_matches_oracle(tmp_path, world, M):
    widths = [20, 16, 12, 8, 5]
    port = _free_port()
    mp.spawn(_stage_worker, args=(world, port, widths, M, 4, 0.05, 0.9, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert (tmp_path / f"ok{r}").exists()
