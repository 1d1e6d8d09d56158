"""Host-side checks of the native library (no GPU): it loads, exports every
symbol include/spectrain.h declares, and its program generator / comm plan match
the oracle bit-exactly and are deadlock-free under strict rendezvous semantics."""
import os
import re

import numpy as np
import pytest

import synthdata as sd
from oracle import spectrain_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def st():
    import paper_1809_02839_b200 as st
    return st


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "spectrain.h")).read()
    return sorted(set(re.findall(r"^ST_API[^(]*?\b(st_\w+)\(", txt, flags=re.M)))


def test_library_exports_every_header_symbol(st):
    from paper_1809_02839_b200 import _lib
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(_lib.lib, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert b"sm_100a" in _lib.lib.st_version()


def test_version_difference_matches_oracle(st):
    for N in range(1, 17):
        for k in range(-1, N + 1):
            for d in (O.FWD, O.BWD):
                assert st.version_difference(k, N, d) == O.version_difference(k, N, d)
    assert st.version_difference(0, 3, 7) == -1


def _oracle_trace(N, M, pred):
    model = sd.mlp([2] * (N + 1), cuts=list(range(1, N)))
    res = O.run(model, sd.glorot_params(model, 0), np.zeros((M, 1, 2)), np.zeros((M, 1), np.int32), 0.01, 0.9,
                pred=pred)
    return res.trace


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 8])
def test_program_bit_exact_vs_oracle(st, N):
    for M in sorted({1, max(1, N - 1), N, 20}):
        for pred, cpred in ((O.PRED_SPECTRAIN, st.ST_PRED_SPECTRAIN), (O.PRED_NONE, st.ST_PRED_NONE),
                            (O.PRED_STASH, st.ST_PRED_STASH), (O.PRED_STALENESS_FREE, st.ST_PRED_STALENESS_FREE)):
            tr = _oracle_trace(N, M, pred)
            for k in range(N):
                assert st.program(N, k, M, cpred) == [e.as_tuple() for e in tr[k]], (N, M, k, pred)


def simulate_streams(N, M, plans, programs, shared=False):
    """The engine's execution model (engine.cpp issue_op / run_task) under strict
    rendezvous semantics: per stage a compute FIFO (the program) and two comm FIFOs
    (activations: kinds 0/1, gradients: kinds 2/3, each in plan order). A send
    completes together with the matching receive, only when both are at the head of
    their FIFOs and their event dependencies are met:
      send_fwd(i) after F(i); send_bwd(j) after B(j);
      recv_fwd(i) after B(i − S) (its stash slot's previous reader, S = N − k);
      recv_bwd(j) after B(j − 2) (two gradient slots);
      F(i) after recv_fwd(i) and send_fwd(i − 2); B(j) after recv_bwd(j) and send_bwd(j − 2).
    shared=True puts both directions in ONE FIFO per stage (one comm stream / one
    communicator for both): the negative control. Returns True when every FIFO drains."""
    done = set()  # ("F"|"B", k, mb) compute tasks, (kind, k, mb) comm ops
    comp = [list(p) for p in programs]
    fifo = [[[(kd, mb) for _, ops in plans[k] for kd, mb in ops if kd in (0, 1)],
             [(kd, mb) for _, ops in plans[k] for kd, mb in ops if kd in (2, 3)]] for k in range(N)]
    if shared:
        fifo = [[[op for _, ops in plans[k] for op in ops]] * 2 for k in range(N)]

    def comm_ready(k, kd, mb):
        S = N - k
        if kd == 0:
            return ("F", k, mb) in done
        if kd == 2:
            return ("B", k, mb) in done
        if kd == 1:
            return mb - S < 0 or ("B", k, mb - S) in done
        return mb - 2 < 0 or ("B", k, mb - 2) in done

    def task_ready(k, d, mb):
        if d == O.FWD:
            return ((k == 0 or (1, k, mb) in done) and
                    (k == N - 1 or mb - 2 < 0 or (0, k, mb - 2) in done))
        return ((k == N - 1 or (3, k, mb) in done) and
                (k == 0 or mb - 2 < 0 or (2, k, mb - 2) in done))

    while True:
        progress = False
        for k in range(N):
            while comp[k] and task_ready(k, *comp[k][0]):
                d, mb = comp[k].pop(0)
                done.add(("F" if d == O.FWD else "B", k, mb))
                progress = True
            for q in (0, 1):
                if not fifo[k][q]:
                    continue
                kd, mb = fifo[k][q][0]
                if kd not in (0, 2):
                    continue  # receives complete from the sender's side
                peer = k + 1 if kd == 0 else k - 1
                rk = 1 if kd == 0 else 3
                pq = fifo[peer][q]
                if (pq and pq[0] == (rk, mb) and comm_ready(k, kd, mb) and comm_ready(peer, rk, mb)):
                    fifo[k][q].pop(0)
                    pq.pop(0)
                    done.add((kd, k, mb))
                    done.add((rk, peer, mb))
                    progress = True
        if all(not comp[k] and not fifo[k][0] and not fifo[k][1] for k in range(N)):
            return True
        if not progress:
            return False


def test_comm_plan_deadlock_free_on_split_streams(st):
    for N in range(1, 9):
        for M in range(1, 14):
            plans = [st.comm_plan(N, k, M) for k in range(N)]
            progs = [O.stage_program(N, k, M) for k in range(N)]
            assert simulate_streams(N, M, plans, progs), (N, M)
            for k in range(N):
                flat = [op for _, ops in plans[k] for op in ops]
                assert all(len(ops) == 1 for _, ops in plans[k])
                for kd in range(4):  # each channel carries mini-batches 0..M-1 in order
                    mbs = [mb for d, mb in flat if d == kd]
                    want = {0: k < N - 1, 1: k > 0, 2: k > 0, 3: k < N - 1}[kd]
                    assert mbs == (list(range(M)) if want else []), (N, M, k, kd)


def test_comm_plan_needs_split_streams(st):
    # negative control: the same single-op plan on ONE comm FIFO per stage deadlocks
    # (stage k sends act(i) to k+1 while k+1 sends grad(j) to k, both waiting for a
    # receive queued behind the other's send) — the reason each direction has its own
    # communicator and stream
    N, M = 4, 8
    plans = [st.comm_plan(N, k, M) for k in range(N)]
    progs = [O.stage_program(N, k, M) for k in range(N)]
    assert not simulate_streams(N, M, plans, progs, shared=True)
    assert simulate_streams(N, M, plans, progs)


def test_comm_plan_issue_points(st):
    # every op sits at the boundary of the task it belongs to: a send right after its
    # task, a receive right before (an interior stage in steady state)
    N, k, M = 4, 1, 10
    plan = st.comm_plan(N, k, M)
    prog = O.stage_program(N, k, M)
    for before, ops in plan:
        (kd, mb), = ops
        if kd in (0, 2):
            assert prog[before - 1] == ((O.FWD if kd == 0 else O.BWD), mb)
        else:
            assert prog[before] == ((O.FWD if kd == 1 else O.BWD), mb)
    # the two directions interleave in the plan but never share a FIFO
    kinds = [ops[0][0] for _, ops in plan]
    assert {0, 1, 2, 3} <= set(kinds)


def test_query_sizes_and_validation(st):
    from paper_1809_02839_b200 import _lib as L
    model = sd.config_mlp_2stage()
    layers = [(l.n_in, l.n_out, L.ST_ACT_RELU if l.act == sd.RELU else L.ST_ACT_NONE, 1) for l in model.layers]
    cfg, keep = L.make_config(layers, model.cuts, 0, 32, 0.05, 0.9)
    s = L.query_sizes(cfg)
    assert s.params == 784 * 256 + 256
    assert (s.s_fwd, s.s_bwd) == (1, 0) and s.wf_bytes > 0 and s.wb_bytes == 0
    assert s.stash_bytes == 2 * 32 * 784 * 4
    cfg1, keep1 = L.make_config(layers, model.cuts, 1, 32, 0.05, 0.9)
    s1 = L.query_sizes(cfg1)
    assert s1.params == 256 * 256 + 256 + 256 * 10 + 10 and (s1.s_fwd, s1.s_bwd) == (0, 0)
    assert s1.wf_bytes == 0 and s1.wb_bytes == 0
    bad, k2 = L.make_config([(784, 256, 1, 1), (200, 10, 0, 1)], [1], 0, 32, 0.05, 0.9)
    with pytest.raises(L.SpecTrainError, match="SHAPE"):
        L.query_sizes(bad)
    bad, k3 = L.make_config(layers, model.cuts, 2, 32, 0.05, 0.9)
    with pytest.raises(L.SpecTrainError, match="INPUT"):
        L.query_sizes(bad)
    bad, k4 = L.make_config(layers, model.cuts, 0, 32, 0.05, 1.5)
    with pytest.raises(L.SpecTrainError, match="gamma"):
        L.query_sizes(bad)
    # N=8 deep MLP: s_F/s_B per stage equal SURVEY App. A, WB separate only when 0 < s_B != s_F
    deep = sd.config_deep_mlp(8, width=64)
    dl = [(l.n_in, l.n_out, 1 if l.act == sd.RELU else 0, 1) for l in deep.layers]
    for k, (sf, sb) in enumerate([(7, 0), (6, 0), (6, 1), (5, 1), (5, 2), (4, 2), (4, 3), (3, 3)]):
        c, kk = L.make_config(dl, deep.cuts, k, 16, 0.02, 0.9)
        z = L.query_sizes(c)
        assert (z.s_fwd, z.s_bwd) == (sf, sb)
        assert (z.wb_bytes > 0) == (0 < sb != sf)


def test_replica_config_sizes_and_validation(st):
    """Hybrid DP × PP configs (st_config.replicas, NEXT-4): a replica's arenas hold its row
    slice (stash B/R rows), its parameters are the whole stage's; the limits of the
    header are enforced by st_query_sizes (no device work)."""
    from paper_1809_02839_b200 import _lib as L
    model = sd.mlp([784, 256, 192, 128, 10], cuts=[1, 3])
    layers = [(l.n_in, l.n_out, L.ST_ACT_RELU if l.act == sd.RELU else L.ST_ACT_NONE, 1) for l in model.layers]
    B = 32
    full, k0 = L.make_config(layers, model.cuts, 0, B, 0.05, 0.9)
    rep, k1 = L.make_config(layers, model.cuts, 0, B, 0.05, 0.9, replicas=[4, 1, 1], replica=3)
    sf, sr = L.query_sizes(full), L.query_sizes(rep)
    assert sr.params == sf.params and sr.w_bytes == sf.w_bytes
    assert sr.stash_bytes * 4 == sf.stash_bytes  # 3 slots × (B/4) rows × 784
    nxt, k2 = L.make_config(layers, model.cuts, 1, B, 0.05, 0.9, replicas=[4, 1, 1])
    assert L.query_sizes(nxt).stash_bytes == L.query_sizes(L.make_config(layers, model.cuts, 1, B, 0.05, 0.9)[0]).stash_bytes
    bad_cases = [
        ([1, 1, 2], 0, "last stage"),          # the last stage owns the batch-mean loss
        ([2, 2, 1], 0, "adjacent"),            # neighbouring replicated stages
        ([3, 1, 1], 0, "divisible"),           # 32 rows over 3 replicas
        ([2, 1, 1], 2, "replica"),             # replica index outside [0, 2)
        ([0, 1, 1], 0, "must be >= 1"),
    ]
    for reps, r, msg in bad_cases:
        c, kk = L.make_config(layers, model.cuts, 0, B, 0.05, 0.9, replicas=reps, replica=r)
        with pytest.raises(L.SpecTrainError, match=msg):
            L.query_sizes(c)
    c, kk = L.make_config(layers, model.cuts, 0, B, 0.05, 0.9, transport=L.ST_TRANSPORT_P2P, replicas=[2, 1, 1])
    with pytest.raises(L.SpecTrainError, match="NCCL or LOCAL"):
        L.query_sizes(c)
    lm = sd.lstm_lm(vocab=32, hidden=16, layers=2, cuts=[1, 3], seq_len=4)
    ll = [(l.n_in, l.n_out, 0, 1 if l.bias else 0, {sd.EMBED: L.ST_LAYER_EMBED, sd.LSTM: L.ST_LAYER_LSTM,
                                                  sd.DENSE: L.ST_LAYER_DENSE}[l.kind]) for l in lm.layers]
    c, kk = L.make_config(ll, lm.cuts, 1, 8, 0.1, 0.9, seq_len=4, replicas=[1, 2, 1])
    with pytest.raises(L.SpecTrainError, match="seq_len"):
        L.query_sizes(c)


# ---------------------------------------------------------------- st_partition (NEXT-4)

def _brute_partition(cost, N):
    import itertools
    L = len(cost)
    best, best_cuts = None, None
    for cuts in itertools.combinations(range(1, L), N - 1):  # lexicographic order
        b = (0,) + cuts + (L,)
        m = max(sum(cost[b[i]:b[i + 1]]) for i in range(N))
        if best is None or m < best:
            best, best_cuts = m, list(cuts)
    return best_cuts, best


def test_partition_brute_force(st):
    """Integer costs (exact in double): the optimum and the lexicographically smallest
    optimal cut vector equal exhaustive search; every stage non-empty."""
    rng = np.random.default_rng(0)
    for _ in range(300):
        L = int(rng.integers(1, 9))
        N = int(rng.integers(1, L + 1))
        cost = [int(x) for x in rng.integers(0, 20, L)]
        cuts, best = st.partition(cost, N)
        bc, bb = _brute_partition(cost, N)
        assert best == bb and cuts == bc, (cost, N, cuts, best, bc, bb)
        assert all(a < b for a, b in zip([0] + cuts, cuts + [L]))


def test_partition_errors_and_vgg_flops(st):
    with pytest.raises(st.SpecTrainError, match="INPUT"):
        st.partition([1.0, 2.0], 3)
    with pytest.raises(st.SpecTrainError, match="INPUT"):
        st.partition([1.0, -2.0], 1)
    # the flop-balanced VGG-16 8-stage partition of SURVEY §8(d) row 4 is optimal
    m = sd.config_vgg16(8)
    c = [2.0 * 128 * L.hw * L.hw * L.n_in * L.n_out * 9 if L.kind == sd.CONV else
         (2.0 * 128 * L.n_in * L.n_out if L.kind == sd.DENSE else 0.0) for L in m.layers]
    _, best = st.partition(c, 8)
    b = (0,) + tuple(m.cuts) + (len(c),)
    assert best == pytest.approx(max(sum(c[b[i]:b[i + 1]]) for i in range(8)), rel=1e-12)
