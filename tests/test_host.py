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
                            (O.PRED_STASH, st.ST_PRED_STASH)):
            tr = _oracle_trace(N, M, pred)
            for k in range(N):
                assert st.program(N, k, M, cpred) == [e.as_tuple() for e in tr[k]], (N, M, k, pred)


def simulate_plans(plans, N):
    """Strict semantics: a group completes once every op in it is matched by an op
    the peer has POSTED (in its current or an earlier group); a stage posts group
    g+1 only after group g completed. Returns True when every stage finishes."""
    # channel ops in order: chan[(src, dst)] = list of mb for sends / recvs
    sends = {}
    recvs = {}
    idx = []  # per stage, per group: list of (kind, chan, ordinal, mb)
    for k in range(N):
        gl = []
        for before, ops in plans[k]:
            g = []
            for kind, mb in ops:
                if kind in (0, 3):  # send_fwd to k+1 / recv_bwd from k+1
                    peer = k + 1
                else:
                    peer = k - 1
                if kind in (0, 2):
                    ch = (k, peer)
                    lst = sends.setdefault(ch, [])
                    g.append(("s", ch, len(lst), mb))
                    lst.append(mb)
                else:
                    ch = (peer, k)
                    lst = recvs.setdefault(ch, [])
                    g.append(("r", ch, len(lst), mb))
                    lst.append(mb)
            gl.append(g)
        idx.append(gl)
    for ch in set(sends) | set(recvs):
        assert sends.get(ch, []) == recvs.get(ch, []), ("message order mismatch on channel", ch)
    cur = [0] * N
    posted_s = {}
    posted_r = {}

    def post(k):
        if cur[k] < len(idx[k]):
            for t, ch, o, mb in idx[k][cur[k]]:
                d = posted_s if t == "s" else posted_r
                d[ch] = max(d.get(ch, 0), o + 1)

    for k in range(N):
        post(k)
    while True:
        progress = False
        for k in range(N):
            if cur[k] >= len(idx[k]):
                continue
            ok = all((posted_r.get(ch, 0) > o) if t == "s" else (posted_s.get(ch, 0) > o)
                     for t, ch, o, mb in idx[k][cur[k]])
            if ok:
                cur[k] += 1
                post(k)
                progress = True
        if all(cur[k] >= len(idx[k]) for k in range(N)):
            return True
        if not progress:
            return False


def test_comm_plan_deadlock_free_and_paired(st):
    for N in range(1, 9):
        for M in range(1, 14):
            plans = [st.comm_plan(N, k, M) for k in range(N)]
            assert simulate_plans(plans, N), (N, M)
            for k in range(N):
                flat = [op for _, ops in plans[k] for op in ops]
                n_send_f = sum(1 for kd, _ in flat if kd == 0)
                n_recv_f = sum(1 for kd, _ in flat if kd == 1)
                assert n_send_f == (M if k < N - 1 else 0) and n_recv_f == (M if k > 0 else 0)


def test_comm_plan_megatron_pairing(st):
    # steady state at an interior stage: send act(i) grouped with recv grad(j) (same peer)
    plan = st.comm_plan(4, 1, 10)
    assert any(ops == [(0, 5), (3, 3)] for _, ops in plan)
    assert any(ops == [(2, 3), (1, 6)] for _, ops in plan)


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
