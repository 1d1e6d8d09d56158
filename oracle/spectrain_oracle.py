"""CPU oracle of SpecTrain pipelined training (arXiv 1809.02839) — TEST INFRASTRUCTURE.

This module is the plain, slow, obviously-correct reference the CUDA path is
checked against. It is NOT part of the product: only `tests/`,
`__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` / `--impl reference`
leg) may import or execute it. It shares no code with
`paper_1809_02839_b200/` and imports nothing from it; the only shared module is
`synthdata` (seeded input draws, none of the method's arithmetic).

Everything is NumPy float64, written in the paper's order and notation
(P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n; D-numbers are the
readings listed in DESIGN.md §3 / SURVEY §8(c)).

Pins (tests/test_oracle_pins.py): Eq. 5 worked example,
Eq. 1/Eq. 4 closed forms, N=1 == torch.optim.SGD with
dampening=γ (library routine), finite-difference gradients, stage composition
== monolithic autograd, s≡0 == vanilla pipeline, exact-rational App. C vectors
(brute force on a tiny chain, tests/golden/), schedule invariants.
Parity unpinned (decided, not fixed by the paper): D1 apply rule, D2 momentum
convention, D5 backward re-prediction — see DESIGN.md.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Sequence, Tuple

import numpy as np

FWD = 0
BWD = 1

PRED_SPECTRAIN = "spectrain"
PRED_NONE = "none"  # vanilla pipelining, s ≡ 0 (D-A8)
# PipeDream weight stashing (Fig. 6c): the forward of a mini-batch uses the
# stage's current weights and its backward uses the SAME (stashed) weights; no prediction
# (SURVEY §8(f) NEXT-2). The trace records, for a backward, the version its forward used.
PRED_STASH = "stash"
# Staleness-free target: the goal the paper states for SpecTrain —
# "the entire round trip of a mini-batch should adopt the same weight version",
# the version that exists once the previous mini-batch has updated the weights (P:229,
# "the only staleness-free version of weights is W6") — taken per stage: a forward
# predicts across the N−k−1 updates its stage applies before the mini-batch's backward
# arrives (s_F = N−k−1, the local F→B lag of the 1F1B program), the backward uses the
# current weights (s_B = 0). Both passes of mini-batch i then target stage version i.
# Eq. 5/6 add ⌊k/2⌋ to both (reading D6); this variant drops that term.
PRED_STALENESS_FREE = "staleness_free"

MOMENTUM_EMA = "ema"  # Eq. 1 literally: v = γ v + (1-γ) g
MOMENTUM_HEAVY_BALL = "heavy_ball"  # v = γ v + g (TF MomentumOptimizer, D2 flag)

APPLY_MOMENTUM = "momentum"  # D1: W ← W − η·v_new (Momentum SGD)


# --------------------------------------------------------------------------
# §3.2 formulas
# --------------------------------------------------------------------------

def version_difference(k: int, N: int, direction: int) -> int:
    """Eq. 5 (forward): s = ⌊k/2⌋ + N − k − 1.
    Eq. 6 (backward): s = ⌊k/2⌋.
    Returns −1 if not 0 ≤ k < N (mirrors the C-ABI)."""
    if not (0 <= k < N):
        return -1
    if direction == FWD:
        return k // 2 + N - k - 1
    return k // 2


def update_smoothed(v: np.ndarray, g: np.ndarray, gamma: float, momentum: str = MOMENTUM_EMA) -> np.ndarray:
    """Eq. 1: v_t = γ·v_{t−1} + (1−γ)·g_t.  HEAVY_BALL (D2): γ·v + g."""
    if momentum == MOMENTUM_EMA:
        return gamma * v + (1.0 - gamma) * g
    if momentum == MOMENTUM_HEAVY_BALL:
        return gamma * v + g
    raise ValueError(momentum)


def apply_update(W: np.ndarray, v_new: np.ndarray, g: np.ndarray, eta: float, apply: str = APPLY_MOMENTUM) -> np.ndarray:
    """D1: Momentum SGD step W ← W − η·v_t (P:373 'Momentum SGD'; Eq. 3 uses v in place
    of the gradient). Eq. 2's literal plain-SGD form is not offered: no
    path uses it and nothing in the paper would pin it."""
    if apply == APPLY_MOMENTUM:
        return W - eta * v_new
    raise ValueError(apply)


def predict(W: np.ndarray, v: np.ndarray, s: int, eta: float) -> np.ndarray:
    """Eq. 4: Ŵ_{t+s} = W_t − s·η·v_{t−1}.  s = 0 returns W itself."""
    if s == 0:
        return W
    return W - s * eta * v



def prediction_rmse(W_old: np.ndarray, V_old: np.ndarray, W_now: np.ndarray, s: int, eta: float):
    """Prediction accuracy (Fig. 7): with (W_old, V_old) the stage state s
    updates before W_now (V_old = the smoothed gradient stored next to W_old, i.e.
    v_{t−s−1} in the paper's indexing, D4), the predicted weights are
    Ŵ_t = W_old − s·η·V_old (Eq. 4) and the stale ones W_{t−s} = W_old. Returns
    (RMSE(Ŵ_t, W_t), RMSE(W_{t−s}, W_t)) over all elements."""
    W_hat = predict(W_old, V_old, s, eta)
    return float(np.sqrt(np.mean((W_hat - W_now) ** 2))), float(np.sqrt(np.mean((W_old - W_now) ** 2)))

# --------------------------------------------------------------------------
# §3.1 schedule: PipeDream 1F1B round-robin, D8
# --------------------------------------------------------------------------

def stage_program(N: int, k: int, M: int) -> List[Tuple[int, int]]:
    """Stage k's task list: w = min(N−k−1, M) warm-up forwards, then (F, B)
    pairs, then cooldown backwards."""
    w = min(N - k - 1, M)
    prog = [(FWD, i) for i in range(w)]
    for j in range(M - w):
        prog.append((FWD, w + j))
        prog.append((BWD, j))
    prog += [(BWD, j) for j in range(M - w, M)]
    return prog


# --------------------------------------------------------------------------
# Dense stage forward / backward (§2.1; SPEC nn S:115-145)
# --------------------------------------------------------------------------

def unpack_stage(layers, flat: np.ndarray):
    """Stage flat layout: per layer, in order —
    dense: W [in×out] row-major, then b [out] (if bias);
    embed: E [vocab×dim];
    lstm : W_ih [in×4h], W_hh [h×4h], b [4h]."""
    out, off = [], 0

    def take(n, shape):
        nonlocal off
        a = flat[off:off + n].reshape(shape)
        off += n
        return a

    for L in layers:
        kind = getattr(L, "kind", "dense")
        if kind == "pool":
            out.append(())
        elif kind == "conv":
            W = take(9 * L.n_in * L.n_out, (3, 3, L.n_in, L.n_out))
            b = take(L.n_out, (L.n_out,)) if L.bias else None
            out.append((W, b))
        elif kind == "embed":
            out.append((take(L.n_in * L.n_out, (L.n_in, L.n_out)),))
        elif kind == "lstm":
            h = L.n_out
            out.append((take(L.n_in * 4 * h, (L.n_in, 4 * h)), take(h * 4 * h, (h, 4 * h)), take(4 * h, (4 * h,))))
        else:
            W = take(L.n_in * L.n_out, (L.n_in, L.n_out))
            b = take(L.n_out, (L.n_out,)) if L.bias else None
            out.append((W, b))
    assert off == flat.size, (off, flat.size)
    return out


def pack_stage(layers, parts) -> np.ndarray:
    chunks = []
    for L, part in zip(layers, parts):
        for a in part:
            if a is not None:
                chunks.append(np.asarray(a).reshape(-1))
    return np.concatenate(chunks) if chunks else np.zeros(0)


def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def lstm_forward(W_ih, W_hh, b, X, T):
    """LSTM over T time-major steps of X [T·B × in] (reading D18):
    G_t = X_t·W_ih + h_{t−1}·W_hh + b; i, f, o = σ(·), g = tanh(·) (order i, f, g, o);
    c_t = f⊙c_{t−1} + i⊙g; h_t = o⊙tanh(c_t); h_{−1} = c_{−1} = 0."""
    B = X.shape[0] // T
    H = W_hh.shape[0]
    Gx = X @ W_ih + b
    h = np.zeros((B, H))
    c = np.zeros((B, H))
    outs, cache = [], []
    for t in range(T):
        G = Gx[t * B:(t + 1) * B] + h @ W_hh
        i, f, g, o = _sigmoid(G[:, :H]), _sigmoid(G[:, H:2 * H]), np.tanh(G[:, 2 * H:3 * H]), _sigmoid(G[:, 3 * H:])
        c_prev, h_prev = c, h
        c = f * c_prev + i * g
        h = o * np.tanh(c)
        cache.append((i, f, g, o, c_prev, c, h_prev))
        outs.append(h)
    return np.concatenate(outs, axis=0), cache


def lstm_backward(W_ih, W_hh, X, cache, dOut, T, need_dX=True):
    """Backpropagation through time for lstm_forward; returns (gW_ih, gW_hh, gb, dX)."""
    B = X.shape[0] // T
    H = W_hh.shape[0]
    dG_all = np.zeros((T * B, 4 * H))
    dh_next = np.zeros((B, H))
    dc_next = np.zeros((B, H))
    gW_hh = np.zeros_like(W_hh)
    for t in range(T - 1, -1, -1):
        i, f, g, o, c_prev, c, h_prev = cache[t]
        dh = dOut[t * B:(t + 1) * B] + dh_next
        tc = np.tanh(c)
        dc = dc_next + dh * o * (1.0 - tc * tc)
        do = dh * tc
        di = dc * g
        dg = dc * i
        df = dc * c_prev
        dG = np.concatenate([di * i * (1 - i), df * f * (1 - f), dg * (1 - g * g), do * o * (1 - o)], axis=1)
        dG_all[t * B:(t + 1) * B] = dG
        gW_hh += h_prev.T @ dG
        dh_next = dG @ W_hh.T
        dc_next = dc * f
    gW_ih = X.T @ dG_all
    gb = dG_all.sum(axis=0)
    dX = dG_all @ W_ih.T if need_dX else None
    return gW_ih, gW_hh, gb, dX


def conv3x3_forward(W, b, X):
    """3×3 convolution, stride 1, zero padding 1, NHWC:
    Y[n,h,w,o] = b[o] + Σ_{kh,kw,c} Xpad[n, h+kh, w+kw, c] · W[kh, kw, c, o]."""
    n, H, Wd, _ = X.shape
    Xp = np.pad(X, ((0, 0), (1, 1), (1, 1), (0, 0)))
    Y = np.zeros((n, H, Wd, W.shape[3]))
    for kh in range(3):
        for kw in range(3):
            Y += Xp[:, kh:kh + H, kw:kw + Wd, :] @ W[kh, kw]
    if b is not None:
        Y += b
    return Y


def conv3x3_backward(W, X, dY, need_dX=True):
    """Gradients of conv3x3_forward: gW[kh,kw] = Σ Xpad-shiftᵀ·dY, gb = Σ dY,
    dX = the padded scatter of dY·W[kh,kw]ᵀ."""
    n, H, Wd, C = X.shape
    Xp = np.pad(X, ((0, 0), (1, 1), (1, 1), (0, 0)))
    gW = np.zeros_like(W)
    dXp = np.zeros_like(Xp)
    dY2 = dY.reshape(-1, dY.shape[3])
    for kh in range(3):
        for kw in range(3):
            gW[kh, kw] = Xp[:, kh:kh + H, kw:kw + Wd, :].reshape(-1, C).T @ dY2
            if need_dX:
                dXp[:, kh:kh + H, kw:kw + Wd, :] += dY @ W[kh, kw].T
    gb = dY2.sum(axis=0)
    return gW, gb, (dXp[:, 1:-1, 1:-1, :] if need_dX else None)


def maxpool2_forward(X):
    """2×2 max-pool, stride 2, NHWC. The routed position is the first maximum in
    row-major window order (reading D21; ties only occur among ReLU zeros, where the
    routed gradient is masked to 0 anyway)."""
    n, H, Wd, C = X.shape
    w4 = np.stack([X[:, 0::2, 0::2], X[:, 0::2, 1::2], X[:, 1::2, 0::2], X[:, 1::2, 1::2]], axis=0)
    arg = np.argmax(w4, axis=0)  # numpy argmax: first occurrence
    return w4.max(axis=0), arg


def maxpool2_backward(arg, dY, shape):
    dX = np.zeros(shape)
    for q, (dh, dw) in enumerate(((0, 0), (0, 1), (1, 0), (1, 1))):
        dX[:, dh::2, dw::2] += dY * (arg == q)
    return dX


def stage_forward(layers, flat: np.ndarray, A, T: int = 1):
    """Per layer: dense Z = A·W + b, A' = ReLU(Z) (identity when act ==
    'none'); embed A' = E[tokens]; lstm A' = lstm_forward(A). Activations are
    [T·B × width], time-major. Returns (stage output, stash per layer)."""
    stash = []
    for L, prm in zip(layers, unpack_stage(layers, flat)):
        kind = getattr(L, "kind", "dense")
        if kind in ("conv", "pool"):
            n = A.shape[0]
            X = A.reshape(n, L.hw, L.hw, L.n_in)
            if kind == "conv":
                W, b = prm
                Z = conv3x3_forward(W, b, X)
                stash.append((X, Z))
                Y = np.maximum(Z, 0.0) if L.act == "relu" else Z
            else:
                Y, arg = maxpool2_forward(X)
                stash.append((X.shape, arg))
            A = Y.reshape(n, -1)
        elif kind == "embed":
            (E,) = prm
            tok = np.asarray(A).astype(np.int64).reshape(-1)
            stash.append((tok,))
            A = E[tok]
        elif kind == "lstm":
            W_ih, W_hh, b = prm
            out, cache = lstm_forward(W_ih, W_hh, b, A, T)
            stash.append((A, cache))
            A = out
        else:
            W, b = prm
            Z = A @ W
            if b is not None:
                Z = Z + b
            stash.append((A, Z))
            A = np.maximum(Z, 0.0) if L.act == "relu" else Z
    return A, stash


def stage_backward(layers, flat: np.ndarray, stash, dA_out: np.ndarray, need_dA_in: bool = True, T: int = 1):
    """Reverse layers. dense: dZ = dA ⊙ 1[Z>0] (D12: ReLU'(0)=0); g_W = Aᵀ·dZ;
    g_b = Σ_rows dZ; dA_prev = dZ·Wᵀ. embed: g_E[token] += dA rows. lstm: BPTT.
    Returns (flat gradient, dA_in or None)."""
    params = unpack_stage(layers, flat)
    grads = [None] * len(layers)
    dA = dA_out
    for li in range(len(layers) - 1, -1, -1):
        L = layers[li]
        kind = getattr(L, "kind", "dense")
        need = li > 0 or need_dA_in
        if kind in ("conv", "pool"):
            n = dA.shape[0]
            if kind == "conv":
                W, b = params[li]
                X, Z = stash[li]
                dZ = dA.reshape(Z.shape)
                if L.act == "relu":
                    dZ = dZ * (Z > 0.0)
                gW, gb, dX = conv3x3_backward(W, X, dZ, need)
                grads[li] = (gW, gb if L.bias else None)
            else:
                shape, arg = stash[li]
                dX = maxpool2_backward(arg, dA.reshape(arg.shape), shape)
                grads[li] = ()
            dA = dX.reshape(n, -1) if dX is not None else None
        elif kind == "embed":
            (E,) = params[li]
            (tok,) = stash[li]
            gE = np.zeros_like(E)
            np.add.at(gE, tok, dA)
            grads[li] = (gE,)
            dA = None
        elif kind == "lstm":
            W_ih, W_hh, b = params[li]
            X, cache = stash[li]
            gW_ih, gW_hh, gb, dX = lstm_backward(W_ih, W_hh, X, cache, dA, T, need)
            grads[li] = (gW_ih, gW_hh, gb)
            dA = dX
        else:
            W, b = params[li]
            A_in, Z = stash[li]
            dZ = dA * (Z > 0.0) if L.act == "relu" else dA
            gW = A_in.T @ dZ
            gb = dZ.sum(axis=0) if L.bias else None
            grads[li] = (gW, gb)
            dA = dZ @ W.T if need else None
    return pack_stage(layers, grads), dA


def loss_and_grad(kind: str, Z: np.ndarray, target: np.ndarray) -> Tuple[float, np.ndarray]:
    """D11: softmax cross-entropy, mean over the batch, max-subtracted softmax
    (P:105-107 'loss between the prediction and the ground truth');
    'half_mse': mean_b ½‖Z_b − t_b‖² (the App. C scalar chain)."""
    B = Z.shape[0]
    if kind == "softmax_ce":
        m = Z.max(axis=1, keepdims=True)
        e = np.exp(Z - m)
        s = e.sum(axis=1, keepdims=True)
        logp = Z - m - np.log(s)
        y = target.astype(np.int64)
        loss = -logp[np.arange(B), y].mean()
        p = e / s
        onehot = np.zeros_like(Z)
        onehot[np.arange(B), y] = 1.0
        return float(loss), (p - onehot) / B
    if kind == "half_mse":
        d = Z - target
        return float(0.5 * (d * d).sum() / B), d / B
    raise ValueError(kind)


# --------------------------------------------------------------------------
# Pipelined SpecTrain run
# --------------------------------------------------------------------------

@dataclasses.dataclass
class Event:
    """One task record: stage, position in the stage program,
    direction, mini-batch, base version c (updates applied so far), version
    difference s, target version c+s."""

    stage: int
    op_idx: int
    dir: int
    mb: int
    base_version: int
    s: int

    @property
    def target(self) -> int:
        return self.base_version + self.s

    def as_tuple(self) -> Tuple[int, int, int, int, int, int, int]:
        return (self.stage, self.op_idx, self.dir, self.mb, self.base_version, self.s, self.target)


@dataclasses.dataclass
class RunResult:
    W: List[np.ndarray]
    V: List[np.ndarray]
    losses: np.ndarray
    trace: List[List[Event]]


def run(model, W0: Sequence[np.ndarray], X: np.ndarray, Y: np.ndarray, eta: float, gamma: float,
        pred: str = PRED_SPECTRAIN, momentum: str = MOMENTUM_EMA, apply: str = APPLY_MOMENTUM,
        order: str = "round_robin") -> RunResult:
    """Interpret every stage's 1F1B program in a dependency-respecting order.

    F(i,k) needs F(i,k−1)'s output; B(i,k) needs B(i,k+1)'s dA (or, at the last
    stage, its own F(i)). Before each task the stage computes Ŵ = W − s·η·V from
    its CURRENT state (Eq. 4 with Eq. 5/6; D4, D5). After each B: Eq. 1, then
    the D1 apply, then version += 1 (D9). The result does not depend on the
    interpretation order (`order` = 'round_robin' or 'stage_major' exists so a
    test can show that)."""
    N = model.num_stages
    M = X.shape[0]
    T = getattr(model, "seq_len", 1)
    W = [np.array(w, dtype=np.float64, copy=True) for w in W0]
    V = [np.zeros_like(w) for w in W]
    version = [0] * N
    progs = [stage_program(N, k, M) for k in range(N)]
    pc = [0] * N
    act: Dict[Tuple[int, int], np.ndarray] = {}  # (k, i) → stage k's forward output for mb i
    grad: Dict[Tuple[int, int], np.ndarray] = {}  # (k, i) → dA w.r.t. stage k's input for mb i
    stash: Dict[Tuple[int, int], list] = {}
    dlogits: Dict[int, np.ndarray] = {}
    losses = np.full(M, np.nan)
    trace: List[List[Event]] = [[] for _ in range(N)]

    def s_of(k: int, d: int) -> int:
        if pred in (PRED_NONE, PRED_STASH):
            return 0
        if pred == PRED_STALENESS_FREE:
            return (N - k - 1) if d == FWD else 0
        return version_difference(k, N, d)

    wstash: Dict[Tuple[int, int], Tuple[np.ndarray, int]] = {}  # PRED_STASH: (k, i) → (W, version) of F(i)

    def ready(k: int) -> bool:
        d, i = progs[k][pc[k]]
        if d == FWD:
            return k == 0 or (k - 1, i) in act
        return k == N - 1 or (k + 1, i) in grad

    def execute(k: int) -> None:
        d, i = progs[k][pc[k]]
        layers = model.stage_layers(k)
        s = s_of(k, d)
        W_hat = predict(W[k], V[k], s, eta)
        base = version[k]
        if pred == PRED_STASH:
            if d == FWD:
                wstash[(k, i)] = (W_hat.copy(), version[k])  # s = 0: W_hat is the current W
            else:
                W_hat, base = wstash.pop((k, i))  # the forward's weights and their version
        trace[k].append(Event(k, pc[k], d, i, base, s))
        if d == FWD:
            if k == 0:
                A_in = X[i] if getattr(layers[0], "kind", "dense") == "embed" else X[i].astype(np.float64)
            else:
                A_in = act.pop((k - 1, i))
            out, st = stage_forward(layers, W_hat, A_in, T)
            stash[(k, i)] = st
            if k == N - 1:
                losses[i], dlogits[i] = loss_and_grad(model.loss, out, Y[i])
            else:
                act[(k, i)] = out
        else:
            dA = dlogits.pop(i) if k == N - 1 else grad.pop((k + 1, i))
            g, dA_in = stage_backward(layers, W_hat, stash.pop((k, i)), dA, need_dA_in=(k > 0), T=T)
            if k > 0:
                grad[(k, i)] = dA_in
            # Update after each B: Eq. 1, D1 apply, version += 1.
            V[k] = update_smoothed(V[k], g, gamma, momentum)
            W[k] = apply_update(W[k], V[k], g, eta, apply)
            version[k] += 1
        pc[k] += 1

    total = sum(len(p) for p in progs)
    done = 0
    while done < total:
        progressed = False
        for k in range(N):
            if order == "stage_major":
                while pc[k] < len(progs[k]) and ready(k):
                    execute(k)
                    done += 1
                    progressed = True
            else:
                if pc[k] < len(progs[k]) and ready(k):
                    execute(k)
                    done += 1
                    progressed = True
        if not progressed:
            raise RuntimeError("pipeline deadlock (invariant violation)")
    return RunResult(W, V, losses, trace)


def sequential_momentum_sgd(model, W0_flat: np.ndarray, X: np.ndarray, Y: np.ndarray, eta: float,
                            gamma: float, momentum: str = MOMENTUM_EMA) -> Tuple[np.ndarray, np.ndarray]:
    """Single-device momentum SGD over all layers (the staleness-free trainer of
    Fig. 6a). Used to pin the N=1 degenerate case."""
    W = np.array(W0_flat, dtype=np.float64, copy=True)
    V = np.zeros_like(W)
    losses = []
    layers = model.layers
    for i in range(X.shape[0]):
        out, st = stage_forward(layers, W, X[i].astype(np.float64))
        loss, dZ = loss_and_grad(model.loss, out, Y[i])
        g, _ = stage_backward(layers, W, st, dZ, need_dA_in=False)
        V = update_smoothed(V, g, gamma, momentum)
        W = W - eta * V
        losses.append(loss)
    return W, np.array(losses)
