"""Seeded synthetic inputs shared by the CPU oracle and the CUDA path.

This module holds NONE of SpecTrain's arithmetic (no forward/backward, no
momentum, no prediction). It only draws the arrays both sides consume, so that
the oracle (`oracle/`) and the product (`paper_1809_02839_b200/`) never import
each other.

Recipe (DESIGN.md §Readings D13):
- RNG: numpy PCG64 `numpy.random.default_rng(seed)`.
- Weights: Glorot-uniform `U(-r, r)`, `r = sqrt(6/(in+out))`, biases 0
  (SPEC S:150 initialisation; the paper is silent, P:374 fixes only the LR).
- Images: U[0,1) in the input width (784 = MNIST-shaped, P:377 CIFAR/MNIST-like
  synthetic stand-ins).
- Labels: argmax of a fixed N(0,1) "teacher" projection of the image (learnable
  so the loss moves), or uniform when `labels="uniform"` (bench).
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence, Tuple

import numpy as np

RELU = "relu"
NONE = "none"

DENSE = "dense"
EMBED = "embed"
LSTM = "lstm"
CONV = "conv"
POOL = "pool"


@dataclasses.dataclass(frozen=True)
class Layer:
    """One layer of the chain.

    dense: `Z = A·W + b`, `A' = act(Z)`; W [in×out] row-major, then b [out].
    embed: token ids → rows of E [n_in = vocab × n_out = dim] (params: E only).
    lstm : input n_in, hidden n_out; params W_ih [in×4h], W_hh [h×4h], b [4h]
           (gate order i, f, g, o — reading D18)."""

    n_in: int
    n_out: int
    act: str = RELU
    bias: bool = True
    kind: str = DENSE
    hw: int = 1  # conv / pool: input spatial side (square, NHWC activations)

    @property
    def width_in(self) -> int:
        """Per-sample activation width entering the layer."""
        return self.hw * self.hw * self.n_in if self.kind in (CONV, POOL) else self.n_in

    @property
    def width_out(self) -> int:
        if self.kind == CONV:
            return self.hw * self.hw * self.n_out
        if self.kind == POOL:
            return (self.hw // 2) * (self.hw // 2) * self.n_out
        return self.n_out

    @property
    def n_params(self) -> int:
        if self.kind == POOL:
            return 0
        if self.kind == CONV:
            return 9 * self.n_in * self.n_out + (self.n_out if self.bias else 0)
        if self.kind == EMBED:
            return self.n_in * self.n_out
        if self.kind == LSTM:
            return (self.n_in + self.n_out) * 4 * self.n_out + 4 * self.n_out
        return self.n_in * self.n_out + (self.n_out if self.bias else 0)


@dataclasses.dataclass(frozen=True)
class Model:
    """A chain of dense layers cut into contiguous pipeline stages."""

    layers: Tuple[Layer, ...]
    cuts: Tuple[int, ...]  # N-1 strictly increasing layer indices; stage k = [cuts[k-1], cuts[k])
    loss: str = "softmax_ce"  # or "half_mse" (App. C scalar chain)
    seq_len: int = 1  # T: activations are [T·B × width], time-major rows (t·B + b)

    @property
    def num_stages(self) -> int:
        return len(self.cuts) + 1

    def stage_layers(self, k: int) -> Tuple[Layer, ...]:
        bounds = (0,) + tuple(self.cuts) + (len(self.layers),)
        return self.layers[bounds[k]:bounds[k + 1]]

    def stage_bounds(self, k: int) -> Tuple[int, int]:
        bounds = (0,) + tuple(self.cuts) + (len(self.layers),)
        return bounds[k], bounds[k + 1]

    def stage_params(self, k: int) -> int:
        return sum(l.n_params for l in self.stage_layers(k))


def mlp(widths: Sequence[int], cuts: Sequence[int], bias: bool = True, loss: str = "softmax_ce") -> Model:
    """ReLU MLP over `widths` (last layer identity), cut at `cuts` (layer indices)."""
    n = len(widths) - 1
    layers = tuple(
        Layer(widths[i], widths[i + 1], NONE if i == n - 1 else RELU, bias) for i in range(n)
    )
    cuts = tuple(int(c) for c in cuts)
    if any(not (0 < c < n) for c in cuts) or list(cuts) != sorted(set(cuts)):
        raise ValueError(f"invalid cuts {cuts} for {n} layers")
    return Model(layers, cuts, loss)


def even_cuts(num_layers: int, num_stages: int) -> Tuple[int, ...]:
    """Contiguous cuts giving stage sizes that differ by at most one; the extra
    layers go to the LAST stages (so e.g. 9 layers / 8 stages = {L1}..{L7}{L8,L9},
    SURVEY §8(d) config 2)."""
    if not 1 <= num_stages <= num_layers:
        raise ValueError("need 1 <= stages <= layers")
    base, extra = divmod(num_layers, num_stages)
    sizes = [base + (1 if k >= num_stages - extra else 0) for k in range(num_stages)]
    cuts, acc = [], 0
    for s in sizes[:-1]:
        acc += s
        cuts.append(acc)
    return tuple(cuts)


# ---- named configurations (BASELINE.json `configs`) -----------------------

def config_mlp_2stage() -> Model:
    """BJ configs[0]: 4-layer MLP 784-256-256-10, 2 stages {L1}{L2,L3}."""
    return mlp([784, 256, 256, 10], cuts=[1])


def config_deep_mlp(num_stages: int = 8, width: int = 1024, depth: int = 9) -> Model:
    """SURVEY §8(d) row 1b parity model: 784-1024×8-10, one layer per stage, last two merged."""
    widths = [784] + [width] * (depth - 1) + [10]
    return mlp(widths, cuts=even_cuts(depth, num_stages))


def config_wide_fcn(num_stages: int, width: int = 8192, hidden_layers: int = 8) -> Model:
    """BJ configs[1]: wide FCN, `hidden_layers` × `width` units on 784-dim inputs, 10 classes.
    9 weight layers: 784→w, (hidden_layers-1)× w→w, w→10."""
    widths = [784] + [width] * hidden_layers + [10]
    return mlp(widths, cuts=even_cuts(len(widths) - 1, num_stages))


def lstm_lm(vocab: int, hidden: int, layers: int, cuts: Sequence[int], seq_len: int) -> Model:
    """Embedding → `layers` × LSTM(hidden) → dense softmax over the vocabulary
    (BJ configs[2]; reading D18: untied embedding / softmax, h0 = c0 = 0 per mini-batch)."""
    ls = [Layer(vocab, hidden, NONE, False, EMBED)]
    ls += [Layer(hidden, hidden, NONE, True, LSTM) for _ in range(layers)]
    ls += [Layer(hidden, vocab, NONE, True, DENSE)]
    return Model(tuple(ls), tuple(int(c) for c in cuts), "softmax_ce", seq_len)


def config_lstm_lm(num_stages: int = 4, vocab: int = 10000, hidden: int = 1500, seq_len: int = 35) -> Model:
    """BJ configs[2]: 2-layer LSTM LM, hidden 1500, seq 35, vocab 10k; 4 stages
    {Emb}{LSTM1}{LSTM2}{Softmax}."""
    return lstm_lm(vocab, hidden, 2, even_cuts(4, num_stages), seq_len)


VGG16_CIFAR = (64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M")


def vgg(cfg=VGG16_CIFAR, fc=(512, 512), classes: int = 10, hw: int = 32, in_ch: int = 3,
        cuts: Optional[Sequence[int]] = None) -> Model:
    """VGG on hw×hw×in_ch images (reading D19: 13 conv 3×3 pad 1 + ReLU, 2×2 max-pool
    at 'M', FC 512-512-10, no BN / dropout). NHWC activations; the flatten after the
    last pool is implicit (1×1×512 → 512)."""
    ls = []
    c, s = in_ch, hw
    for v in cfg:
        if v == "M":
            ls.append(Layer(c, c, NONE, False, POOL, s))
            s //= 2
        else:
            ls.append(Layer(c, v, RELU, True, CONV, s))
            c = v
    w = c * s * s
    for f in fc:
        ls.append(Layer(w, f, RELU, True, DENSE))
        w = f
    ls.append(Layer(w, classes, NONE, True, DENSE))
    return Model(tuple(ls), tuple(cuts or ()), "softmax_ce", 1)


def vgg16_cuts_8() -> Tuple[int, ...]:
    """SURVEY §8(d) row 4 TF32 (flop-balanced) 8-stage partition, pools attached to
    their conv: {c1_1,c1_2,P}{c2_1}{c2_2,P}{c3_1,c3_2}{c3_3,P}{c4_1,c4_2}{c4_3,P}{c5_*,P,fc×3}.
    Layer indices: c1_1 0, c1_2 1, P 2, c2_1 3, c2_2 4, P 5, c3_1 6, c3_2 7, c3_3 8, P 9,
    c4_1 10, c4_2 11, c4_3 12, P 13, c5_1 14 ..."""
    return (3, 4, 6, 8, 10, 12, 14)


def config_vgg16(num_stages: int = 8) -> Model:
    """BJ configs[3]: VGG-16 on 32×32×3 CIFAR-shaped images, batch 128, 8 stages."""
    if num_stages == 8:
        return vgg(cuts=vgg16_cuts_8())
    n = len(vgg().layers)
    return vgg(cuts=even_cuts(n, num_stages))


def config_large_fcn(num_stages: int, width: int = 16384, hidden_layers: int = 16) -> Model:
    """BJ configs[4]: large FCN 16 × 16384."""
    widths = [784] + [width] * hidden_layers + [10]
    return mlp(widths, cuts=even_cuts(len(widths) - 1, num_stages))


# ---- draws -----------------------------------------------------------------

def glorot_params(model: Model, seed: int) -> List[np.ndarray]:
    """Per-stage flat float64 parameter vectors in the stage layout
    (layer-major: W_l [in×out] row-major, then b_l [out]).
    Embedding: U(-0.1, 0.1). LSTM: W_ih, W_hh Glorot over (in, 4h) / (h, 4h), b = 0."""
    rng = np.random.default_rng(seed)
    out = []
    for k in range(model.num_stages):
        parts = []
        for layer in model.stage_layers(k):
            if layer.kind == EMBED:
                parts.append(rng.uniform(-0.1, 0.1, size=layer.n_in * layer.n_out))
            elif layer.kind == POOL:
                pass
            elif layer.kind == CONV:
                r = math.sqrt(6.0 / (9 * layer.n_in + 9 * layer.n_out))
                parts.append(rng.uniform(-r, r, size=9 * layer.n_in * layer.n_out))
                if layer.bias:
                    parts.append(np.zeros(layer.n_out))
            elif layer.kind == LSTM:
                h = layer.n_out
                r1 = math.sqrt(6.0 / (layer.n_in + 4 * h))
                r2 = math.sqrt(6.0 / (h + 4 * h))
                parts.append(rng.uniform(-r1, r1, size=layer.n_in * 4 * h))
                parts.append(rng.uniform(-r2, r2, size=h * 4 * h))
                parts.append(np.zeros(4 * h))
            else:
                r = math.sqrt(6.0 / (layer.n_in + layer.n_out))
                parts.append(rng.uniform(-r, r, size=layer.n_in * layer.n_out))
                if layer.bias:
                    parts.append(np.zeros(layer.n_out))
        out.append(np.concatenate(parts) if parts else np.zeros(0))
    return out


def glorot_dense_layer_f32(layer: Layer, seed: int, index: int) -> np.ndarray:
    """One dense layer's flat block [W (Glorot-U ±√(6/(in+out))) row-major, b = 0] as
    float32, from its own stream PCG64([seed, index]) — for models too large to draw
    whole on the host (the large FCN: 4.04G parameters); the same block can be redrawn
    layer by layer."""
    rng = np.random.default_rng([seed, index])
    r = np.float32(math.sqrt(6.0 / (layer.n_in + layer.n_out)))
    w = rng.random(layer.n_in * layer.n_out, dtype=np.float32)
    w *= 2 * r
    w -= r
    if layer.bias:
        return np.concatenate([w, np.zeros(layer.n_out, np.float32)])
    return w


def tokens(vocab: int, num_batches: int, batch: int, seq_len: int, seed: int,
           dist: str = "zipf") -> Tuple[np.ndarray, np.ndarray]:
    """Synthetic LM data: X int32 [M, T·B] input tokens (time-major, row t·B + b),
    Y int32 [M, T·B] next-token targets. Zipf(1.0)-like over the vocabulary
    (tokens uniform or Zipf), or uniform."""
    rng = np.random.default_rng(seed)
    if dist == "zipf":
        p = 1.0 / np.arange(1, vocab + 1)
        p /= p.sum()
        seq = rng.choice(vocab, size=(num_batches, batch, seq_len + 1), p=p)
    else:
        seq = rng.integers(0, vocab, size=(num_batches, batch, seq_len + 1))
    x = seq[:, :, :-1].transpose(0, 2, 1).reshape(num_batches, seq_len * batch)
    y = seq[:, :, 1:].transpose(0, 2, 1).reshape(num_batches, seq_len * batch)
    return x.astype(np.int32), y.astype(np.int32)


def images_and_labels(
    n_in: int,
    n_classes: int,
    num_batches: int,
    batch: int,
    seed: int,
    labels: str = "teacher",
) -> Tuple[np.ndarray, np.ndarray]:
    """X: [M, B, n_in] U[0,1); Y: [M, B] int32 labels in [0, n_classes)."""
    rng = np.random.default_rng(seed)
    x = rng.random((num_batches, batch, n_in))
    if labels == "teacher":
        teacher = rng.standard_normal((n_in, n_classes))
        y = np.argmax((x - 0.5) @ teacher, axis=-1).astype(np.int32)
    elif labels == "uniform":
        y = rng.integers(0, n_classes, size=(num_batches, batch), dtype=np.int32)
    else:
        raise ValueError(labels)
    return x, y


def to_f32_params(params: Sequence[np.ndarray]) -> List[np.ndarray]:
    """The fp32 copies the GPU consumes; the oracle is fed the SAME values widened to fp64."""
    return [np.ascontiguousarray(p, dtype=np.float32) for p in params]


def widen(params_f32: Sequence[np.ndarray]) -> List[np.ndarray]:
    return [np.asarray(p, dtype=np.float64) for p in params_f32]


def parity_inputs(model: Model, num_batches: int, batch: int, seed: int = 0,
                  labels: str = "teacher") -> Tuple[List[np.ndarray], np.ndarray, np.ndarray]:
    """(W0 per stage as fp32, X as fp32 [M,B,in], Y int32 [M,B]) — fp32-representable
    inputs so oracle (fp64) and GPU (fp32) start from bit-identical values. Images of
    conv models are NHWC, flattened per sample."""
    w0 = to_f32_params(glorot_params(model, seed))
    x, y = images_and_labels(model.layers[0].width_in, model.layers[-1].n_out, num_batches, batch,
                             seed + 1, labels)
    return w0, x.astype(np.float32), y
