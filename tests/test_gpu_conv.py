"""VGG conv stages on the GPU (-m gpu): 3×3 convolution (im2col + tcgen05 GEMMs,
col2im gather), ReLU, 2×2 max-pool and the FC head through the C-ABI, against the
fp64 oracle. Gates: trace bit-exact, W and loss ≤ 1e-4 rel-L2."""
import numpy as np
import pytest
import torch

import synthdata as sd
from tests.gpu_helpers import assert_parity, build_pipeline, oracle_run, rel_l2, run_pipeline

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def st():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1809_02839_b200 as st
    return st


def _vgg_parity(st, model, batch, M, lr, seed=0, gemm=None):
    w0, X, Y = sd.parity_inputs(model, M, batch, seed)
    stages = build_pipeline(model, batch, lr, gemm=gemm, max_mb=M)
    try:
        res = run_pipeline(stages, w0, X, Y)
    finally:
        for s in stages:
            s.close()
    ref = oracle_run(model, w0, X, Y, lr)
    assert_parity(model, res, ref)
    assert rel_l2(np.concatenate(ref.W), np.concatenate(sd.widen(w0))) > 1e-4


def test_vgg_small_4stage_tma_widths(st):
    """conv(4→8) pool conv(8→16) conv(16→16) pool FC — channel counts whose im2col
    widths (9·C) take the TMA / tcgen05 path; pools at stage boundaries and inside."""
    model = sd.vgg(cfg=(8, "M", 16, 16, "M"), fc=(32,), classes=10, hw=16, in_ch=4, cuts=[1, 3, 5])
    _vgg_parity(st, model, 8, 10, 0.05)


def test_vgg_small_single_stage_rgb(st):
    """RGB input (9·3 = 27-wide im2col: CUDA-core GEMM path) on one stage, and a
    stage that starts with a pool (mask of the previous stage's conv applied there)."""
    model = sd.vgg(cfg=(8, 8, "M", 16, "M"), fc=(16,), classes=10, hw=8, in_ch=3, cuts=[])
    _vgg_parity(st, model, 4, 8, 0.05, seed=1)
    model = sd.vgg(cfg=(8, "M", 16, "M"), fc=(16,), classes=10, hw=8, in_ch=4, cuts=[1, 2])
    _vgg_parity(st, model, 4, 8, 0.05, seed=2)


def test_vgg_simt_mode(st):
    model = sd.vgg(cfg=(8, "M", 16, "M"), fc=(16,), classes=10, hw=8, in_ch=4, cuts=[2])
    _vgg_parity(st, model, 4, 6, 0.05, seed=3, gemm=st.ST_GEMM_SIMT)


# Implicit-GEMM conv path (channel counts multiples of 32: 4-D TMA windows, no im2col).
# Geometries: 16×16 (pixel box 8 rows × 16), 8×8 (2 images × 8 × 8), 4×4 (8 images),
# 2×2 (32 images); batch 3 makes every P = 3·H·W tile ragged except at 16×16.

def test_vgg_implicit_conv_3stage(st):
    model = sd.vgg(cfg=(32, 32, "M", 64, "M", 64, "M", 32, "M"), fc=(32,), classes=10, hw=16, in_ch=32,
                   cuts=[2, 5])
    _vgg_parity(st, model, 3, 10, 0.05, seed=4)


def test_vgg_implicit_after_rgb(st):
    """3-channel first conv (CUDA-core im2col path) feeding implicit convs; dX of the
    implicit conv carries the ReLU mask of its producer across a stage boundary."""
    model = sd.vgg(cfg=(32, "M", 32, 64, "M", 64), fc=(16,), classes=10, hw=8, in_ch=3, cuts=[1, 3])
    _vgg_parity(st, model, 5, 8, 0.05, seed=5)


def test_vgg_implicit_batch1(st):
    """FP32X3 (the parity mode) at batch 1 — single-image tiles, P < 128 everywhere."""
    model = sd.vgg(cfg=(32, "M", 64, "M"), fc=(16,), classes=10, hw=8, in_ch=32, cuts=[])
    _vgg_parity(st, model, 1, 6, 0.05, seed=6)


def test_vgg_wide_conv_pair_kernel(st):
    """Cout ≥ 256 (256 / 384 channels). By default (ST_CONV_PAIR=0 in the dev build, run by
    tests/test_gpu_variants.py, selects the single-CTA kernel) the conv forward is the CTA-pair TMEM-A kernel (weights on M,
    64-pixel window boxes per CTA, activation lo split once); 384 output channels leave a
    padding CTA in the last pair; 8×8 and 4×4 images, ragged pixel tiles (batch 3)."""
    model = sd.vgg(cfg=(32, 384, "M", 256, "M"), fc=(16,), classes=10, hw=8, in_ch=32, cuts=[2])
    _vgg_parity(st, model, 3, 8, 0.02, seed=7)  # 4×4 stage: P = 48 < 128 → single-CTA kernel
    model = sd.vgg(cfg=(32, 256, 256, "M"), fc=(16,), classes=10, hw=8, in_ch=32, cuts=[1])
    _vgg_parity(st, model, 5, 6, 0.02, seed=8)  # P = 320: two full and one ragged pixel tile
