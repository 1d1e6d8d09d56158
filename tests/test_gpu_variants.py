"""The kernel variants behind the development knobs (ST_GEMM_PAIR=0: single-CTA fwd / dX
kernel; ST_STREAM_K=1 with it: stream-K work split; the opt-in conv paths) against the
same fp64 references and the same pipeline parity gate as the default path. The product
library reads no knobs (csrc/knobs.hpp): these run the existing tests in a child pytest
against the development build (build.build_dev(), loaded through ST_LIB_PATH)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _dev_env(env):
    import importlib.util
    spec = importlib.util.spec_from_file_location("_st_build", os.path.join(ROOT, "paper_1809_02839_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    lib = b.build_dev()
    return dict(os.environ, ST_LIB_PATH=lib, **env)

CASES = [
    "tests/test_gpu_kernels.py::test_stage_gemms_vs_fp64",
    "tests/test_gpu_pipeline.py::test_deep_mlp_8stage",
    "tests/test_gpu_pipeline.py::test_ragged_shapes_and_M_smaller_than_depth",
    "tests/test_gpu_pipeline.py::test_mlp_2stage_config0",
]


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{"ST_GEMM_PAIR": "0"}, {"ST_GEMM_PAIR": "0", "ST_STREAM_K": "1"}],
                         ids=["single_cta", "stream_k"])
def test_gemm_variants_pass_parity(env):
    e = _dev_env(env)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "-k", "not tf32", *CASES], cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


CONV_CASES = ["tests/test_gpu_conv.py"]


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{"ST_CONV_PAIR": "0"}, {"ST_CONV_OVERLAP": "1"}, {"ST_TS_SPLIT_ACC": "0"},
                                 {"ST_TSG_NARROW": "0"}],
                         ids=["conv_single_cta", "conv_overlap", "one_accumulator", "tsg_4_stages"])
def test_conv_variants_pass_parity(env):
    """Non-default conv paths: the single-CTA conv forward, side-stream overlap of the conv dW +
    update, the single-accumulator pair kernel, the 4-stage TMEM-A ring for N ≤ 64."""
    e = _dev_env(env)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        *CONV_CASES], cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_lstm_persistent_recurrence_variant():
    """Development opt-in ST_LSTM_PERSIST=1: the LSTM recurrence as one persistent
    cooperative launch per layer and direction (k_lstm_rec.cu) — the LSTM parity tests
    (incl. the single-stage shapes and their launch-count invariant) and the full-size LM
    at one stage against the same gates."""
    e = _dev_env({"ST_LSTM_PERSIST": "1"})
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_lstm.py",
                        "tests/test_gpu_fullsize.py::test_lstm_lm_full_size_single_stage_bench_path"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_tall_forward_on_pair_kernel_variant():
    """ST_FWD_TSG=0: the tall dense forward (T·B rows) back on the CTA-pair kernel — the
    LSTM parity tests and the explicit-im2col conv cases against the same gates."""
    e = _dev_env({"ST_FWD_TSG": "0"})
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_lstm.py", "tests/test_gpu_conv.py"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
