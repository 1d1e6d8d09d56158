"""SpecTrain (arXiv 1809.02839) pipelined training step, B200-native.

The product is libspectrain.so (include/spectrain.h): hand-written sm_100a
kernels + NCCL between adjacent stages. This package is its thin Python binding.
"""
from ._lib import (ST_ACT_NONE, ST_ACT_RELU, ST_LAYER_CONV, ST_LAYER_DENSE, ST_LAYER_EMBED, ST_LAYER_LSTM, ST_LAYER_POOL, ST_BWD, ST_FWD, ST_GEMM_FP32X3, ST_GEMM_SIMT, ST_GEMM_TF32,
                   ST_MOMENTUM_EMA, ST_MOMENTUM_HEAVY_BALL, ST_PRED_NONE, ST_PRED_SPECTRAIN, ST_PRED_STASH, ST_PRED_STALENESS_FREE, ST_TRANSPORT_LOCAL,
                   ST_TRANSPORT_NCCL, ST_TRANSPORT_P2P, SpecTrainError, comm_plan, nccl_id, partition, program, version_difference)
from .stage import (Stage, connect_local, connect_p2p, connect_p2p_local, p2p_connect, p2p_export, dw_update_raw, gemm_raw, prediction_error_raw, run_group, softmax_ce_raw,
                    update_predict_raw)

__all__ = [
    "Stage", "connect_local", "connect_p2p", "connect_p2p_local", "p2p_connect", "p2p_export", "run_group", "gemm_raw", "prediction_error_raw", "dw_update_raw", "softmax_ce_raw", "update_predict_raw", "program",
    "comm_plan", "nccl_id", "partition", "version_difference", "SpecTrainError", "ST_FWD", "ST_BWD", "ST_ACT_NONE",
    "ST_ACT_RELU", "ST_LAYER_DENSE", "ST_LAYER_EMBED", "ST_LAYER_LSTM", "ST_LAYER_CONV", "ST_LAYER_POOL", "ST_PRED_SPECTRAIN", "ST_PRED_NONE", "ST_PRED_STASH", "ST_PRED_STALENESS_FREE", "ST_MOMENTUM_EMA", "ST_MOMENTUM_HEAVY_BALL",
    "ST_GEMM_FP32X3", "ST_GEMM_TF32", "ST_GEMM_SIMT", "ST_TRANSPORT_NCCL", "ST_TRANSPORT_LOCAL", "ST_TRANSPORT_P2P",
]
