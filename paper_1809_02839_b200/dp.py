"""Data-parallel comparator on the same kernels.

The paper's central throughput claim is pipelined model parallelism against data
parallelism: every GPU holds the whole model, takes
its shard of the global mini-batch, and the gradients are averaged across GPUs before
the (identical) momentum update — no weight prediction, no staleness (s ≡ 0). Here each
rank is a one-stage library context (the whole layer chain, ST_PRED_NONE); per step:

    st_stage_forward(mb) → st_stage_backward(mb) [writes G] →
    all-reduce(G, average) over the process group → st_predict_and_update

The forward / backward / K-B update run in the library's kernels; the all-reduce is
torch.distributed (NCCL on GPUs, gloo in tests) on the caller-owned G arena, ordered on
the stage's stream. One bucket per step (the whole G, no overlap with the backward):
the plain baseline the paper compares against, not a tuned DDP.

Reading (D23): with equal shards, averaging the per-shard batch-mean
gradients equals the gradient of the global batch mean, so N-way data parallelism with
per-rank batch B is sequential momentum SGD with batch N·B (pinned in
tests/test_oracle_pins.py).
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L
from .stage import Stage


class DataParallelStage:
    """One data-parallel replica: the whole model as a single library stage."""

    def __init__(self, layers, batch_per_rank: int, lr: float, gamma: float = 0.9,
                 momentum: int = L.ST_MOMENTUM_EMA, gemm: int = L.ST_GEMM_FP32X3, device: int = 0,
                 max_minibatches: int = 64, group: Optional[dist.ProcessGroup] = None, seq_len: int = 1):
        self.stage = Stage(layers, [], 0, batch_per_rank, lr, gamma, pred=L.ST_PRED_NONE, momentum=momentum,
                           gemm=gemm, transport=L.ST_TRANSPORT_NCCL, device=device,
                           max_minibatches=max_minibatches, seq_len=seq_len)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.G = self.stage.G[:4 * self.stage.params].view(torch.float32)
        self.mb = 0

    @property
    def stream(self) -> torch.cuda.Stream:
        return self.stage.stream

    def set_params(self, host: np.ndarray) -> None:
        self.stage.set_params(host)
        self.mb = 0

    def get_params(self):
        return self.stage.get_params()

    def allreduce_grad(self) -> None:
        if self.world == 1:
            return
        with torch.cuda.stream(self.stage.stream):  # ordered after the backward's G writes
            if dist.get_backend(self.group) == "nccl":
                dist.all_reduce(self.G, op=dist.ReduceOp.AVG, group=self.group)
            else:  # gloo: no AVG
                dist.all_reduce(self.G, op=dist.ReduceOp.SUM, group=self.group)
                self.G.div_(self.world)

    def step(self, x: torch.Tensor, y: torch.Tensor, want_loss: bool = False) -> Optional[float]:
        """One data-parallel training step on this rank's shard (x [B × in], y [B])."""
        loss = self.stage.forward(self.mb, x, y, want_loss=want_loss)
        self.stage.backward(self.mb)
        self.allreduce_grad()
        self.stage.predict_and_update()
        self.mb += 1
        return loss

    def run(self, xs: torch.Tensor, ys: torch.Tensor, want_losses: bool = False) -> Optional[np.ndarray]:
        out = []
        for i in range(xs.shape[0]):
            out.append(self.step(xs[i], ys[i], want_loss=want_losses))
        return np.array(out, np.float64) if want_losses else None

    def close(self) -> None:
        self.stage.close()
