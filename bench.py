#!/usr/bin/env python
"""Benchmark: SpecTrain pipelined training throughput on B200 (BASELINE.json metric
"training samples/sec at 1/2/4/8-stage pipeline; update-kernel HBM GB/s vs peak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N ...

A step = one mini-batch (B samples) through the whole pipeline: F on every
stage, loss, B on every stage, the fused K-B update on every stage. Workload
(config.workload): BASELINE.json configs[4], the large FCN (784 → 16 × 16384 → 10,
batch 128) — the one config BASELINE.json quotes at 1/2/4/8 stages — cut into N
contiguous stages, one stage per GPU (N=1: one stage, s_F = s_B = 0; --workload
picks the other configs). Warm-up and timed mini-batches run as ONE pipeline session
(`st_run` of W + K mini-batches); the timed window is the paper's steady-state window
(SURVEY §8(d)): CUDA events recorded on each rank's compute stream right after
its backward of mini-batch W−1 and of mini-batch W+K−1 (`st_record_after_backward`),
so K mini-batches complete inside it with the pipeline full; max over ranks. Weights
(16 GB) exceed L2 (126 MB), so no flush is needed between steps.

One JSON line on rank 0 (schema in the task contract), with `roofline` for the
dominant kernel (K-B), `cpu_baseline` (the oracle on the host cores), `e2e`
(st_run_host: host buffers, H2D/D2H inside the timed region) and `clocks`.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "training samples/sec at 1/2/4/8-stage pipeline; update-kernel HBM GB/s vs peak"
UNIT = "samples/s"
DEFAULT_GEMM = "fp32x3"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="large_fcn", choices=["wide_fcn", "large_fcn", "mlp", "deep_mlp", "lstm_lm", "vgg16"])
    p.add_argument("--stages", type=int, default=0, help="pipeline depth (default = --gpus); >N only with N=1")
    p.add_argument("--gemm", default=DEFAULT_GEMM, choices=["fp32x3", "tf32", "simt"])
    p.add_argument("--pred", default="spectrain", choices=["spectrain", "none", "stash", "staleness_free"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--lr", type=float, default=1e-3)
    p.add_argument("--partition", default="fixed", choices=["fixed", "auto", "profiled"],
                   help="fixed: the BJ / SURVEY §8(d) stage cuts; auto: st_partition over per-layer roofline "
                        "times; profiled: st_partition over per-layer times measured on this GPU (NEXT-4)")
    p.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                   help="on: every st_run session captured into one CUDA graph (st_set_graph_mode; contexts "
                        "linked with st_connect_local stay eager); auto (default): on at N = 1, off under torchrun")
    p.add_argument("--replicas", default="",
                   help="hybrid DP x PP (NEXT-4, P:380): comma list of replicas per stage, e.g. 2,1,1,1 — one "
                        "context per replica (N > 1: WORLD_SIZE = their sum, one per GPU; N = 1: co-located)")
    p.add_argument("--parallel", default="pp", choices=["pp", "dp"],
                   help="pp: the SpecTrain pipeline (default); dp: the data-parallel comparator (NEXT-1)")
    return p.parse_args()


def workload(name: str, S: int):
    import synthdata as sd
    if name == "wide_fcn":
        return sd.config_wide_fcn(S), 128, "wide_fcn_784-8x8192-10_b128"
    if name == "large_fcn":
        return sd.config_large_fcn(S), 128, "large_fcn_784-16x16384-10_b128"
    if name == "deep_mlp":
        return sd.config_deep_mlp(S), 128, "deep_mlp_784-8x1024-10_b128"
    if name == "vgg16":
        return sd.config_vgg16(S if S in (1, 8) else S), 128, "vgg16_cifar_32x32x3_b128"
    if name == "lstm_lm":
        return sd.config_lstm_lm(min(S, 4)), 128, "lstm_lm_v10k_h1500_2layer_t35_b128"
    return sd.mlp([784, 256, 256, 10], cuts=sd.even_cuts(3, S)), 32, "mlp_784-256-256-10_b32"


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def measured_tensor_peak():
    """Dense bf16 TF/s (MEASURED_PEAKS.json burst, else the guide's fallback) and the
    3xTF32 effective peak derived from it: tf32 = bf16 × 1.1/2.25 (nominal ratio), and
    one fp32-faithful product costs 3 tf32 MMAs."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            bf16 = float(json.load(f)["bf16_tflops"])
        src = "measured (MEASURED_PEAKS.json bf16_tflops)"
    except Exception:
        bf16, src = 1590.0, "fallback (B200_PROFILING.md 1.59 PFLOP/s bf16)"
    tf32 = bf16 * 1.1 / 2.25
    return bf16, tf32, tf32 / 3.0, src


def stage_work(model, k: int, B: int, pred: str):
    """Algorithmic HBM bytes and fp32 FLOPs of one mini-batch (F + B + update) on stage k
    (SURVEY §8(d)): per parameter 4 B read by F (Ŵ_F), 4 B by dX (Ŵ_B; none for the first
    layer of stage 0), 16 B for the update (W, V read + written) + 4 B per predicted copy
    written (WF if s_F > 0, WB if s_B > 0 and ≠ s_F); activations: each layer's input and
    output read / written once per pass (3 passes), fp32; the LM softmax logits 12 B each.
    FLOPs: 2·rows·in·out per GEMM pass (fwd, dX, dW; conv ×9·H·W, LSTM 4H·(in+H)·T)."""
    import synthdata as sd
    N = model.num_stages
    sF = {"spectrain": k // 2 + N - k - 1, "staleness_free": N - k - 1}.get(pred, 0)
    sB = {"spectrain": k // 2}.get(pred, 0)
    upd = 16 + (4 if sF > 0 else 0) + (4 if (sB > 0 and sB != sF) else 0)
    if pred == "stash":  # PipeDream weight stashing: the update writes W' into the stash slot
        upd = 20
    T = model.seq_len
    R = B * T
    byts, flops = 0.0, 0.0
    layers = model.stage_layers(k)
    for i, L in enumerate(layers):
        first = (k == 0 and i == 0)
        p = L.n_params
        if L.kind == sd.EMBED:
            byts += p * upd + 2 * R * L.n_out * 4 * 3
            continue
        passes = 2 if first else 3
        byts += p * (upd + 4 + (0 if first else 4))
        byts += 3 * R * (L.width_in + L.width_out) * 4
        if L.kind == sd.DENSE:
            flops += passes * 2.0 * R * L.n_in * L.n_out
        elif L.kind == sd.CONV:
            flops += passes * 2.0 * B * L.hw * L.hw * L.n_in * L.n_out * 9
        elif L.kind == sd.LSTM:
            flops += passes * 2.0 * R * (L.n_in + L.n_out) * 4 * L.n_out
            byts += 3 * R * 6 * L.n_out * 4  # gates + cell state stash
    if k == N - 1:
        byts += 12.0 * R * model.layers[-1].n_out
    return byts, flops


def auto_partition(model, B: int, S: int, hbm_gbs: float, tf32x3_tflops: float):
    """NEXT-4: stage cuts from st_partition over per-layer roofline times (the stage_work
    model for each layer alone: max(bytes / HBM, fp32 FLOPs / 3xTF32 peak), vanilla
    16 B/param update) instead of the fixed BJ partitions."""
    import dataclasses

    import paper_1809_02839_b200 as st
    import synthdata as sd
    costs = []
    for i, L in enumerate(model.layers):
        one = sd.Model((L,), (), model.loss, model.seq_len)
        b, f = stage_work(one, 0, B, "none")
        if i != 0:  # stage_work treats its first layer as the network's first (no dX)
            b += 4.0 * L.n_params
            if L.kind == sd.DENSE:
                f += 2.0 * B * model.seq_len * L.n_in * L.n_out
            elif L.kind == sd.CONV:
                f += 2.0 * B * L.hw * L.hw * L.n_in * L.n_out * 9
            elif L.kind == sd.LSTM:
                f += 2.0 * B * model.seq_len * (L.n_in + L.n_out) * 4 * L.n_out
        costs.append(max(b / (hbm_gbs * 1e9), f / (tf32x3_tflops * 1e12)))
    cuts, _ = st.partition(costs, S)
    return dataclasses.replace(model, cuts=tuple(cuts))


def profiled_partition(model, B: int, S: int, dev, lr: float, gemm: int, warm: int = 3, reps: int = 3):
    """NEXT-4, PipeDream-style: profile each layer on this GPU, then cut.
    The whole model runs as one library stage; with ST_PROF_LAYERS the engine brackets
    every layer's forward and (serialised) backward work with CUDA events
    (st_get_layer_profile); the per-layer cost is its mean forward + backward time over
    `reps` profiled mini-batches after `warm` unprofiled ones, and st_partition (min-max
    contiguous DP) turns the costs into S stages. Returns the re-cut model and the
    per-layer costs in µs."""
    import dataclasses

    import torch

    import paper_1809_02839_b200 as st
    import synthdata as sd
    kinds = {sd.DENSE: st.ST_LAYER_DENSE, sd.EMBED: st.ST_LAYER_EMBED, sd.LSTM: st.ST_LAYER_LSTM,
             sd.CONV: st.ST_LAYER_CONV, sd.POOL: st.ST_LAYER_POOL}
    layers = [(l.n_in, l.n_out, st.ST_ACT_RELU if l.act == sd.RELU else st.ST_ACT_NONE, 1 if l.bias else 0,
               kinds[l.kind], l.hw) for l in model.layers]
    whole = dataclasses.replace(model, cuts=())
    T = model.seq_len
    R = B * T
    M = warm + reps
    s = st.Stage(layers, [], 0, B, lr, 0.9, pred=st.ST_PRED_NONE, gemm=gemm, transport=st.ST_TRANSPORT_NCCL,
                 device=dev.index or 0, max_minibatches=M, seq_len=T)
    try:
        g = torch.Generator(device=dev)
        g.manual_seed(4321)
        init_params(s, whole.layers, dev, g)
        if model.layers[0].kind == sd.EMBED:
            xs = torch.randint(0, model.layers[0].n_in, (M, R), device=dev, dtype=torch.int32, generator=g)
        else:
            xs = torch.rand(M, R, model.layers[0].width_in, device=dev, generator=g)
        ys = torch.randint(0, model.layers[-1].n_out, (M, R), device=dev, dtype=torch.int32, generator=g)
        s.run(warm, xs[:warm], ys[:warm])
        s.set_layer_profiling(True)
        s.run(reps, xs[warm:], ys[warm:])
        ms, cnt = s.layer_profile()
        s.set_layer_profiling(False)
    finally:
        s.close()
    costs = [float(ms[i, 0] / max(1, cnt[i, 0]) + ms[i, 1] / max(1, cnt[i, 1])) for i in range(len(layers))]
    cuts, _ = st.partition(costs, S)
    return dataclasses.replace(model, cuts=tuple(cuts)), [round(c * 1e3, 1) for c in costs]


def pipeline_roofline(model, B: int, pred: str, hbm_gbs: float, tf32x3_tflops: float):
    """Per-stage roofline time t_k = max(bytes_k / HBM peak, flops_k / 3xTF32 peak) and the
    pipeline bound B / max_k t_k (SURVEY §8(d) 'Roofline definition')."""
    ts = []
    for k in range(model.num_stages):
        b, f = stage_work(model, k, B, pred)
        ts.append((max(b / (hbm_gbs * 1e9), f / (tf32x3_tflops * 1e12)), b, f))
    t_max = max(t for t, _, _ in ts)
    return {"samples_per_s": B / t_max, "stage_us": [round(t * 1e6, 1) for t, _, _ in ts],
            "bound": ["hbm" if b / (hbm_gbs * 1e9) >= f / (tf32x3_tflops * 1e12) else "tensor" for _, b, f in ts],
            "bytes_per_minibatch": [b for _, b, _ in ts], "fp32_flops_per_minibatch": [f for _, _, f in ts]}


def recorded_traffic(workload_name: str, kernel: str):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(workload_name, {}).get(kernel)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi-equivalent sampling through NVML during the timed region."""

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": getattr(nv, "nvmlClocksEventReasonGpuIdle", 0x1),
            "applications_clocks_setting": 0x2,
            "sw_power_cap": 0x4,
            "hw_slowdown": 0x8,
            "sync_boost": 0x10,
            "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80,
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for n, bit in names.items():
                    if r & bit and n != "gpu_idle":
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU oracle

def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def oracle_sample_rate(model_full, B: int, steps: int = 1, seed: int = 0, width_cap: int = 0):
    """Time the oracle as it stands on a bounded slice of the workload: a 1-stage
    784-w-w-10 net with the workload's hidden width w (capped at width_cap if > 0),
    `steps` mini-batches each (F, loss, B, update). Returns (samples/s extrapolated
    linearly in parameters to the full model, description, threads, per-step seconds)."""
    import synthdata as sd
    from oracle import spectrain_oracle as O
    w = max(l.n_out for l in model_full.layers[:-1]) if len(model_full.layers) > 1 else model_full.layers[0].n_out
    if width_cap:
        w = min(w, width_cap)
    slice_model = sd.mlp([model_full.layers[0].n_in, w, w, model_full.layers[-1].n_out], cuts=[])
    P_slice = sum(l.n_params for l in slice_model.layers)
    P_full = sum(l.n_params for l in model_full.layers)
    w0 = sd.glorot_params(slice_model, seed)
    X, Y = sd.images_and_labels(slice_model.layers[0].n_in, slice_model.layers[-1].n_out, steps, B, seed + 1,
                                "uniform")
    t0 = time.perf_counter()
    O.run(slice_model, w0, X, Y, 1e-3, 0.9)
    dt = time.perf_counter() - t0
    try:
        from threadpoolctl import threadpool_info
        threads = max(i.get("num_threads", 1) for i in threadpool_info()) if threadpool_info() else 1
    except Exception:
        threads = os.cpu_count() or 1
    rate = steps * B / dt * (P_slice / P_full)
    desc = (f"oracle.run (NumPy fp64) on a 1-stage {slice_model.layers[0].n_in}-{w}-{w}-"
            f"{slice_model.layers[-1].n_out} slice ({P_slice / 1e6:.1f}M params), {steps} mini-batch(es) of B={B} "
            f"in {dt:.2f} s measured; samples/s EXTRAPOLATED linearly in params to the {P_full / 1e6:.1f}M-param "
            f"workload")
    return rate, desc, threads, dt / steps


def cpu_baseline(model, B: int):
    """The oracle on the host cores (all BLAS threads), plus a 1-thread run on a
    narrower slice, the CPU model and the core count (SURVEY §8(d) 'Oracle timing')."""
    rate, desc, threads, step_s = oracle_sample_rate(model, B, 1)
    out = {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc,
           "slice_s_per_step": step_s, "cpu_model": cpu_model(), "nproc": os.cpu_count()}
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):
            r1, d1, _, s1 = oracle_sample_rate(model, B, 1, width_cap=2048)
        out["one_thread"] = {"value": r1, "unit": UNIT, "cores": 1, "sample": d1, "slice_s_per_step": s1}
    except Exception as e:  # report, never fail the bench line for the context number
        out["one_thread"] = {"error": repr(e)}
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    S = args.stages or args.gpus
    model, B, wname = workload(args.workload, S)
    # the oracle takes seconds per mini-batch on the wide FCN slice: warm-up and timed steps
    # share a wall-clock budget (ST_REF_BUDGET_S, default 150 s) so the arm ends within a few
    # minutes; at least one warm-up and one timed step always run, the count is reported
    budget = float(os.environ.get("ST_REF_BUDGET_S", "150"))
    t_start = time.perf_counter()
    for i in range(max(1, args.warmup)):
        if i > 0 and time.perf_counter() - t_start > budget / 3:
            break
        oracle_sample_rate(model, B, 1)
    rates, step_s = [], []
    desc, threads = "", 1
    for i in range(args.steps):
        if i > 0 and time.perf_counter() - t_start > budget:
            break
        r, desc, threads, s = oracle_sample_rate(model, B, 1)
        rates.append(r)
        step_s.append(s)
    value = float(statistics.mean(rates))
    desc += f"; {len(rates)} timed step(s) of the requested {args.steps} (wall-clock budget {budget:.0f} s)"
    slice_s = float(sum(step_s))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "timed_steps": len(rates), "warmup": args.warmup, "ms_per_step": B / value * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wname, "stages": S, "batch": B, "parallelism": f"pp{S}"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc,
                         "cpu_model": cpu_model(), "nproc": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "measured_wall_s": slice_s,
        "note": "ms_per_step is B / value (the extrapolated full-model rate); measured_wall_s is the measured oracle "
                "time of the timed slice steps",
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm

def init_params(s, layers, dev, g):
    """Bench-only device-side Glorot / embedding / LSTM init of one stage's arena."""
    import torch
    import synthdata as sd
    w = torch.empty(s.params, device=dev)
    off = 0
    for L in layers:
        if L.kind == sd.POOL:
            pass
        elif L.kind == sd.CONV:
            r = (6.0 / (9 * L.n_in + 9 * L.n_out)) ** 0.5
            w[off:off + 9 * L.n_in * L.n_out].uniform_(-r, r, generator=g)
            w[off + 9 * L.n_in * L.n_out:off + L.n_params].zero_()
        elif L.kind == sd.EMBED:
            w[off:off + L.n_params].uniform_(-0.1, 0.1, generator=g)
        elif L.kind == sd.LSTM:
            h = L.n_out
            r1, r2 = (6.0 / (L.n_in + 4 * h)) ** 0.5, (6.0 / (5 * h)) ** 0.5
            w[off:off + L.n_in * 4 * h].uniform_(-r1, r1, generator=g)
            w[off + L.n_in * 4 * h:off + (L.n_in + h) * 4 * h].uniform_(-r2, r2, generator=g)
            w[off + (L.n_in + h) * 4 * h:off + L.n_params].zero_()
        else:
            r = (6.0 / (L.n_in + L.n_out)) ** 0.5
            w[off:off + L.n_in * L.n_out].uniform_(-r, r, generator=g)
            w[off + L.n_in * L.n_out:off + L.n_params].zero_()
        off += L.n_params
    s.set_params(w.cpu().numpy())
    del w


def run_dp(args):
    """NEXT-1 comparator (paper_1809_02839_b200/dp.py): N data-parallel replicas of the
    whole model, per-rank batch B (weak scaling: global batch N·B), G averaged by an
    NCCL all-reduce (one bucket) before the K-B update; s ≡ 0."""
    import torch
    import torch.distributed as dist

    import paper_1809_02839_b200 as st
    import synthdata as sd
    from paper_1809_02839_b200.dp import DataParallelStage
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    N = args.gpus
    if world != N:
        raise SystemExit(f"--gpus {N} but WORLD_SIZE={world}: launch N>1 with torchrun")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if N > 1:
        dist.init_process_group("nccl", device_id=dev)
    model, B, wname = workload(args.workload, 1)
    if model.seq_len != 1 or any(l.kind != sd.DENSE for l in model.layers):
        raise SystemExit("--parallel dp: dense workloads only")
    layers = [(l.n_in, l.n_out, st.ST_ACT_RELU if l.act == sd.RELU else st.ST_ACT_NONE, 1 if l.bias else 0)
              for l in model.layers]
    K, W_ = args.steps, args.warmup
    r = DataParallelStage(layers, B, args.lr, 0.9, device=local, max_minibatches=K + W_)
    g = torch.Generator(device=dev)
    g.manual_seed(1234)  # identical replicas
    init_params(r.stage, model.layers, dev, g)
    g.manual_seed(99 + rank)  # each rank its own shard
    xs = torch.rand(K + W_, B, model.layers[0].n_in, device=dev, generator=g)
    ys = torch.randint(0, model.layers[-1].n_out, (K + W_, B), device=dev, dtype=torch.int32, generator=g)

    def barrier():
        torch.cuda.synchronize()
        if N > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(W_):
        r.step(xs[i], ys[i])
    barrier()
    l0 = r.stage.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    with sampler:
        e0.record(r.stream)
        for i in range(W_, W_ + K):
            r.step(xs[i], ys[i])
        e1.record(r.stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    launches = r.stage.kernel_launches() - l0
    if N > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = N * B * K / (ms / 1e3)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": K, "warmup": W_,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": wname, "parallelism": f"dp{N}", "batch_per_rank": B, "global_batch": N * B,
                       "gemm": args.gemm, "allreduce": "one NCCL all-reduce (AVG) of the whole G per step",
                       "role": "NEXT-1 comparator (data parallelism on the same kernels), not the headline"},
            "gpu_launches": launches, "clocks": sampler.summary()}), flush=True)
    r.close()
    if N > 1:
        dist.destroy_process_group()


def nccl_parity_leg(args, N: int, rank: int, local: int, dev):
    """Under torchrun (N > 1), before timing: the NCCL transport checked on the real
    ranks — the deep MLP 784-1024×8-10 cut into N stages, one per
    rank over NCCL (two communicators, comm streams), M = 20, B = 128, η = 0.02, 3xTF32,
    against the oracle on rank 0: trace bit-exact, W and loss rel-L2 ≤ 1e-4 (north_star
    gates) and ΔW = W − W0 rel-L2 ≤ 1e-2. The ΔW gate follows reading D24: the oracle's own
    arithmetic in float32 spreads ΔW from its float64 run by 2.3e-3 / 3.8e-3 / 1.0e-3 at
    N = 2 / 4 / 8 on exactly these inputs (tools/d24_pipeline.py deep_mlp_N --M 20 →
    profiles/r2_d24_deep_mlp_N_M20.json: ReLU decisions within rounding of 0), so the
    gate is above 2x that spread (a skipped update gives ΔW rel-L2 = 1)."""
    import torch
    import torch.distributed as dist

    import paper_1809_02839_b200 as st
    import synthdata as sd
    model = sd.config_deep_mlp(N)
    M, B, lr = 20, 128, 0.02
    w0, X, Y = sd.parity_inputs(model, M, B, seed=0)
    obj = [st.nccl_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    layers = [(l.n_in, l.n_out, st.ST_ACT_RELU if l.act == sd.RELU else st.ST_ACT_NONE, 1 if l.bias else 0)
              for l in model.layers]
    s = st.Stage(layers, model.cuts, rank, B, lr, 0.9, transport=st.ST_TRANSPORT_NCCL, device=local,
                 max_minibatches=M, nccl_id=obj[0])
    s.set_params(w0[rank])
    xs = torch.from_numpy(X).to(dev) if s.is_first else None
    ys = torch.from_numpy(Y.astype(np.int32)).to(dev) if s.is_last else None
    t0 = time.perf_counter()
    losses = s.run(M, xs, ys, want_losses=s.is_last)
    W, _, _ = s.get_params()
    wall = time.perf_counter() - t0
    tr = s.trace()
    s.close()
    got = [None] * N if rank == 0 else None
    dist.gather_object((W, tr, losses), got, dst=0)
    if rank != 0:
        return None
    from oracle import spectrain_oracle as O
    ref = O.run(model, sd.widen(w0), X.astype(np.float64), Y, float(np.float32(lr)), float(np.float32(0.9)))

    def rel(a, b):
        return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))
    Wg = np.concatenate([g[0] for g in got])
    Wr = np.concatenate(ref.W)
    trace_ok = all(got[k][1] == [e.as_tuple() for e in ref.trace[k]] for k in range(N))
    rw = rel(Wg, Wr)
    rl = rel(got[N - 1][2], ref.losses)
    dw = rel(Wg - np.concatenate(w0), Wr - np.concatenate(sd.widen(w0)))
    return {"model": "deep_mlp_784-1024x8-10_b128", "stages": N, "minibatches": M, "transport": "nccl (2 comms)",
            "trace_bit_exact": bool(trace_ok), "w_rel_l2": rw, "loss_rel_l2": rl, "dw_rel_l2": dw,
            "gates": {"w": 1e-4, "loss": 1e-4, "dw": 1e-2},
            "pass": bool(trace_ok and rw <= 1e-4 and rl <= 1e-4 and dw <= 1e-2), "wall_s": wall}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1809_02839_b200 as st
    import synthdata as sd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    N = args.gpus
    if world != N:
        raise SystemExit(f"--gpus {N} but WORLD_SIZE={world}: launch N>1 with torchrun")
    reps = [int(v) for v in args.replicas.split(",")] if args.replicas else None
    if reps:
        S = len(reps)
        if args.stages and args.stages != S:
            raise SystemExit("--stages must equal the number of --replicas entries")
        if N > 1 and sum(reps) != N:
            raise SystemExit(f"--replicas {args.replicas}: WORLD_SIZE must be {sum(reps)} (one context per GPU)")
    else:
        S = args.stages or N
        if N > 1 and S != N:
            raise SystemExit("--stages must equal --gpus when N > 1")
    shared_gpu = N > 1 and os.environ.get("ST_BENCH_SHARED_GPU") == "1"
    if shared_gpu:
        # validation of the torchrun path on a one-GPU box (tools/gpu_torchrun.sh): every rank
        # on cuda:0, each rank its own NCCL "host" so NCCL accepts two ranks on one device.
        # The ranks time-slice the GPU: the numbers are not a scaling measurement.
        os.environ["NCCL_HOSTID"] = f"st-bench-host-{rank}"
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if N > 1:
        dist.init_process_group("nccl", device_id=dev)
    model, B, wname = workload(args.workload, S)
    gemm = {"fp32x3": st.ST_GEMM_FP32X3, "tf32": st.ST_GEMM_TF32, "simt": st.ST_GEMM_SIMT}[args.gemm]
    layer_cost_us = None
    if args.partition == "auto" and S > 1:
        hbm_, _ = measured_peaks()
        model = auto_partition(model, B, S, hbm_, measured_tensor_peak()[2])
    elif args.partition == "profiled" and S > 1:
        # every rank profiles the same model on its own GPU; rank 0's cut is broadcast
        model_p, layer_cost_us = profiled_partition(model, B, S, dev, args.lr, gemm)
        obj = [list(model_p.cuts) if rank == 0 else None]
        if N > 1:
            dist.broadcast_object_list(obj, src=0)
        import dataclasses
        model = dataclasses.replace(model, cuts=tuple(obj[0]))
    pred = {"spectrain": st.ST_PRED_SPECTRAIN, "none": st.ST_PRED_NONE, "stash": st.ST_PRED_STASH,
            "staleness_free": st.ST_PRED_STALENESS_FREE}[args.pred]
    kinds = {sd.DENSE: st.ST_LAYER_DENSE, sd.EMBED: st.ST_LAYER_EMBED, sd.LSTM: st.ST_LAYER_LSTM,
             sd.CONV: st.ST_LAYER_CONV, sd.POOL: st.ST_LAYER_POOL}
    layers = [(l.n_in, l.n_out, st.ST_ACT_RELU if l.act == sd.RELU else st.ST_ACT_NONE, 1 if l.bias else 0,
               kinds[l.kind], l.hw) for l in model.layers]
    T = model.seq_len
    R = B * T
    W_, K = args.warmup, args.steps
    if K < 1:
        raise SystemExit("--steps must be >= 1")
    M = W_ + K  # one session: W warm-up mini-batches, then the K timed ones

    if reps:
        # stage-major contexts: context i = (stage k, replica r); NCCL rank i = i (one per GPU)
        ctx_of = [(k, r) for k in range(S) for r in range(reps[k])]
        if N > 1:
            obj = [st.nccl_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            k, r = ctx_of[rank]
            my_stages = [st.Stage(layers, model.cuts, k, B, args.lr, 0.9, pred=pred, gemm=gemm,
                                  transport=st.ST_TRANSPORT_NCCL, device=local, max_minibatches=M, nccl_id=obj[0],
                                  seq_len=T, replicas=reps, replica=r)]
        else:
            my_stages = [st.Stage(layers, model.cuts, k, B, args.lr, 0.9, pred=pred, gemm=gemm,
                                  transport=st.ST_TRANSPORT_LOCAL, device=local, max_minibatches=M, seq_len=T,
                                  replicas=reps, replica=r) for k, r in ctx_of]
            st.connect_local(my_stages)
    elif N > 1:
        obj = [st.nccl_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        my_stages = [st.Stage(layers, model.cuts, rank, B, args.lr, 0.9, pred=pred, gemm=gemm,
                              transport=st.ST_TRANSPORT_NCCL, device=local, max_minibatches=M, nccl_id=obj[0],
                              seq_len=T)]
    elif S == 1:
        my_stages = [st.Stage(layers, model.cuts, 0, B, args.lr, 0.9, pred=pred, gemm=gemm,
                              transport=st.ST_TRANSPORT_NCCL, device=local, max_minibatches=M, seq_len=T)]
    else:
        my_stages = [st.Stage(layers, model.cuts, k, B, args.lr, 0.9, pred=pred, gemm=gemm,
                              transport=st.ST_TRANSPORT_LOCAL, device=local, max_minibatches=M, seq_len=T)
                     for k in range(S)]
        st.connect_local(my_stages)

    use_graph = args.graph == "on" or (args.graph == "auto" and N == 1)
    if use_graph:
        for s in my_stages:
            s.set_graph_mode(True)
    # parameters: Glorot on device (bench-only, SURVEY §8(d) seeds), labels uniform
    for s in my_stages:  # seeded per stage: the replicas of a stage start identical
        gk = torch.Generator(device=dev)
        gk.manual_seed(1234 + s.k)
        init_params(s, model.stage_layers(s.k), dev, gk)
    g = torch.Generator(device=dev)
    g.manual_seed(4321)
    n_in, n_cls = model.layers[0].width_in, model.layers[-1].n_out
    first = my_stages[0].is_first
    last = my_stages[-1].is_last
    if model.layers[0].kind == sd.EMBED:
        xs = torch.randint(0, n_in, (M, R), device=dev, dtype=torch.int32, generator=g) if first else None
    else:
        xs = torch.rand(M, R, n_in, device=dev, generator=g) if first else None
    ys = torch.randint(0, n_cls, (M, R), device=dev, dtype=torch.int32, generator=g) if last else None

    def barrier():
        torch.cuda.synchronize()
        if N > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def session(n: int, host=None):
        if host is not None:
            my_stages[0].run_host(n, *host)
        elif len(my_stages) == 1:
            my_stages[0].run(n, xs, ys)
        else:
            st.run_group(my_stages, n, xs, ys, want_losses=False)

    def windowed(host=None):
        """One session of M = W + K mini-batches; returns the CUDA-event time between
        stage 0's (this rank's) backward of mini-batch W−1 and of mini-batch M−1 —
        the paper's steady-state window."""
        s0 = my_stages[0]
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        if W_ >= 1:
            s0.record_after_backward(W_ - 1, e0)
        else:
            e0.record(s0.stream)
        s0.record_after_backward(M - 1, e1)
        session(M, host)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    def max_over_ranks(x: float) -> float:
        if N == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    nccl_parity = nccl_parity_leg(args, N, rank, local, dev) if (N > 1 and not reps) else None

    # the timed session: only the dominant kernel class is bracketed with CUDA events
    # (two event records per launch; events pre-created); the all-class breakdown comes
    # from a separate short session after it
    for s in my_stages:
        s.set_profiling(True, ["gemm_dw"])
    launches0 = sum(s.kernel_launches() for s in my_stages)
    sampler = ClockSampler(local)
    barrier()
    with sampler:
        ms = windowed()
    barrier()
    launches = sum(s.kernel_launches() for s in my_stages) - launches0
    profs = [s.profile() for s in my_stages]
    # breakdown session (not timed for `value`): every kernel class bracketed
    n_brk = min(K, 20)
    for s in my_stages:
        s.set_profiling(True)
    barrier()
    session(n_brk)
    barrier()
    brk = [s.profile() for s in my_stages]
    for s in my_stages:
        s.set_profiling(False)
    # per-stage busy time (compute classes, comm excluded) of the breakdown session
    busy_local = [((s.k, s.replica), sum(p[c][0] for c in ("update", "gemm_fwd", "gemm_dx", "gemm_dw", "loss"))
                   / n_brk) for s, p in zip(my_stages, brk)]
    if N > 1:
        allb = [None] * N
        dist.all_gather_object(allb, busy_local)
        busy_local = [b for part in allb for b in part]
    busy_ms = [b for _, b in sorted(busy_local)]
    stage_busy = {"ms_per_minibatch": [round(b, 4) for b in busy_ms],
                  "imbalance_max_over_mean": round(max(busy_ms) * len(busy_ms) / sum(busy_ms), 3) if sum(busy_ms) > 0
                  else None,
                  "note": "per stage: its fwd / dX / dW+update GEMM, loss and update kernel time per mini-batch "
                          "(CUDA events, breakdown session, comm excluded); the step can be no faster than the "
                          "busiest stage (P:460-470)"}
    t_max = max_over_ranks(ms)
    if N > 1:
        lt = torch.tensor([launches], device=dev, dtype=torch.int64)
        dist.all_reduce(lt, op=dist.ReduceOp.SUM)
        launches = int(lt.item())
    value = K * B / (t_max / 1e3)

    # roofline of the dominant kernel: the dW GEMM with the fused K-B update
    # (k_gemm_tc.cu tc_dw_kernel<x3, UPD> + its lo-split and bias-update launches — the
    # engine's "gemm_dw" class). Algorithmic bytes per launch = the update stream of that
    # layer: read W, V + write W, V [+ WF] [+ WB] = 16 / 20 / 24 B per parameter
    # (operand reads of dZ and X, ~B·(in+out)·8 B, are left out: < 1%).
    kb_bytes, kb_ms, kb_n, stage_ms = 0.0, 0.0, 0, 0.0
    for s, pr in zip(my_stages, profs):
        bpp = 16 + (4 if s.sizes.wf_bytes > 0 else 0) + (4 if s.sizes.wb_bytes > 0 else 0)  # + WF / WB (or stash) writes
        ms_k, n_k = pr["gemm_dw"]
        kb_bytes += bpp * s.params * M  # the class is bracketed over the whole session (M mini-batches)
        kb_ms += ms_k
        kb_n += n_k
        stage_ms += sum(v[0] for v in brk[my_stages.index(s)].values())
    brk_dw = sum(p["gemm_dw"][0] for p in brk) / n_brk
    agg = torch.tensor([kb_bytes, kb_ms, kb_n, stage_ms / n_brk, brk_dw], device=dev, dtype=torch.float64)
    if N > 1:
        dist.all_reduce(agg)
    kb_bytes, kb_ms, kb_n, stage_ms, brk_dw = [float(v) for v in agg.tolist()]
    peak, peak_src = measured_peaks()
    achieved = kb_bytes / (kb_ms / 1e3) / 1e9 if kb_ms > 0 else None
    bf16_pk, tf32_pk, x3_pk, tpk_src = measured_tensor_peak()
    roof = pipeline_roofline(model, B, args.pred, peak, x3_pk)
    # GEMM tensor fraction: the forward GEMM class (fp32-faithful 3xTF32 products) of the
    # breakdown session, algorithmic fp32 FLOPs of the forward pass of every rank's stages
    fwd_flops = 0.0
    for s_ in my_stages:
        import synthdata as sd
        for i, L in enumerate(model.stage_layers(s_.k)):
            if L.kind == sd.DENSE:
                fwd_flops += 2.0 * R * L.n_in * L.n_out
            elif L.kind == sd.CONV:
                fwd_flops += 2.0 * B * L.hw * L.hw * L.n_in * L.n_out * 9
            elif L.kind == sd.LSTM:
                fwd_flops += 2.0 * R * (L.n_in + L.n_out) * 4 * L.n_out
    fwd_ms = sum(p["gemm_fwd"][0] for p in brk) / n_brk
    gf = torch.tensor([fwd_flops, fwd_ms], device=dev, dtype=torch.float64)
    if N > 1:
        dist.all_reduce(gf)
    fwd_flops, fwd_ms = [float(v) for v in gf.tolist()]
    gemm_tf = fwd_flops / (fwd_ms / 1e3) / 1e12 if fwd_ms > 0 else None
    gemm_prof = {k: round(sum(p[k][0] for p in brk) / n_brk, 4) for k in brk[0]}

    # end-to-end: the same metric through st_run_host (pinned host inputs, per-mini-batch H2D
    # and loss D2H inside the same steady-state window)
    e2e = None
    if not args.no_e2e and len(my_stages) == 1:
        s = my_stages[0]
        xh = xs.cpu().pin_memory() if first else None
        yh = ys.cpu().pin_memory() if last else None
        lh = torch.empty(M, dtype=torch.float32).pin_memory() if last else None
        barrier()
        ems = max_over_ranks(windowed((xh, yh, lh)))
        barrier()
        x_bytes = R * 4 if model.layers[0].kind == sd.EMBED else R * n_in * 4
        e2e = {"value": K * B / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": (x_bytes if first else 0) + (R * 4 if last else 0),
               "d2h_bytes_per_step": 4 if last else 0,
               "api": "st_run_host (same W + K session and window as `value`)"}

    # dominant kernel class = the gemm_dw class (largest share on every workload). FCN / MLP:
    # the fused dW + K-B update, HBM-bound (bytes above). Conv / LSTM workloads: the dW GEMMs
    # (implicit-conv dW, tall dense dW on the TMEM-A kernel) are tensor-bound: fp32 FLOPs of
    # the dW pass ÷ the class time, against the 3xTF32 effective peak.
    if args.workload in ("vgg16", "lstm_lm"):
        dw_flops = 0.0
        for s_ in my_stages:
            for L in model.stage_layers(s_.k):
                if L.kind == sd.DENSE:
                    dw_flops += 2.0 * R * L.n_in * L.n_out
                elif L.kind == sd.CONV:
                    dw_flops += 2.0 * B * L.hw * L.hw * L.n_in * L.n_out * 9
                elif L.kind == sd.LSTM:
                    dw_flops += 2.0 * R * (L.n_in + L.n_out) * 4 * L.n_out
        t_ = torch.tensor([dw_flops], device=dev, dtype=torch.float64)
        if N > 1:
            dist.all_reduce(t_)
        dw_flops = float(t_.item())
        ach_t = dw_flops * M / (kb_ms / 1e3) / 1e12 if kb_ms > 0 else None
        roofline_key = {"kernel": "gemm_dw class: k_gemm_tc.cu tc_tsg_kernel (implicit-conv dW / tall dense dW, "
                                  "3xTF32) + the K-B update of those layers",
                        "bound": "tensor", "achieved": ach_t, "peak": x3_pk, "unit": "TFLOP/s",
                        "frac": (ach_t / x3_pk) if ach_t else None, "traffic": None,
                        "peak_source": tpk_src + "; fp32 FLOP/s of 3xTF32 products = tf32 peak / 3",
                        "launches": int(kb_n), "per": "all dW launches of one step",
                        "ms_per_step": kb_ms / M,
                        "share_of_stage_time": (brk_dw / stage_ms) if stage_ms else None,
                        "algorithmic_flops_per_step": dw_flops}
    else:
        roofline_key = {"kernel": "k_gemm_tc.cu tc_dw_kernel<FP32X3, fused K-B update> (dW + Eq.1/apply/predict)",
                        "bound": "hbm",
                        "achieved": achieved, "peak": peak, "unit": "GB/s",
                        "frac": (achieved / peak) if achieved else None,
                        "traffic": recorded_traffic(wname, "dw_update_per_step"),
                        "peak_source": peak_src, "launches": int(kb_n),
                        "per": "all dW+update launches of one step (one per layer)",
                        "ms_per_step": kb_ms / M,
                        "share_of_stage_time": (brk_dw / stage_ms) if stage_ms else None,
                        "algorithmic_bytes_per_step": kb_bytes / M}
    if rank == 0:
        cpu = None
        if not args.no_cpu and N == 1:  # the oracle baseline: rank 0 at N = 1 only
            cpu = cpu_baseline(model, B)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": K,
            "warmup": W_, "ms_per_step": t_max / K, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": wname, "stages": S, "batch": B, "seq_len": T, "gemm": args.gemm, "pred": args.pred,
                       "cuts": list(model.cuts), "partition": args.partition,
                       **({"layer_cost_us": layer_cost_us} if layer_cost_us else {}),
                       "parallelism": (f"pp{S}" if not reps else f"pp{S}xdp" + "-".join(map(str, reps))),
                       **({"replicas": reps} if reps else {}),
                       **({"shared_gpu_validation": "all ranks on one GPU: not a scaling number"} if shared_gpu else {}),
                       "cuda_graph": use_graph, "l2": "no flush: per-step working set (weights) >> 126 MB L2",
                       "session": "one 1F1B session of warmup + steps mini-batches; timed window = CUDA events "
                                  "after stage 0's B(warmup-1) and B(warmup+steps-1) (P:415 steady state)"},
            "roofline": roofline_key,
            "pipeline_roofline": {"samples_per_s": roof["samples_per_s"], "frac": value / roof["samples_per_s"],
                                  "stage_us": roof["stage_us"], "stage_bound": roof["bound"],
                                  "peaks": {"hbm_gbs": peak, "tf32x3_tflops": x3_pk, "source": [peak_src, tpk_src]},
                                  "model": "t_k = max(bytes_k / HBM, fp32 flops_k / (tf32 peak / 3)); "
                                           "bench.py stage_work(), SURVEY §8(d)"},
            "gemm_tensor": {"class": "gemm_fwd (k_gemm_tc.cu tc_ts2_kernel<FWD> + split-K epilogue)",
                            "achieved_tflops": gemm_tf, "peak_tflops": x3_pk,
                            "frac": (gemm_tf / x3_pk) if gemm_tf else None,
                            "unit": "fp32 TFLOP/s (each product = 3 tf32 MMAs; peak = tf32 / 3)",
                            "tf32_peak_tflops": tf32_pk, "bf16_peak_tflops": bf16_pk},
            "paper_context": "context only (4x P40 over PCIe, TensorFlow; BASELINE.md §1): pipelined MP over DP "
                             "8.91x best (FCN/RNN), 3.10x FCN/RNN average, +98.5% average over 6 models; "
                             "no absolute samples/s published",
            "kernel_ms_per_step": gemm_prof,
            "stage_busy": stage_busy,
            "kernel_ms_note": f"per kernel class, ms per mini-batch, from a separate {n_brk}-mini-batch session "
                              "with every class bracketed (rank 0's stages)",
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(round(launches * K / M)),
            "gpu_launches_note": f"library kernel launches of the {M}-mini-batch session x {K}/{M} (timed share)",
            "nccl_parity": nccl_parity,
            "clocks": sampler.summary(),
        }
        print(json.dumps(line), flush=True)
    for s in my_stages:
        s.close()
    if N > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    # diagnostics only: if a run stalls, dump every thread's Python stack to stderr
    # (repeating; never kills the run)
    import faulthandler
    faulthandler.dump_traceback_later(float(os.environ.get("ST_BENCH_WATCHDOG_S", "240")), repeat=True)
    if args.impl == "reference":
        run_reference(args)
    elif args.parallel == "dp":
        run_dp(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
