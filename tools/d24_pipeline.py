"""Reading D24 for a whole pipelined run, without the GPU: the oracle's SpecTrain run
(O.run, every stage, every mini-batch, the paper's predictions) in NumPy float32 against
float64 on the inputs of a tests/test_gpu_fullsize.py case — the spread of V and ΔW that
fp32-faithful arithmetic alone produces through the ReLU / max-pool decisions.

    python tools/d24_pipeline.py {vgg16_8,vgg16_1,deep_mlp_N} [--M 10]   ->  profiles/r2_d24_<case>_M<M>.json
"""
import argparse, json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synthdata as sd  # noqa: E402
from oracle import spectrain_oracle as O  # noqa: E402


def oracle_float32():
    """A second copy of the oracle module whose `np.float64` is float32: its run() then keeps
    W, V, activations and gradients in float32 (NumPy float32 GEMMs and elementwise) — the
    same code in fp32 arithmetic, for this analysis only (the oracle itself is unchanged)."""
    import importlib.util
    import types
    spec = importlib.util.spec_from_file_location("oracle_fp32", os.path.join(ROOT, "oracle", "spectrain_oracle.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules["oracle_fp32"] = mod  # dataclasses look their module up
    spec.loader.exec_module(mod)
    np32 = types.ModuleType("numpy_fp32")
    np32.__dict__.update(np.__dict__)
    np32.float64 = np.float32
    mod.np = np32
    return mod


def rel(a, b):
    a, b = np.asarray(a, np.float64).ravel(), np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("case", choices=["deep_mlp_2", "deep_mlp_4", "deep_mlp_8", "vgg16_8", "vgg16_1"])
    ap.add_argument("--M", type=int, default=10)
    a = ap.parse_args()
    if a.case.startswith("deep_mlp"):  # bench.py's NCCL parity leg: 784-1024×8-10, B = 128, η = 0.02
        LR, B = 0.02, 128
        model = sd.config_deep_mlp(int(a.case.rsplit("_", 1)[1]))
    else:
        LR, B = 0.01, 128
        model = sd.config_vgg16(8 if a.case == "vgg16_8" else 1)
    w0, X, Y = sd.parity_inputs(model, a.M, B, seed=0)
    t0 = time.time()
    r64 = O.run(model, sd.widen(w0), X.astype(np.float64), Y, float(np.float32(LR)), float(np.float32(0.9)))
    t1 = time.time()
    r32 = oracle_float32().run(model, [np.asarray(w, np.float32) for w in w0], X.astype(np.float32), Y, float(np.float32(LR)),
                float(np.float32(0.9)))
    t2 = time.time()
    # the float32 copy must really have run in float32 (the conv / pool paths of the oracle
    # cast to float64 in places the module-level patch does not reach: refuse those cases)
    if np.concatenate(r32.V).dtype != np.float32:
        raise SystemExit(f"{a.case}: the float32 oracle copy did not stay in float32")
    W0 = np.concatenate(sd.widen(w0))
    W64, W32 = np.concatenate(r64.W), np.concatenate(r32.W)
    out = {"case": a.case, "M": a.M, "B": B, "lr": LR,
           "fp32_vs_fp64": {"loss": rel(r32.losses, r64.losses), "w": rel(W32, W64), "dw": rel(W32 - W0, W64 - W0),
                            "v": rel(np.concatenate(r32.V), np.concatenate(r64.V))},
           "dtype_check": str(np.concatenate(r32.V).dtype), "seconds": [round(t1 - t0, 1), round(t2 - t1, 1)]}
    path = os.path.join(ROOT, "profiles", f"r2_d24_{a.case}_M{a.M}.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1))
