"""Small round-2 scenarios for compute-sanitizer (profiles/sanitizer/r2_*):
  hybrid  — co-located hybrid DP x PP (stage 0 replicated x2, LOCAL, in-place replica reduce)
  graph   — graph-captured sessions (MLP and an LSTM LM, two sessions each)
  p2p_rank <rank> <port> <dir> — one rank of a 2-stage P2P pipeline (CUDA IPC); run each
            rank as its own process under compute-sanitizer
  layers  — per-layer profiling session"""
import os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from pathlib import Path

if __name__ == "__main__":
    what = sys.argv[1]
    if what == "hybrid":
        from tests import test_gpu_hybrid as T
        import synthdata as sd
        model = sd.mlp([784, 256, 192, 128, 10], cuts=[1, 3])
        w0, X, Y = sd.parity_inputs(model, 4, 32, seed=1)
        ctxs = T._hybrid_local(model, [2, 1, 1], 32, 0.05, 4)
        try:
            T._check(model, [2, 1, 1], ctxs, w0, X, Y, 0.05)
        finally:
            for s in ctxs:
                s.close()
    elif what == "graph":
        from tests import test_gpu_graph as T
        for name, mk, M, B, lr in T.CASES:
            if name in ("mlp", "lstm_lm"):
                model = mk()
                w0, X, Y = T._inputs(model, M, B)
                T._run(model, B, lr, w0, X, Y, True, sessions=(M // 2,))
    elif what == "p2p":
        from tests import test_gpu_p2p as T
        d = Path(tempfile.mkdtemp())
        codes = T._spawn(2, "mlp", 4, 32, 0.05, d)
        assert all(c == 0 for c in codes), codes
    elif what == "p2p_rank":  # one rank of a 2-stage P2P pipeline (run each under compute-sanitizer)
        from tests import test_gpu_p2p as T
        rank, port, out = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
        T._worker(rank, 2, port, "mlp", 4, 32, 0.05, out, -1, 120)
        assert (Path(out) / f"status{rank}.npy").exists()
    elif what == "layers":
        from tests import test_gpu_partition as T
        import synthdata as sd
        import paper_1809_02839_b200 as st
        model = sd.mlp([784, 512, 256, 10], cuts=[])
        w0, X, Y = sd.parity_inputs(model, 3, 64, seed=3)
        T._run_one_stage(st, model, w0, X, Y, 0.05, profile=True)
    print(what, "done")
