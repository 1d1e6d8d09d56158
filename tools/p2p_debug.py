"""Debug a P2P pipeline of separate processes on one GPU (tests/test_gpu_p2p.py's
worker): short ST_COMM_TIMEOUT_S, each stage's error (with its flag block) printed as
soon as it appears."""
import os, sys, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from pathlib import Path
import torch.multiprocessing as mp
from tests import test_gpu_p2p as T

if __name__ == "__main__":
    os.environ["CUDA_LAUNCH_BLOCKING"] = os.environ.get("CUDA_LAUNCH_BLOCKING", "1")
    os.environ["P2P_DEBUG"] = "1"
    os.environ["ST_P2P_TRACE"] = "1"
    name, world, M, B = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    hang = int(sys.argv[5]) if len(sys.argv) > 5 else -1
    d = Path(tempfile.mkdtemp())
    port = T._free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=T._worker, args=(r, world, port, name, M, B, 0.1, str(d), hang, 5)) for r in range(world)]
    for p in procs:
        p.start()
    seen = set()
    t0 = time.time()
    while time.time() - t0 < 60 and any(p.is_alive() for p in procs):
        for f in sorted(d.iterdir()):
            if f.name not in seen and f.name.startswith(("err", "status")):
                seen.add(f.name)
                print(f"{time.time() - t0:.0f}s", f.name, f.read_text() if f.suffix == ".txt" else "", flush=True)
        time.sleep(1)
    for f in sorted(d.iterdir()):
        if f.name not in seen and f.name.startswith(("err", "status")):
            print(f.name, f.read_text() if f.suffix == ".txt" else "", flush=True)
    print("alive:", [p.is_alive() for p in procs], "codes:", [p.exitcode for p in procs], flush=True)
    for p in procs:
        if p.is_alive():
            p.kill()
