"""Build libspectrain.so in-tree with nvcc for sm_100a (no JIT cache: the .so
travels to the GPU box with the repo snapshot)."""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libspectrain.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _site_packages() -> str:
    return sysconfig.get_paths()["purelib"]


def nccl_paths():
    base = os.path.join(_site_packages(), "nvidia", "nccl")
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _needs(obj: str, src: str, deps) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src, *deps])


def build(verbose: bool = False, force: bool = False, defines=(), lib: str = LIB, build_dir: str = BUILD) -> str:
    """defines / lib / build_dir: development variants (e.g. ring depths) built beside the product .so."""
    nccl_inc, nccl_lib = nccl_paths()
    BUILD, LIB = build_dir, lib
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh"))]
    headers.append(os.path.join(INCLUDE, "spectrain.h"))
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden", f"-I{INCLUDE}",
              f"-I{CSRC}", f"-I{nccl_inc}", *ARCH, "-Xptxas", "-v" if verbose else "-O3", *[f"-D{d}" for d in defines]]
    objs, jobs = [], []
    for src in sources():
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _needs(obj, src, headers):
            cmd = ["nvcc", *common, "-c", src, "-o", obj]
            if src.endswith(".cpp"):
                cmd = ["nvcc", "-x", "cu", *common, "-c", src, "-o", obj]
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(run, jobs))
    if jobs or not os.path.exists(LIB):
        link = ["nvcc", "-shared", *ARCH, "-o", LIB, *objs, f"-L{nccl_lib}", "-l:libnccl.so.2",
                f"-Xlinker", f"-rpath,{nccl_lib}", "-lpthread"]
        run(link)
    return LIB


DEV_DIR = os.path.join(HERE, "_var", "dev")
DEV_LIB = os.path.join(DEV_DIR, "libspectrain.so")


def build_dev(verbose: bool = False, force: bool = False) -> str:
    """The development variant: the same sources with -DST_DEV_KNOBS (csrc/knobs.hpp), so
    the A/B switches and opt-in kernel variants are read from the environment. Used by
    tests/test_gpu_variants.py (ST_LIB_PATH); the product library reads no knobs."""
    return build(verbose=verbose, force=force, defines=("ST_DEV_KNOBS",), lib=DEV_LIB,
                 build_dir=os.path.join(DEV_DIR, "_build"))


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
