"""Build libmpr.so (sm_100a) in-tree with nvcc. Called by __graft_entry__.build()."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libmpr.so")
SOURCES = ["api.cu", "params.cu", "sweep.cu", "calib.cu", "comm.cu"]
HEADERS = ["device_math.cuh", "internal.cuh", "comm.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xcompiler", "-ffp-contract=off",  # host-side decision arithmetic (ARITH §K) unfused
    "-prec-div=true", "-ftz=false", "-prec-sqrt=true",
    "-Xptxas", "-v",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "mpr.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    return res.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every source to an object in parallel (one nvcc per translation unit), then
    link libmpr.so; the library is replaced atomically."""
    from concurrent.futures import ThreadPoolExecutor
    import tempfile
    if not force and not _stale():
        return LIB
    with tempfile.TemporaryDirectory(prefix="mpr_build_") as tmpdir:
        objs = [os.path.join(tmpdir, os.path.splitext(s)[0] + ".o") for s in SOURCES]
        cmds = [[NVCC, *FLAGS, "-I", os.path.join(ROOT, "include"), "-c", "-o", o, os.path.join(CSRC, s)]
                for s, o in zip(SOURCES, objs)]
        with ThreadPoolExecutor(max_workers=len(cmds)) as ex:
            logs = list(ex.map(_run, cmds))
        tmp = LIB + f".tmp{os.getpid()}"
        logs.append(_run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, "-ldl", "-lpthread"]))
    if verbose:
        print("\n".join(logs))
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(LIB)
