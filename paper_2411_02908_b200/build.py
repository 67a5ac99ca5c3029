"""Build libphoton.so in-tree: nvcc for sm_100a, one object per source, then a
shared-library link.  Incremental (mtime-based), parallel.

    python -m paper_2411_02908_b200.build [--clean] [-v]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# PHOTON_BUILD_TRACE=1 builds an instrumented copy (libphoton_trace.so, separate
# objects) with per-phase clock64 stamps in the attention kernels (tools/attn_trace.py).
TRACE = os.environ.get("PHOTON_BUILD_TRACE") == "1"
LIB = os.path.join(PKG, "libphoton_trace.so" if TRACE else "libphoton.so")
OBJ = os.path.join(PKG, "_build_trace" if TRACE else "_build")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
          f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}", "--expt-relaxed-constexpr",
          "-diag-suppress", "177"]
# Per-source extra flags.  optim.cu must not contract a*b+c into FMA: its f64
# kernels reproduce the reference's FMA-free x86-64 arithmetic bit for bit.
EXTRA = {"optim.cu": ["-fmad=false"]}


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.hpp")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))


def _needs(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, verbose: bool):
    name = os.path.basename(src)
    obj = os.path.join(OBJ, name + ".o")
    if not _needs(obj, [src] + _headers()):
        return obj, None
    cmd = [NVCC] + ARCH + COMMON + EXTRA.get(name, []) + (["-DPHOTON_ATTN_TRACE"] if TRACE else [])
    if src.endswith(".cpp"):
        cmd += ["-x", "cu"]  # host code that includes device headers
    if name.startswith("gemm_tc") or name.startswith("attn_tc"):
        cmd += ["-Xptxas", "-v"] if verbose else []
    cmd += ["-c", src, "-o", obj]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"nvcc failed for {name}:\n{' '.join(cmd)}\n{out.stdout}{out.stderr}")
    return obj, (out.stdout + out.stderr) if verbose else None


def build(verbose: bool = False, clean: bool = False) -> str:
    if clean and os.path.isdir(OBJ):
        shutil.rmtree(OBJ)
    os.makedirs(OBJ, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                print(log)
    if _needs(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + [
            "-lcudart", "-lcuda", "-ldl", f"-L{CUDA}/lib64", f"-L{CUDA}/lib64/stubs",
            "-Xlinker", f"-rpath={CUDA}/lib64"]
        out = subprocess.run(cmd, capture_output=True, text=True)
        if out.returncode != 0:
            raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{out.stdout}{out.stderr}")
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--clean", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args(argv)
    print(build(verbose=a.verbose, clean=a.clean))


if __name__ == "__main__":
    sys.exit(main())
