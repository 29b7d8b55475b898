"""Builds libfastlk_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2003_13493_b200.build [--force] [-v]

Every translation unit under csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked into one
shared library that exports only the C ABI (``FLK_API`` symbols); the CUDA
runtime is linked statically so the library has no dependency on a particular
libcudart on the box. Objects are rebuilt when a source or header is newer.
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
OBJ = os.path.join(PKG, "_obj")
LIB = os.path.join(PKG, "libfastlk_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# fp64 LK tracker: no a*b+c contraction, so products and sums round like the
# reference's x86-64 build (SSE2, no FMA) -- see csrc/session.cu
NO_FMA = {"session.cu"}
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden,-Wall",
          f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _deps() -> float:
    files = glob.glob(os.path.join(CSRC, "*")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    return max(os.path.getmtime(f) for f in files)


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    cmd = [nvcc()] + ARCH + COMMON + os.environ.get("FLKB_NVCC_FLAGS", "").split() + [
        "-c", src, "-o", obj]
    if os.path.basename(src) in NO_FMA:
        cmd += ["-fmad=false"]
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"] if verbose else []
        cmd += ["--expt-relaxed-constexpr"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr:
        sys.stderr.write(res.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    if (not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _deps()
            and os.path.getmtime(LIB) >= os.path.getmtime(__file__)):
        build_cli()
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    tmp = LIB + ".tmp"
    cmd = [nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs + [
        "-Xlinker", "-Bsymbolic", "-Xlinker", "--exclude-libs,ALL", "-lpthread", "-ldl", "-lrt"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB)
    build_cli()
    return LIB


CLI_SRC = os.path.join(PKG, "cli", "fastlk_cli.cpp")
CLI_BIN = os.path.join(PKG, "fastlk_b200")


def build_cli() -> str:
    """The sequence harness (cli/fastlk_cli.cpp) linked against the library."""
    if (os.path.exists(CLI_BIN) and os.path.getmtime(CLI_BIN) >= os.path.getmtime(CLI_SRC)
            and os.path.getmtime(CLI_BIN) >= os.path.getmtime(LIB)):
        return CLI_BIN
    cmd = ["g++", "-O2", "-std=c++17", "-Wall", "-Wextra", f"-I{os.path.join(ROOT, 'include')}",
           CLI_SRC, f"-L{PKG}", "-lfastlk_b200", "-Wl,-rpath,$ORIGIN", "-o", CLI_BIN]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"CLI build failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    return CLI_BIN


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))


if __name__ == "__main__":
    main()
