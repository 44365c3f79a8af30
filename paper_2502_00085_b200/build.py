"""Build libtriedecode.so in-tree for sm_100a (nvcc only; no torch extension machinery).

    python -m paper_2502_00085_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# TRIE_BUILD_OUT: write an alternative build elsewhere (A/B experiments, see _lib.TRIE_LIB)
LIB = os.environ.get("TRIE_BUILD_OUT") or os.path.join(HERE, "libtriedecode.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "--expt-relaxed-constexpr", "-Xptxas", "-v",
    "-I" + os.path.join(ROOT, "include"),
]
# experiment builds: TRIE_BUILD_DEFINES="TRIE_UMMA_TRACE=1" (use --force; see scripts/umma_trace.py)
FLAGS += ["-D" + d for d in os.environ.get("TRIE_BUILD_DEFINES", "").split() if d]
OBJDIR = os.path.join(HERE, "build_obj" + ("_alt" if os.environ.get("TRIE_BUILD_OUT") else ""))


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    deps += glob.glob(os.path.join(ROOT, "include", "*.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(OBJDIR, exist_ok=True)
    procs, objs = [], []
    for src in sources():  # one nvcc per translation unit, in parallel
        obj = os.path.join(OBJDIR, os.path.basename(src) + ".o")
        objs.append(obj)
        procs.append((src, subprocess.Popen([NVCC] + FLAGS + ["-c", src, "-o", obj],
                                            stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    log, failed = [], False
    for src, p in procs:
        out, err = p.communicate()
        log.append(f"==== {os.path.basename(src)}\n{out}{err}")
        if p.returncode != 0:
            failed = True
            sys.stderr.write(out + err)
    with open(os.path.join(HERE, "ptxas.log"), "w") as f:
        f.write("\n".join(log))
    if verbose:
        sys.stderr.write("\n".join(log))
    if failed:
        raise RuntimeError("nvcc failed building libtriedecode.so")
    tmp = LIB + ".tmp"
    res = subprocess.run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a"] + objs +
                         ["-o", tmp, "-lcuda"], capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed for libtriedecode.so")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
