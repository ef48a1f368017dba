"""Build libgks.so in-tree: nvcc for sm_100a (CUDA kernels + C ABI) and g++
(host setup: stencils / reconstruction operators, OpenMP).

    python -m paper_2304_09485_b200.build [--verbose]

The shared library lands next to this file so it travels with the repo
snapshot to the GPU box (it is git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
INCLUDE = HERE.parent / "include"
LIB = HERE / "libgks.so"
BUILD = HERE.parent / "build" / "gks"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fopenmp",
              "--expt-relaxed-constexpr", "-I", str(INCLUDE)]
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-fopenmp", "-march=x86-64-v2", "-I", str(INCLUDE)]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"command failed: {' '.join(cmd[:3])} ...")
    if verbose and (res.stdout or res.stderr):
        print(res.stdout + res.stderr)
    return res


def sources():
    cu = sorted(CSRC.glob("*.cu"))
    cpp = sorted(CSRC.glob("*.cpp"))
    return cu, cpp


def build(verbose=False, force=False, ptxas_verbose=False, defines=(), out=None):
    """Compile libgks.so (out: alternative path for experiment variants)."""
    global LIB, BUILD
    if out is not None:
        lib_saved, build_saved = LIB, BUILD
        LIB = Path(out)
        BUILD = LIB.parent / "obj"
        try:
            return build(verbose, True, ptxas_verbose, defines, None)
        finally:
            LIB, BUILD = lib_saved, build_saved
    cu, cpp = sources()
    deps = cu + cpp + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [INCLUDE / "gks.h", Path(__file__)]
    if LIB.exists() and not force:
        newest = max(p.stat().st_mtime for p in deps)
        if LIB.stat().st_mtime >= newest:
            return LIB
    BUILD.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    extra = ["-Xptxas", "-v"] if ptxas_verbose else []
    dflags = [f"-D{d}" for d in defines] + os.environ.get("GKS_NVCC_EXTRA", "").split()
    # gks_setup_dev.cu: no FMA contraction, so the device-built operators
    # equal the host build (g++ -ffp-contract=off) bit for bit
    jobs = [([nvcc, *ARCH, *NVCC_FLAGS, *dflags, *extra, *(["-fmad=false"] if src.stem == "gks_setup_dev" else []),
              "-c", str(src), "-o", str(BUILD / (src.stem + ".o"))], verbose or ptxas_verbose) for src in cu]
    jobs += [(["g++", *CXX_FLAGS, "-ffp-contract=off", "-c", str(src), "-o", str(BUILD / (src.stem + ".o"))], verbose)
             for src in cpp]
    # translation units compile independently: run them concurrently
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
        list(ex.map(lambda j: _run(*j), jobs))
    objs = [BUILD / (src.stem + ".o") for src in cu + cpp]
    tmp = LIB.with_suffix(".so.tmp")
    _run([nvcc, *ARCH, "-shared", "-cudart", "static", "-Xcompiler", "-fopenmp", "-o", str(tmp),
          *map(str, objs), "-lgomp"], verbose)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    lib = build(verbose="--verbose" in sys.argv, force=True, ptxas_verbose="--ptxas" in sys.argv, defines=defs,
                out=outs[0] if outs else None)
    print(lib)
