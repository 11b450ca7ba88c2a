"""Build the native library in-tree: paper_2601_02540_b200/_native/libhsgn_b200.so.

nvcc cross-compiles for sm_100a only (no other targets, no PTX fallback).
``--fmad=false`` is part of the parity contract:
the reference build has no FMA contraction, so neither may the kernels; the
only fused multiply-adds are the explicit __fma_rn of the correctly rounded
division in sgn_device.cuh.
"""
from __future__ import annotations

import concurrent.futures
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.environ.get("HSGN_BUILD_DIR") or os.path.join(HERE, "_native")  # variants: experiments only
LIB = os.path.join(OUT_DIR, "libhsgn_b200.so")
SOURCES = ["sgn_stage.cu", "sgn_aux.cu", "hsgn_host.cu", "hsgn_scenarios.cpp"]
# sgn_stage.cu is also compiled once per stencil kind and kernel family (its
# instantiation units, see the end of the file), so the kernels build in parallel
UNITS = [(src, os.path.splitext(src)[0], []) for src in SOURCES] + [
    ("sgn_stage.cu", f"sgn_stage_{fam}{k}", [f"-DHSGN_INST_KIND={k}", f"-DHSGN_INST_S12={int(fam == 's12_k')}"])
    for fam in ("s12_k", "mode_k") for k in (0, 1, 2)]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(HERE, "..", "include", "hsgn_b200.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    extra = os.environ.get("HSGN_NVCC_EXTRA", "").split()  # experiments only (e.g. -DHSGN_MIN_BLOCKS=4)

    def compile_unit(unit):
        src, name, defs = unit
        obj = os.path.join(OUT_DIR, name + ".o")
        # host C++ (the scenario registry): no FP contraction, like the reference build
        host = ["-Xcompiler", "-ffp-contract=off"] if src.endswith(".cpp") else []
        cmd = [nvcc(), *ARCH, *FLAGS, *host, *defs, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return obj, r

    jobs = int(os.environ.get("HSGN_BUILD_JOBS", "0")) or max(1, min(len(UNITS), os.cpu_count() or 1))
    with concurrent.futures.ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(compile_unit, UNITS))
    objs, log = [], []
    for (src, _, _), (obj, r) in zip(UNITS, results):
        log.append(r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        objs.append(obj)
    tmp = LIB + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, LIB)
    with open(os.path.join(OUT_DIR, "ptxas.log"), "w") as fh:
        fh.write("\n".join(log))
    if verbose:
        print("\n".join(log))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
