"""Build libhc.so (the C-ABI library of include/hc.h) in-tree for sm_100a.

    python -m paper_2310_15711_b200.build          # builds if sources changed
    python -m paper_2310_15711_b200.build --force

nvcc cross-compiles for sm_100a without a GPU.  The library is written next
to this file so it travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libhc.so")
# translation units: (source, extra flags, object name); hc_inst.cu once per q-gram
# length so that the kernel instantiations compile in parallel
UNITS = [("hc_api.cpp", [], "hc_api.o"), ("hc_launch.cu", [], "hc_launch.o")] + [
    ("hc_inst.cu", [f"-DHC_Q={q}"], f"hc_inst_q{q}.o") for q in range(1, 9)]
HEADERS = ["hc_internal.h", "hc_device.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
OBJDIR = os.path.join(HERE, "build_obj")


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found (CUDA 12.9 toolkit required)")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f, _, _ in UNITS] + [os.path.join(CSRC, h) for h in HEADERS]
    deps += [os.path.join(INCLUDE, "hc.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(OBJDIR, exist_ok=True)
    common = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
              "-Xptxas", "-v" if verbose else "-O3", "-I", INCLUDE, "-I", CSRC]

    def compile_unit(u):
        src, flags, obj = u
        out = os.path.join(OBJDIR, obj)
        r = subprocess.run(common + flags + ["-c", os.path.join(CSRC, src), "-o", out],
                           capture_output=True, text=True)
        if r.returncode != 0 or verbose:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise subprocess.CalledProcessError(r.returncode, src)
        return out

    with ThreadPoolExecutor(min(len(UNITS), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_unit, UNITS))
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([nvcc(), *ARCH, "-shared", *objs, "-o", tmp])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
