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
# instrumented build (HC_INSTRUMENT=1): opts.debug modes and %globaltimer traces compiled
# in, for tools/ only; the product library rejects them (HC_EINVAL)
LIB_INSTR = os.path.join(HERE, "libhc_instr.so")
# bounds-checked build (HC_BOUNDS=1: every text access checked, traps outside; only the few
# (q, s) instantiations tools/sanitize_case.py uses): tests/test_gpu_tools.py
LIB_CHK = os.path.join(HERE, "libhc_chk.so")
OBJ = os.path.join(ROOT, "build_obj")
SOURCES = ["hc_api.cpp", "hc_launch.cu", "hc_stream.cu", "hc_gather.cu", "hc_mstream.cu",
           "hc_finish.cu", "hc_shc.cu", "hc_staged.cu", "hc_scan.cu"]
HEADERS = ["hc_internal.h", "hc_device.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found (CUDA 12.9 toolkit required)")


def _stale(lib: str) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(INCLUDE, "hc.h"),
                                                                 __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, obj: str, defs: list, verbose: bool) -> None:
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
           "-Xptxas", "-v" if verbose else "-O3", *defs, "-I", INCLUDE, "-I", CSRC,
           "-c", os.path.join(CSRC, src), "-o", obj]
    subprocess.check_call(cmd)


def build_bounds_checked(force: bool = False) -> str:
    return build(force=force, variant="chk", defines=("HC_BOUNDS=1", "HC_FEW_BUILDS=1"))


def build(force: bool = False, verbose: bool = False, instrument: bool = False,
          variant: str | None = None, defines: tuple = ()) -> str:
    """Compiles every translation unit (in parallel) and links the shared library.
    variant/defines: an experiment build libhc_<variant>.so with extra -D flags (A/B runs
    in tools/, loaded through HC_LIB)."""
    lib = LIB_INSTR if instrument else LIB
    if variant:
        lib = os.path.join(HERE, f"libhc_{variant}.so")
    if not force and not _stale(lib):
        return lib
    from concurrent.futures import ThreadPoolExecutor
    tag = variant or ("instr" if instrument else "prod")
    os.makedirs(os.path.join(OBJ, tag), exist_ok=True)
    defs = [f"-DHC_INSTRUMENT={1 if instrument else 0}", *[f"-D{d}" for d in defines]]
    objs = [os.path.join(OBJ, tag, os.path.splitext(s)[0] + ".o") for s in SOURCES]
    with ThreadPoolExecutor(max_workers=max(1, min(len(SOURCES), os.cpu_count() or 1))) as ex:
        list(ex.map(lambda so: _compile(so[0], so[1], defs, verbose), zip(SOURCES, objs)))
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([nvcc(), *ARCH, "-shared", *objs, "-o", tmp])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), None)
    defs = tuple(a.split("=", 1)[1] for a in sys.argv if a.startswith("--define="))
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                instrument="--instrument" in sys.argv, variant=var, defines=defs))
