"""Fault injection and compute-sanitizer runs over every kernel of libhc
(test hooks and race detection).

* Fault injection: the instrumented build (libhc_instr.so, HC_INSTRUMENT=1) has a
  test hook (opts.debug = 9) that shifts the first ordered position by one.  The
  parity driver tools/sanitize_case.py (every path against brute force) must FAIL
  with the hook on and pass with it off: the parity check catches a corrupted
  kernel.
* Bounds-checked build (libhc_chk.so, HC_BOUNDS=1): traps on any text access outside the text
  or the CTA's shared memory; the parity driver must pass under it.
* compute-sanitizer: opt-in (HC_SANITIZER=memcheck|racecheck|synccheck), one tool per
  run, because several sanitizer tools in one GPU session are not safe on this pool
  (B200_PROFILING.md); logs of the runs are kept in profiles/.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASE = os.path.join(ROOT, "tools", "sanitize_case.py")
INSTR = os.path.join(ROOT, "paper_2310_15711_b200", "libhc_instr.so")
CHK = os.path.join(ROOT, "paper_2310_15711_b200", "libhc_chk.so")


def _run(args, env_extra=None, prefix=(), timeout=900):
    env = dict(os.environ)
    env.update(env_extra or {})
    return subprocess.run([*prefix, sys.executable, CASE, *args], capture_output=True, text=True,
                          env=env, timeout=timeout, cwd=ROOT)


@pytest.mark.skipif(not os.path.exists(INSTR), reason="libhc_instr.so not built")
def test_fault_injection_is_caught():
    red = _run(["--inject", "--small"], {"HC_LIB": INSTR})
    assert red.returncode == 1, red.stdout + red.stderr
    assert "MISMATCH" in red.stdout
    green = _run(["--small"], {"HC_LIB": INSTR})
    assert green.returncode == 0, green.stdout + green.stderr


@pytest.mark.skipif(not os.path.exists(CHK), reason="libhc_chk.so not built")
def test_bounds_checked_build():
    """Our own memcheck (compute-sanitizer is closed on this pool): the bounds-checked build
    (HC_BOUNDS=1) checks every text access (aligned global words must hold a byte of [y, y + n), shared
    accesses must lie inside the CTA's shared memory, copies must read inside the text) and
    traps outside.  Every path, aligned and unaligned texts, odd lengths, edge chunks: no
    trap, every result equal to brute force."""
    r = _run(["--small", "--unaligned"], {"HC_LIB": CHK})
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    assert "0 mismatches" in r.stdout


@pytest.mark.skipif(os.environ.get("HC_SANITIZER") not in ("memcheck", "racecheck", "synccheck"),
                    reason="opt-in: HC_SANITIZER=memcheck|racecheck|synccheck")
def test_compute_sanitizer():
    tool = os.environ["HC_SANITIZER"]
    r = _run(["--small"], {"PYTORCH_NO_CUDA_MEMORY_CACHING": "1"},
             prefix=("compute-sanitizer", "--tool", tool, "--target-processes", "all"),
             timeout=3000)
    out = r.stdout + r.stderr
    log = os.environ.get("HC_SANITIZER_LOG")
    if log:
        with open(log, "w") as f:
            f.write(out)
    assert r.returncode == 0, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
