"""C-ABI library checks that need no GPU: libhc.so loads, exports every symbol
include/hc.h declares, and its host-side Preprocessing (hc_build_table, a
separate implementation of Fig. 3) equals the oracle's table."""
import json
import os
import re

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def hc():
    from paper_2310_15711_b200 import build
    build.build()
    from paper_2310_15711_b200 import hc as _hc
    return _hc


def header_functions():
    src = open(os.path.join(ROOT, "include", "hc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hc_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(hc):
    names = header_functions()
    assert set(names) == set(hc.EXPORTS), names
    for name in names:
        assert hasattr(hc.lib(), name), name
    assert "sm_100a" in hc.version()


def test_strerror_covers_codes(hc):
    for code in range(-7, 1):
        assert hc.lib().hc_strerror(code).decode()
    assert hc.lib().hc_strerror(-99).decode() == "unknown error"


@pytest.mark.parametrize("x,q,alpha,code", [
    (b"ab", 3, 8, -2),        # q > m: HC_ETOOSHORT
    (b"", 1, 8, -1),          # m = 0: HC_EINVAL
    (b"abc", 0, 8, -1),       # q < 1
    (b"abcdefghij", 9, 8, -1),  # q > 8 (kernel q-gram window)
    (b"abc", 2, 0, -3),       # alpha < 1: HC_EALPHA
    (b"abc", 2, 16, -3),      # alpha > 15
])
def test_build_table_errors(hc, x, q, alpha, code):
    with pytest.raises(hc.HCError) as ei:
        hc.build_table(x, q, alpha)
    assert ei.value.code == code
    assert hc.lib().hc_last_error() == code


def test_build_table_fig2(hc, golden_dir):
    g = json.load(open(os.path.join(golden_dir, "fig2_example.json")))
    t = hc.build_table(g["x"].encode(), g["q"], g["alpha"])
    assert {str(i): int(v) for i, v in enumerate(t.F) if v} == g["F_w32_DERIVED"]
    assert t.hv == g["hv"] and t.s == g["s"] and t.w == 32


def test_build_table_equals_oracle(hc):
    rng = np.random.default_rng(41)
    for _ in range(800):
        sigma = int(rng.choice([2, 4, 20, 90, 256]))
        q = int(rng.integers(1, 9))
        m = int(rng.integers(q, 300))
        alpha = int(rng.integers(1, 16))
        x = rng.integers(0, sigma, m, dtype=np.uint8)
        if sigma == 256 and rng.random() < 0.5:
            x |= 0x80          # bytes >= 0x80 (signedness, reading R3)
        t = hc.build_table(x, q, alpha)
        o = oracle.preprocess(x, q, alpha, w=32)
        assert np.array_equal(t.F.astype(np.uint64), o.F), (m, q, alpha)
        assert t.hv == o.hv and t.s == o.s
