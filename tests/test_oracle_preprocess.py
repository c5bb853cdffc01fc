"""Pins for the oracle's Fig. 3 Preprocessing.

Pins: the Fig. 1 computation order and H_11 = H_v, the P:104
chain listing, the hand-derived Fig. 2 table (tests/golden), the closed forms
of S:46 / S:116 / S:144 / S:149, and the two defining properties of Eq. 1
and Eq. 2 (every adjacent non-overlapping pair is linked; every q-gram of x
is a recognised factor), checked directly on x rather than through the
chain loop.
"""
import json
import os

import numpy as np
import pytest

import oracle


def test_fig1_order_and_hv():
    # Fig. 1: m = 13, q = 3 -> 3 chains (ends 12, 11, 10) of sizes 4, 4, 3.
    # Fig. 3 processes i = 3, 2, 1 -> chains ending at 10, 11, 12; the chain ending at
    # m-1 = 12 is last so its last hash (the 11th computed) is H_v ("H_11").
    x = bytes(np.random.default_rng(1).integers(97, 100, 13, dtype=np.uint8))
    t = oracle.preprocess(x, 3, 11, trace=True)
    chain_order = [10, 7, 4, 11, 8, 5, 2, 12, 9, 6, 3]
    assert t.trace[:11] == chain_order
    # lines 14-17 re-hash the first q q-grams (ends q-1 .. 2q-2)
    assert t.trace[11:] == [2, 3, 4]
    # P:209 / S:149: (m-q+1) + min(q, m-q+1) hash evaluations
    assert len(t.trace) == (13 - 3 + 1) + min(3, 13 - 3 + 1) == 14
    # H_11 is the hash of the q-gram ending at 3 (= x[1..3])
    assert t.hv == oracle.hash_qgram(x, 3, 3, 11 // 3, (1 << 11) - 1)


def test_p104_chains(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "fig2_example.json")))
    x = g["x"].encode()
    t = oracle.preprocess(x, 4, 4, w=4, trace=True)
    # chain walk (first 13 traced hashes) groups by end index mod q; each group read
    # forwards is one P:104 chain
    ends = t.trace[:13]
    groups = {}
    for e in ends:
        groups.setdefault((e - 3) % 4, []).append(e)
    got = {}
    for off, es in groups.items():
        got[str(off)] = [x[e - 3:e + 1].decode() for e in sorted(es)]
    assert got == g["chains_P104"]


def test_fig2_table(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "fig2_example.json")))
    x = g["x"].encode()
    for w, key in ((4, "F_w4_DERIVED"), (32, "F_w32_DERIVED")):
        t = oracle.preprocess(x, g["q"], g["alpha"], w=w)
        got = {str(i): int(v) for i, v in enumerate(t.F) if v}
        assert got == g[key]
        assert t.hv == g["hv"]
        assert t.s == g["s"]
    # popcount 8 <= m - q + 1 = 13
    t = oracle.preprocess(x, 4, 4, w=4)
    assert sum(bin(int(v)).count("1") for v in t.F) == 8


def _rand_pattern(rng, sigma, m):
    return bytes(rng.integers(0, sigma, m, dtype=np.uint8) + (97 if sigma <= 26 else 0))


def test_table_properties_randomized():
    rng = np.random.default_rng(21)
    for trial in range(600):
        sigma = int(rng.choice([2, 4, 20, 64, 256]))
        q = int(rng.integers(1, 9))
        m = int(rng.integers(q, 130))
        alpha = int(rng.integers(4, 13))
        w = int(rng.choice([4, 8, 16, 32, 64]))
        x = _rand_pattern(rng, sigma, m)
        t = oracle.preprocess(x, q, alpha, w=w)
        s, mask = alpha // q, (1 << alpha) - 1
        h = [oracle.hash_qgram(x, e, q, s, mask) for e in range(q - 1, m)]   # h[i] = q-gram at start i
        # popcount <= m - q + 1
        assert sum(bin(int(v)).count("1") for v in t.F) <= m - q + 1
        # Eq. 2 + Eq. 1: every q-gram of x is recognised (F != 0)
        for i in range(m - q + 1):
            assert t.F[h[i]] != 0
        # Eq. 1: every pair u1 = x[i..i+q-1], u2 = x[i+q..i+2q-1], 0 <= i <= m-2q
        for i in range(0, m - 2 * q + 1):
            assert int(t.F[h[i + q]]) & (1 << (h[i] & (w - 1)))
        # only words of x's q-grams are non-zero
        nz = set(np.nonzero(t.F)[0].tolist())
        assert nz <= set(h)
        # S:46 closed form: H_v = hash of the q-gram starting at m mod q
        assert t.hv == h[m % q]
        # words only hold bits below w
        assert all(int(v) < (1 << w) for v in t.F)


def test_m_equals_q_single_word():
    # P:102 / S:116: m = q -> one chain, one q-gram; the only non-zero word is 1
    for q in range(1, 9):
        x = bytes(range(100, 100 + q))
        t = oracle.preprocess(x, q, 12)
        nz = np.nonzero(t.F)[0]
        hx = oracle.hash_qgram(x, q - 1, q, 12 // q, 4095)
        assert nz.tolist() == [hx] and t.F[hx] == 1 and t.hv == hx


def test_chain_accounting_exhaustive():
    # S:145 / S:397: min(q, m-q+1) chains, sizes sum to m-q+1, chain for m-1 has floor(m/q)
    for m in range(1, 257):
        for q in range(1, min(m, 8) + 1):
            t = oracle.preprocess(bytes(m), q, 8, trace=True)
            nchain = min(q, m - q + 1)
            chain_part = t.trace[:m - q + 1]
            assert len(t.trace) == (m - q + 1) + nchain
            assert sorted(chain_part) == list(range(q - 1, m))
            assert sum(1 for e in chain_part if (e - (m - 1)) % q == 0) == m // q


@pytest.mark.parametrize("m,q,alpha,w", [(3, 4, 8, 32), (5, 0, 8, 32), (5, 2, 0, 32),
                                         (5, 2, 31, 32), (5, 2, 8, 12)])
def test_invalid_params(m, q, alpha, w):
    with pytest.raises(ValueError):
        oracle.preprocess(bytes(m), q, alpha, w=w)
