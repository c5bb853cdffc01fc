"""Pins for the oracle's searching phase (O1 brute force, O2 Fig. 5 HC / SHC).

O1 is pinned by SPEC's worked examples, closed forms and an independent
Python loop (bytes.find).  O2 is pinned to O1 on exhaustive tiny inputs (all
windows of de Bruijn texts), randomized trials, and closed forms for
its instrumentation.
"""
import itertools

import numpy as np
import pytest

import oracle


def py_find_all(x: bytes, y: bytes):
    """Independent second loop: repeated bytes.find."""
    out, k = [], y.find(x)
    while k != -1:
        out.append(k)
        k = y.find(x, k + 1)
    return out


def de_bruijn(k: int, n: int, alphabet: bytes) -> bytes:
    """Standard de Bruijn sequence B(k, n) (Lyndon-word construction), made
    linear by appending its first n-1 symbols: every length-n string over the
    alphabet occurs exactly once."""
    a = [0] * k * n
    seq = []

    def db(t, p):
        if t > n:
            if n % p == 0:
                seq.extend(a[1:p + 1])
        else:
            a[t] = a[t - p]
            db(t + 1, p)
            for j in range(a[t - p] + 1, k):
                a[t] = j
                db(t + 1, t)

    db(1, 1)
    s = bytes(alphabet[i] for i in seq)
    return s + s[:n - 1]


# ---------------------------------------------------------------- O1 pins
def test_brute_spec_examples():
    assert oracle.brute(b"aa", b"aaaa").tolist() == [0, 1, 2]
    assert oracle.brute(b"abc", b"zzzz").tolist() == []
    assert oracle.brute(b"abc", b"ab").tolist() == []                # n < m
    assert oracle.brute(b"x", b"").tolist() == []
    with pytest.raises(ValueError):
        oracle.brute(b"", b"abc")


def test_brute_closed_form_runs():
    # a^m in a^n: n - m + 1 occurrences
    y = b"a" * 100_000
    assert len(oracle.brute(b"a" * 64, y)) == 100_000 - 63
    assert len(oracle.brute_threaded(b"a" * 64, b"a" * 1_000_000, threads=4)) == 1_000_000 - 63


def test_brute_vs_python_find():
    rng = np.random.default_rng(31)
    for _ in range(300):
        sigma = int(rng.choice([2, 3, 4, 26, 256]))
        n = int(rng.integers(0, 3000))
        m = int(rng.integers(1, 12))
        y = bytes(rng.integers(0, sigma, n, dtype=np.uint8))
        if n >= m and rng.random() < 0.7:
            o = int(rng.integers(0, n - m + 1))
            x = y[o:o + m]
        else:
            x = bytes(rng.integers(0, sigma, m, dtype=np.uint8))
        assert oracle.brute(x, y).tolist() == py_find_all(x, y)


def test_brute_threaded_equals_single():
    rng = np.random.default_rng(32)
    y = rng.integers(0, 2, 50_000, dtype=np.uint8)
    for m in (1, 3, 9):
        x = y[1000:1000 + m]
        assert np.array_equal(oracle.brute_threaded(x, y, threads=7), oracle.brute(x, y))


# ---------------------------------------------------------------- O2 vs O1
def test_hc_spec_example_aa():
    # ("aa", "aaaa") -> {0,1,2}.  Reading R1: the literal Fig. 5 index j-q would
    # give {-1, 0, 1}; the fixed index gives the brute-force answer.
    for q in (1, 2):
        assert oracle.hc_search(b"aa", b"aaaa", q, 8).tolist() == [0, 1, 2]
        assert oracle.shc_search(b"aa", b"aaaa", q, 8).tolist() == [0, 1, 2]


def _check_all(x, y, q, alpha, w):
    want = py_find_all(x, y)
    got = oracle.hc_search(x, y, q, alpha, w).tolist()
    assert got == want, (x, q, alpha, w)
    assert oracle.shc_search(x, y, q, alpha, w).tolist() == want, (x, q, alpha, w)


def test_hc_exhaustive_binary_de_bruijn():
    # every x in {a,b}^1..6 against B(2, 12) (contains every binary 12-gram), all
    # q <= m, alpha in 1..6 and 11, w in {4, 32}
    y = de_bruijn(2, 12, b"ab")
    for m in range(1, 7):
        for xs in itertools.product(b"ab", repeat=m):
            x = bytes(xs)
            for q in range(1, m + 1):
                for alpha in (1, 2, 3, 4, 6, 11):
                    for w in (4, 32):
                        _check_all(x, y, q, alpha, w)


def test_hc_exhaustive_ternary_de_bruijn():
    y = de_bruijn(3, 7, b"abc")
    for m in range(1, 5):
        for xs in itertools.product(b"abc", repeat=m):
            x = bytes(xs)
            for q in range(1, m + 1):
                for alpha in (2, 5, 8):
                    _check_all(x, y, q, alpha, 32)


def test_hc_exhaustive_short_texts():
    # all y in {a,b}^0..10 and x in {a,b}^1..4: text-boundary cases (n < m, n = m, ...)
    ys = [bytes(t) for L in range(0, 11) for t in itertools.product(b"ab", repeat=L)]
    xs = [bytes(t) for L in range(1, 5) for t in itertools.product(b"ab", repeat=L)]
    for x in xs:
        for q in range(1, len(x) + 1):
            tbl = oracle.preprocess(x, q, 3)
            for y in ys:
                assert oracle.hc_search(x, y, q, 3, table=tbl).tolist() == py_find_all(x, y)


def test_hc_randomized_spec_grid():
    # S:395 (scaled: 1500 trials, n <= 2*10^4): sigma in {2,4,20,64,256}, q in 1..8,
    # m in [q, 128], alpha in 8..12
    rng = np.random.default_rng(33)
    for _ in range(1500):
        sigma = int(rng.choice([2, 4, 20, 64, 256]))
        q = int(rng.integers(1, 9))
        m = int(rng.integers(q, 129))
        alpha = int(rng.integers(8, 13))
        n = int(rng.integers(0, 20_000))
        y = rng.integers(0, sigma, n, dtype=np.uint8)
        if n >= m and rng.random() < 0.8:
            o = int(rng.integers(0, n - m + 1))
            x = y[o:o + m].copy()
            if rng.random() < 0.3:   # plant extra copies, incl. at the very end
                for p in (0, n - m, int(rng.integers(0, n - m + 1))):
                    y[p:p + m] = x
        else:
            x = rng.integers(0, sigma, m, dtype=np.uint8)
        want = oracle.brute(x, y)
        assert np.array_equal(oracle.hc_search(x, y, q, alpha), want)
        assert np.array_equal(oracle.shc_search(x, y, q, alpha), want)


def test_hc_periodic_and_planted():
    # a^m in a^n and planted copies at every offset near both text ends
    assert len(oracle.hc_search(b"a" * 64, b"a" * 1_000_000, 6, 12)) == 1_000_000 - 63
    rng = np.random.default_rng(34)
    x = bytes(rng.integers(0, 4, 40, dtype=np.uint8))
    for p in list(range(0, 45)) + list(range(955, 961)):
        y = bytearray(rng.integers(4, 8, 1000, dtype=np.uint8))
        y[p:p + 40] = x
        y = bytes(y[:1000])
        assert oracle.hc_search(x, y, 4, 10).tolist() == py_find_all(x, y)


# ---------------------------------------------------------------- O2 properties
def test_filter_soundness_invariant():
    """For every true occurrence s: F[h(end s+m-1)] != 0, every link test along the
    chain ending at s+m-1 passes, and the last hash equals H_v."""
    rng = np.random.default_rng(35)
    for _ in range(300):
        sigma = int(rng.choice([2, 4, 20]))
        q = int(rng.integers(1, 9))
        m = int(rng.integers(q, 80))
        alpha = int(rng.integers(4, 13))
        w = int(rng.choice([4, 32]))
        y = rng.integers(0, sigma, 3000, dtype=np.uint8)
        x = y[100:100 + m].copy()
        t = oracle.preprocess(x, q, alpha, w)
        s, mask = alpha // q, (1 << alpha) - 1
        for st in oracle.brute(x, y):
            e = int(st) + m - 1
            v = oracle.hash_qgram(y, e, q, s, mask)
            z = int(t.F[v])
            assert z != 0
            j = e
            while j >= e - m + 2 * q:          # the Fig. 5 walk bound i = e - m + 2q
                j -= q
                v = oracle.hash_qgram(y, j, q, s, mask)
                assert z & (1 << (v & (w - 1)))
                z = int(t.F[v])
            assert v == t.hv


def test_segmented_runs_are_exact():
    # reading R11 / SURVEY.md 8(a).2: HC started at any window end a with bound b finds
    # exactly the occurrences ending in [a, b); partitions concatenate to the answer.
    rng = np.random.default_rng(36)
    for _ in range(150):
        sigma = int(rng.choice([2, 4, 20]))
        q = int(rng.integers(1, 7))
        m = int(rng.integers(q, 50))
        alpha = int(rng.integers(6, 13))
        y = rng.integers(0, sigma, 5000, dtype=np.uint8)
        x = y[77:77 + m].copy()
        want = oracle.brute(x, y)
        S = m - q + 1
        for seg in (1, 7, S, 2 * S + 3, 33 * S):
            assert np.array_equal(oracle.hc_search_segmented(x, y, q, alpha, seg), want)
        assert np.array_equal(oracle.hc_threaded(x, y, q, alpha, threads=5), want)


def test_metrics_all_fast_path():
    # "b"^m vs "a"^n: every window takes the F[v]=0 path;
    # windows = qgram_hashes = ceil((n-m+1)/(m-q+1))
    for m, q, n in [(8, 4, 1000), (16, 6, 12345), (5, 5, 77), (32, 3, 100_000)]:
        pos, met = oracle.hc_search(b"b" * m, b"a" * n, q, 12, metrics=True)
        S = m - q + 1
        want = -(-(n - m + 1) // S)
        assert len(pos) == 0 and met.windows == want and met.qgram_hashes == want
        assert met.min_shift == met.max_shift == S


def test_metrics_full_window_work():
    # S:146 / S:398: text = pattern: the single window is fully scanned with floor(m/q)
    # hashes, then verified once
    rng = np.random.default_rng(37)
    for m in range(1, 65):
        for q in range(1, min(m, 8) + 1):
            x = bytes(rng.integers(0, 256, m, dtype=np.uint8))
            pos, met = oracle.hc_search(x, x, q, 12, metrics=True)
            assert pos.tolist() == [0]
            assert met.windows == 1 and met.qgram_hashes == m // q
            assert met.completed_walks == 1 and met.verifications == 1


def test_metrics_invariants_and_hv_gate():
    # S:147 shifts in [1, m-q+1]; S:148 hv_rejections + verifications = completed walks;
    # S:401 the H_v gate rejects some completed walks (alpha = 4, w = 4 force collisions;
    # at alpha = 8, w = 32 random m = 32 patterns complete no walk at all in 10^6 bytes)
    rng = np.random.default_rng(38)
    acgt = np.frombuffer(b"ACGT", dtype=np.uint8)
    y = acgt[rng.integers(0, 4, 1_000_000)]
    total_rej = total_ver = total_done = 0
    for _ in range(20):
        x = acgt[rng.integers(0, 4, 32)]
        pos, met = oracle.hc_search(x, y, 4, 4, w=4, metrics=True)
        assert met.hv_rejections + met.verifications == met.completed_walks
        assert 1 <= met.min_shift <= met.max_shift <= 32 - 4 + 1
        assert met.verifications >= len(pos)
        total_rej += met.hv_rejections
        total_ver += met.verifications
        total_done += met.completed_walks
    assert total_rej > 0 and total_ver < total_done


def test_sublinearity_proxy():
    # sigma=4, n=10^6, q=6, alpha=12: qgram_hashes < n for m in {32..256} and
    # hashes per byte fall as m doubles
    rng = np.random.default_rng(39)
    y = rng.integers(0, 4, 1_000_000, dtype=np.uint8)
    per_byte = []
    for m in (32, 64, 128, 256):
        tot = 0
        for k in range(10):
            o = int(rng.integers(0, len(y) - m))
            _, met = oracle.hc_search(y[o:o + m], y, 6, 12, metrics=True)
            assert met.qgram_hashes < len(y)
            tot += met.qgram_hashes
        per_byte.append(tot / 10 / len(y))
    for a, b in zip(per_byte, per_byte[1:]):
        assert b < a * 1.1
