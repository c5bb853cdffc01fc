"""Pins for the oracle's primitives: Eq. 3 hash, Eq. 4 shift, Eq. 5 link hash.

Each expected value comes from the paper / SPEC worked examples or a hand
evaluation written out in the test, never from the oracle itself.
"""
import json
import os

import numpy as np
import pytest

import oracle


def test_shift_spec_examples():
    # S:75-77 (Eq. 4)
    assert oracle.shift(12, 6) == 2
    assert oracle.shift(11, 3) == 3
    assert oracle.shift(4, 4) == 1
    # reading R6: q > alpha gives s = 0
    assert oracle.shift(3, 8) == 0


def test_hash_spec_examples():
    # q = 1: a single character, no shift before the only add
    assert oracle.hash_qgram(b"a", 0, 1, 7, 255) == 97
    # ((98*16) + 97) mod 256 = 1665 mod 256 = 129 -- the LAST character of the
    # q-gram ('b') is the one shifted (Fig. 3 Hash starts at x[p]).
    assert oracle.hash_qgram(b"ab", 1, 2, 4, 255) == 129
    # the opposite nesting would give ((97*16)+98) mod 256 = 1650 mod 256 = 114
    assert oracle.hash_qgram(b"ab", 1, 2, 4, 255) != 114


def test_hash_fig2_hand_values(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "fig2_example.json")))
    x = g["x"].encode()
    # hand evaluation, P:159-163 with s = 1: ((t*2 + g)*2 + c)*2 + a
    assert ((116 * 2 + 103) * 2 + 99) * 2 + 97 == 1635
    assert oracle.hash_qgram(x, 3, 4, 1, 15) == 1635 % 16 == 3
    assert ((103 * 2 + 116) * 2 + 103) * 2 + 99 == 1593
    assert oracle.hash_qgram(x, 4, 4, 1, 15) == 1593 % 16 == 9
    for end, v in g["qgram_hash_by_end_DERIVED"].items():
        assert oracle.hash_qgram(x, int(end), 4, 1, 15) == v, end


def _eq3_recursive(u: bytes, s: int, alpha: int) -> int:
    """Eq. 3 as printed: h(x) = 0 if |x| = 0, else
    (h(x[1..]) * 2^s + x[0]) mod 2^alpha."""
    if len(u) == 0:
        return 0
    return (_eq3_recursive(u[1:], s, alpha) * (1 << s) + u[0]) % (1 << alpha)


def test_hash_eq3_recursion_equals_fig3_loop():
    # reading R4: Eq. 3's recursion and Fig. 3's loop are the same function.
    rng = np.random.default_rng(11)
    for _ in range(300):
        q = int(rng.integers(1, 9))
        alpha = int(rng.integers(1, 16))
        s = alpha // q
        u = bytes(rng.integers(0, 256, q, dtype=np.uint8))
        assert oracle.hash_qgram(u, q - 1, q, s, (1 << alpha) - 1) == _eq3_recursive(u, s, alpha)


def test_hash_closed_form_sum():
    # closed form: h = sum_k c_k 2^(s*k) mod 2^alpha, c_0 = first byte of the q-gram
    rng = np.random.default_rng(12)
    for _ in range(300):
        q = int(rng.integers(1, 9))
        alpha = int(rng.integers(1, 31))
        s = alpha // q
        u = bytes(rng.integers(0, 256, q, dtype=np.uint8))
        want = sum(c << (s * k) for k, c in enumerate(u)) % (1 << alpha)
        assert oracle.hash_qgram(u, q - 1, q, s, (1 << alpha) - 1) == want


def test_hash_backward_rolling_identity():
    # algebraic identity: h(j-1) = ((h(j) - (y[j] << s(q-1))) << s) + y[j-q]
    rng = np.random.default_rng(13)
    for q, alpha in [(2, 11), (3, 11), (4, 12), (6, 12), (8, 12), (5, 15)]:
        s = alpha // q
        mask = (1 << alpha) - 1
        y = rng.integers(0, 256, 400, dtype=np.uint8)
        for j in range(q, 400):
            hj = oracle.hash_qgram(y, j, q, s, mask)
            hm = oracle.hash_qgram(y, j - 1, q, s, mask)
            assert ((((hj - (int(y[j]) << (s * (q - 1)))) << s) + int(y[j - q])) & mask) == hm


def test_hash_range_and_unsigned_bytes():
    # S:140 range; reading R3: bytes >= 0x80 are unsigned
    assert oracle.hash_qgram(bytes([0xFF]), 0, 1, 0, (1 << 12) - 1) == 255
    assert oracle.hash_qgram(bytes([0x80, 0xFF]), 1, 2, 6, (1 << 12) - 1) == (0xFF * 64 + 0x80) % 4096
    rng = np.random.default_rng(14)
    for _ in range(200):
        alpha = int(rng.integers(1, 16))
        v = oracle.hash_qgram(rng.integers(0, 256, 8, dtype=np.uint8), 7, 8, alpha // 8,
                              (1 << alpha) - 1)
        assert 0 <= v < (1 << alpha)


@pytest.mark.parametrize("v,w,want", [(0, 4, 0b0001), (5, 4, 0b0010), (31, 32, 1 << 31),
                                      (32, 32, 1), (63, 64, 1 << 63)])
def test_link_hash_spec_examples(v, w, want):
    # S:95-97, Eq. 5
    assert oracle.link_hash(v, w) == want


def test_link_hash_popcount_one():
    for w in (4, 8, 16, 32, 64):
        for v in range(0, 1 << 12, 37):
            lv = oracle.link_hash(v, w)
            assert bin(lv).count("1") == 1 and lv < (1 << w)
