"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no hashing, no table, no
search): only the text / pattern generators and the per-(corpus, m) (q, alpha)
parameter table.  It is the one module both sides import (task rule 3).

The paper measures on the Pizza&Chili genome / protein / English 100 MB files
(P:379).  Those files are not available, so the seeded i.i.d. stand-ins below
(BASELINE.json configs, recipe in SURVEY.md 8(d) and DESIGN.md "Inputs")
replace them, keeping the paper's alphabet sizes and m sweep.
Patterns are copied from the text at seeded uniform offsets ("randomly
extracted from the sequences"), so every pattern occurs at least once.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

DNA = b"ACGT"
PROTEIN = b"ACDEFGHIKLMNPQRSTVWY"
# 90 printable symbols: 0x20..0x7E minus ` ~ ^ | \  (SURVEY.md 8(d), C4)
_NL_EXCLUDED = set(b"`~^|\\")
NL_SYMBOLS = bytes(c for c in range(0x20, 0x7F) if c not in _NL_EXCLUDED)
NL_HEAD = b" etaoinshrdlucmfwypvbgkjqxz"   # ranks 1..27
assert len(NL_SYMBOLS) == 90 and len(NL_HEAD) == 27


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    seed: int
    kind: str                  # dna | protein | nl | stress
    ms: tuple                  # pattern lengths
    patterns_per_m: int
    qa: dict                   # m -> (q, alpha), from the paper's tables


# (q, alpha) per m: the HC row of Table 1, Table 2, Table 3
# (P:512); m outside the paper's 8..1024 take the nearest column of the same
# table (reading R12); sigma=256 (stress) uses the English table.
QA_GENOME = {8: (4, 12), 16: (6, 12), 32: (6, 12), 64: (6, 12), 128: (6, 12),
             256: (6, 12), 512: (6, 12), 1024: (8, 12)}
QA_PROTEIN = {4: (3, 11), 8: (3, 11), 16: (3, 11), 32: (3, 11), 64: (6, 12),
              128: (3, 11), 256: (3, 11), 512: (4, 12), 1024: (4, 12)}
QA_ENGLISH = {2: (2, 11), 4: (3, 11), 8: (3, 11), 16: (3, 11), 32: (6, 12),
              64: (6, 12), 128: (3, 11), 256: (3, 11), 512: (4, 12), 1024: (4, 12),
              2048: (4, 12), 4096: (4, 12)}

CONFIGS = {
    "C1": Config("C1-dna-1MiB", 1 << 20, 1, "dna", (32,), 20, {32: (6, 12)}),
    "C2": Config("C2-dna-256MiB", 1 << 28, 2, "dna", (8, 16, 32, 64, 128, 256, 512, 1024),
                 100, QA_GENOME),
    "C3": Config("C3-protein-256MiB", 1 << 28, 3, "protein",
                 (4, 8, 16, 32, 64, 128, 256, 512, 1024), 100, QA_PROTEIN),
    "C4": Config("C4-nl-256MiB", 1 << 28, 4, "nl",
                 (2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096), 100, QA_ENGLISH),
    "C5": Config("C5-stress-1GiB", 1 << 30, 5, "stress", (32, 256), 50,
                 {32: QA_ENGLISH[32], 256: QA_ENGLISH[256]}),
}


def nl_probabilities() -> np.ndarray:
    """Zipf(s=1.1) rank frequencies p_k ~ k^-1.1, k = 1..90."""
    k = np.arange(1, 91, dtype=np.float64)
    p = k ** -1.1
    return p / p.sum()


def nl_alphabet(seed: int) -> np.ndarray:
    """Symbol of each rank: space, 'etaoinshrdlucmfwypvbgkjqxz', then the other
    63 symbols shuffled by the seed."""
    rest = np.array([c for c in NL_SYMBOLS if c not in set(NL_HEAD)], dtype=np.uint8)
    rng = np.random.default_rng([seed, 90])
    rng.shuffle(rest)
    return np.concatenate([np.frombuffer(NL_HEAD, dtype=np.uint8), rest])


def gen_text(kind: str, n: int, seed: int) -> np.ndarray:
    """Seeded text of n bytes (numpy PCG64 via default_rng)."""
    rng = np.random.default_rng(seed)
    if kind == "dna":
        return np.frombuffer(DNA, dtype=np.uint8)[rng.integers(0, 4, n)]
    if kind == "protein":
        return np.frombuffer(PROTEIN, dtype=np.uint8)[rng.integers(0, 20, n)]
    if kind == "nl":
        sym = nl_alphabet(seed)
        idx = rng.choice(90, n, p=nl_probabilities())
        return sym[idx]
    if kind == "stress":
        return gen_stress(n, seed)[0]
    if kind == "uniform256":
        return rng.integers(0, 256, n, dtype=np.uint8)
    raise ValueError(kind)


SLAB = 64 << 20


def gen_stress(n: int, seed: int):
    """C5: one seeded random 64-byte block over 256 symbols tiled to n bytes
    ('clean'), then per 64 MiB slab a Bernoulli(0.01) mask of bytes replaced by
    uniform random bytes.  Returns (text, clean_block)."""
    rng = np.random.default_rng(seed)
    block = rng.integers(0, 256, 64, dtype=np.uint8)
    y = np.tile(block, -(-n // 64))[:n].copy()
    for lo in range(0, n, SLAB):
        hi = min(n, lo + SLAB)
        mask = rng.random(hi - lo, dtype=np.float32) < 0.01
        cnt = int(mask.sum())
        seg = y[lo:hi]
        seg[mask] = rng.integers(0, 256, cnt, dtype=np.uint8)
    return y, block


def clean_text(block: np.ndarray, lo: int, length: int) -> np.ndarray:
    """Bytes [lo, lo+length) of the unmutated periodic text."""
    idx = (np.arange(lo, lo + length) % 64)
    return block[idx]


def pattern_offsets(cfg_seed: int, m: int, n: int, count: int, salt: int = 0) -> np.ndarray:
    """Uniform offsets over [0, n-m] from default_rng([text_seed, m(, salt)])."""
    key = [cfg_seed, m] if salt == 0 else [cfg_seed, m, salt]
    rng = np.random.default_rng(key)
    return rng.integers(0, n - m + 1, count)


def patterns(cfg: Config, text: np.ndarray, m: int, count: int | None = None,
             salt: int = 0, block: np.ndarray | None = None):
    """List of (offset, pattern bytes as uint8 array).  For the stress config the
    pattern is cut from the unmutated periodic text (block rotation)."""
    cnt = cfg.patterns_per_m if count is None else count
    offs = pattern_offsets(cfg.seed, m, len(text), cnt, salt)
    out = []
    for o in offs:
        o = int(o)
        if cfg.kind == "stress":
            assert block is not None
            out.append((o, clean_text(block, o, m)))
        else:
            out.append((o, text[o:o + m].copy()))
    return out


def config_text(cfg: Config, n: int | None = None):
    """Text of the config (optionally truncated to n bytes for small tests);
    returns (text, block_or_None)."""
    nn = cfg.n if n is None else n
    if cfg.kind == "stress":
        return gen_stress(nn, cfg.seed)
    return gen_text(cfg.kind, nn, cfg.seed), None


def sha256(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
