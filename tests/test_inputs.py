"""Seeded input generators (paper_2310_15711_b200/inputs.py): determinism and
the shape of the stand-in workloads."""
import numpy as np

from paper_2310_15711_b200 import inputs as I


def test_deterministic():
    a = I.gen_text("dna", 100_000, 2)
    b = I.gen_text("dna", 100_000, 2)
    assert np.array_equal(a, b) and I.sha256(a) == I.sha256(b)
    assert not np.array_equal(a, I.gen_text("dna", 100_000, 3))


def test_alphabets():
    assert set(np.unique(I.gen_text("dna", 50_000, 1)).tobytes()) == set(b"ACGT")
    assert set(np.unique(I.gen_text("protein", 50_000, 3)).tobytes()) == set(I.PROTEIN)
    nl = I.gen_text("nl", 400_000, 4)
    assert set(np.unique(nl).tobytes()) <= set(I.NL_SYMBOLS)
    # rank 1 = space with p1 ~ 0.2374, rank 2 = 'e'
    f = np.bincount(nl, minlength=256) / len(nl)
    assert abs(f[ord(" ")] - I.nl_probabilities()[0]) < 0.01
    assert f[ord("e")] > f[ord("t")] > f[ord("z")]
    assert abs(I.nl_probabilities()[0] - 0.2374) < 1e-3


def test_dna_frequencies():
    y = I.gen_text("dna", 1_000_000, 42)
    f = np.bincount(y, minlength=256)[list(b"ACGT")] / len(y)
    assert np.all(np.abs(f - 0.25) < 0.0025)     # within 1% of n/4


def test_stress_shape():
    y, block = I.gen_stress(3 * 1024 * 1024, 5)
    clean = I.clean_text(block, 0, len(y))
    frac = np.mean(y != clean)
    assert 0.0095 < frac < 0.0105                  # ~1% replaced, ~0.996% changed
    assert np.array_equal(I.clean_text(block, 64, 64), block)


def test_patterns_occur_at_offsets():
    cfg = I.CONFIGS["C1"]
    y, _ = I.config_text(cfg)
    assert len(y) == 1 << 20
    for o, x in I.patterns(cfg, y, 32):
        assert len(x) == 32 and np.array_equal(y[o:o + 32], x)
    assert [o for o, _ in I.patterns(cfg, y, 32)] == [o for o, _ in I.patterns(cfg, y, 32)]


def test_qa_table_covers_config_ms():
    for cfg in I.CONFIGS.values():
        for m in cfg.ms:
            q, a = cfg.qa[m]
            assert 1 <= q <= m and 8 <= a <= 15
