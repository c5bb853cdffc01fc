"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (default options): C2-C4 (256 MiB) and C5 (1 GiB), a sample of each
config's patterns per m, compared bit-exact with the oracle (O1 brute force,
threaded over the host cores) and, for C5, with an independent closed form
of the occurrence set."""
import os

import numpy as np
import pytest

import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2310_15711_b200 import hc  # noqa: E402
from paper_2310_15711_b200 import inputs as I  # noqa: E402

PER_M = int(os.environ.get("HC_TEST_PATTERNS_PER_M", "3"))


def run_config(key, per_m=PER_M):
    cfg = I.CONFIGS[key]
    y, block = I.config_text(cfg)
    yd = torch.from_numpy(y).cuda()
    checked = 0
    for m in cfg.ms:
        q, a = cfg.qa[m]
        for o, x in I.patterns(cfg, y, m, block=block)[:per_m]:
            h = hc.prepare(x, q, a)
            got = hc.search(h, yd).cpu().numpy()
            want = oracle.brute_threaded(x, y)
            assert np.array_equal(got, want), (key, m, o, len(got), len(want))
            if cfg.kind != "stress":
                assert o in set(want[:100000].tolist()) or o in set(want.tolist())
            checked += 1
    return checked


def test_c2_dna_full():
    assert run_config("C2") == 8 * PER_M


def test_c3_protein_full():
    assert run_config("C3") == 9 * PER_M


def test_c4_nl_full():
    assert run_config("C4") == 12 * PER_M


def test_c5_stress_closed_form():
    """C5: occurrences of a block rotation x = clean[o:o+m] are exactly the p = o mod 64
    whose window has no mutated byte, when the 64-byte block is primitive (checked)."""
    cfg = I.CONFIGS["C5"]
    y, block = I.config_text(cfg)
    clean = np.tile(block, len(y) // 64)
    # primitive block: no proper rotation equals it
    assert all(not np.array_equal(np.roll(block, r), block) for r in range(1, 64))
    bad = np.concatenate([[0], np.cumsum(y != clean, dtype=np.int64)])
    yd = torch.from_numpy(y).cuda()
    for m in cfg.ms:
        q, a = cfg.qa[m]
        for o, x in I.patterns(cfg, y, m, block=block)[:2]:
            p = np.arange(o % 64, len(y) - m + 1, 64, dtype=np.int64)
            closed = p[bad[p + m] - bad[p] == 0]
            got = hc.search(hc.prepare(x, q, a), yd).cpu().numpy()
            assert np.array_equal(got, closed), (m, o, len(got), len(closed))
            # and the brute-force oracle on a 16 MiB slice with its own offsets
            lo, hi = 300 << 20, (316 << 20) + m - 1
            want = oracle.brute_threaded(x, y[lo:hi]) + lo
            sel = got[(got >= lo) & (got <= hi - m)]
            assert np.array_equal(sel, want)


def test_c2_batch_multi_pattern_full():
    """The bench's batch launch configuration at full size: hc_search_batch over C2's
    text with 4 patterns per m (one multi-pattern launch each for m <= 32), every
    result equal to the brute-force oracle."""
    cfg = I.CONFIGS["C2"]
    y, block = I.config_text(cfg)
    yd = torch.from_numpy(y).cuda()
    for m in (8, 16, 32, 64):
        q, a = cfg.qa[m]
        pats = [x for _, x in I.patterns(cfg, y, m, block=block)[:4]]
        got = hc.search_batch(hc.prepare_batch(pats, q, a), yd)
        for x, g in zip(pats, got):
            assert np.array_equal(g.cpu().numpy(), oracle.brute_threaded(x, y)), m
