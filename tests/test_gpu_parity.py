"""GPU parity: the CUDA path (through the C-ABI) against the oracle, element by
element, on seeded inputs sized so the oracle finishes in seconds but the
kernels see many tiles, many lane chunks and ragged tails.  Bit-exact: same
count, same ascending position list (integer work)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2310_15711_b200 import hc  # noqa: E402
from paper_2310_15711_b200 import inputs as I  # noqa: E402

PATHS = [hc.PATH_STAGED, hc.PATH_GATHER, hc.PATH_STREAM, hc.PATH_SHC, hc.PATH_SCAN, hc.PATH_AUTO]


def to_dev(y: np.ndarray, offset: int = 0):
    """y on the device starting `offset` bytes past a 256-aligned allocation."""
    buf = torch.empty(len(y) + offset + 1, dtype=torch.uint8, device="cuda")
    buf[len(y) + offset:] = 0xA5
    if len(y):
        buf[offset:offset + len(y)] = torch.from_numpy(np.ascontiguousarray(y)).cuda()
    return buf[offset:offset + len(y)]


def gpu(h, y_dev, max_out=None, **kw):
    res = hc.search(h, y_dev, max_out=max_out, **kw)
    torch.cuda.synchronize()
    return res.cpu().numpy()


def test_table_parity_with_oracle():
    rng = np.random.default_rng(51)
    for _ in range(100):
        q = int(rng.integers(1, 9))
        m = int(rng.integers(q, 200))
        alpha = int(rng.integers(1, 16))
        x = rng.integers(0, 256, m, dtype=np.uint8)
        h = hc.prepare(x, q, alpha)
        t = h.table()
        o = oracle.preprocess(x, q, alpha, w=32)
        assert np.array_equal(t.F.astype(np.uint64), o.F) and t.hv == o.hv and t.s == o.s


def test_spec_examples():
    y = to_dev(np.frombuffer(b"aaaa", np.uint8))
    for q in (1, 2):
        for path in PATHS:
            assert gpu(hc.prepare(b"aa", q, 8), y, path=path).tolist() == [0, 1, 2]
    y = to_dev(np.frombuffer(b"zzzz", np.uint8))
    assert gpu(hc.prepare(b"abc", 2, 8), y).tolist() == []


@pytest.mark.parametrize("path", PATHS)
def test_random_small(path):
    rng = np.random.default_rng(52 + path)
    for trial in range(120):
        sigma = int(rng.choice([2, 4, 20, 64, 256]))
        q = int(rng.integers(1, 9))
        m = int(rng.integers(q, 140))
        alpha = int(rng.integers(1, 16))
        n = int(rng.integers(0, 60_000))
        y = rng.integers(0, sigma, n, dtype=np.uint8)
        if n >= m and rng.random() < 0.8:
            o = int(rng.integers(0, n - m + 1))
            x = y[o:o + m].copy()
            for p in rng.integers(0, n - m + 1, 5):
                y[p:p + m] = x
        else:
            x = rng.integers(0, sigma, m, dtype=np.uint8)
        want = oracle.brute(x, y)
        h = hc.prepare(x, q, alpha)
        off = int(rng.integers(0, 16))
        got = gpu(h, to_dev(y, off), path=path)
        assert np.array_equal(got, want), (trial, m, q, alpha, n, off, len(want), len(got))


@pytest.mark.parametrize("path", [hc.PATH_STAGED, hc.PATH_GATHER, hc.PATH_STREAM, hc.PATH_SHC,
                                  hc.PATH_SCAN])
@pytest.mark.parametrize("max_ctas,stages", [(1, 2), (2, 3), (3, 4), (5, 1)])
def test_many_tiles_per_cta(path, max_ctas, stages):
    # tiny tiles / few CTAs: every CTA cycles its TMA ring many times
    rng = np.random.default_rng(53)
    y = I.gen_text("dna", 300_001, 53)
    for m, q in [(8, 4), (16, 6), (32, 6), (33, 3), (100, 8), (7, 7)]:
        x = y[12345:12345 + m].copy()
        yy = y.copy()
        for p in rng.integers(0, len(y) - m, 40):
            yy[p:p + m] = x
        want = oracle.brute(x, yy)
        h = hc.prepare(x, q, 12)
        got = gpu(h, to_dev(yy, 3), path=path, tile_bytes=64, stages=stages, max_ctas=max_ctas,
                  seg_per_lane=1)
        assert np.array_equal(got, want), (m, q)


@pytest.mark.parametrize("path", PATHS)
def test_plant_at_every_offset_near_tile_and_text_edges(path):
    # occurrences at every offset within +-m of text ends; texts of every length
    # around m and ragged tails
    rng = np.random.default_rng(54)
    for m, q in [(5, 2), (16, 6), (40, 4)]:
        x = rng.integers(200, 256, m, dtype=np.uint8)  # bytes >= 0x80
        for n in list(range(0, m + 3)) + [m + 31, 2 * m + 17, 1000, 4099]:
            base = rng.integers(0, 4, n, dtype=np.uint8)
            ps = [p for p in range(0, max(0, n - m + 1)) if p < m + 2 or p > n - 2 * m - 2]
            for p in ps[:: max(1, len(ps) // 12)] if ps else [None]:
                y = base.copy()
                if p is not None:
                    y[p:p + m] = x
                want = oracle.brute(x, y)
                for off in (0, 7, 15):
                    got = gpu(hc.prepare(x, q, 11), to_dev(y, off), path=path)
                    assert np.array_equal(got, want), (m, n, p, off)


@pytest.mark.parametrize("path", PATHS)
def test_all_positions_match(path):
    # a^m in a^n: n-m+1 occurrences: every window completes its walk and verifies
    for m, q, n in [(1, 1, 5000), (2, 2, 70_000), (8, 3, 40_000), (64, 6, 100_000), (300, 8, 50_000)]:
        h = hc.prepare(b"a" * m, q, 12)
        got = gpu(h, to_dev(np.full(n, ord("a"), np.uint8), 5), path=path)
        assert len(got) == n - m + 1
        assert np.array_equal(got, np.arange(n - m + 1))


@pytest.mark.parametrize("path", PATHS)
def test_max_out_and_count_only(path):
    rng = np.random.default_rng(55)
    y = rng.integers(0, 2, 200_000, dtype=np.uint8)
    x = y[500:510].copy()
    want = oracle.brute(x, y)
    assert len(want) > 100
    h = hc.prepare(x, 5, 10)
    yd = to_dev(y)
    assert hc.count(h, yd, path=path) == len(want)
    for k in (1, 7, len(want) - 1, len(want), len(want) + 10):
        got = gpu(h, yd, max_out=k, path=path)
        assert np.array_equal(got, want[:k])


def test_scratch_overflow_rerun():
    # more occurrences than the default scratch (2^16): the library re-runs with room
    n = 300_000
    y = np.zeros(n, np.uint8)
    h = hc.prepare(bytes(3), 3, 12)
    res, st = hc.search(h, to_dev(y), max_out=10, stats=True)
    assert st["reruns"] == 1
    assert res.cpu().numpy().tolist() == list(range(10))
    assert hc.count(h, to_dev(y)) == n - 2


def test_host_entry_point():
    rng = np.random.default_rng(56)
    y = rng.integers(0, 4, 123_457, dtype=np.uint8)
    x = y[999:1031].copy()
    h = hc.prepare(x, 6, 12)
    assert np.array_equal(hc.search_host(h, y), oracle.brute(x, y))
    assert hc.search_host(h, y[:10]).tolist() == []


def test_batch_host_entry_point():
    """hc_search_batch_host: host text in, host positions out, every pattern equal to brute
    force (mixed m, an absent pattern, max_out truncation, counts only)."""
    rng = np.random.default_rng(58)
    y = rng.integers(0, 4, 1_000_003, dtype=np.uint8)
    pats = []
    for m, q, a in [(8, 4, 12), (32, 6, 12), (300, 6, 12), (3, 2, 8)]:
        o = int(rng.integers(0, len(y) - m))
        pats.append((y[o:o + m].copy(), q, a))
    pats.append((np.frombuffer(b"ACGTZ", np.uint8), 2, 10))
    hs = [hc.prepare(x, q, a) for x, q, a in pats]
    want = [oracle.brute(x, y) for x, _, _ in pats]
    for g, w in zip(hc.search_batch_host(hs, y), want):
        assert np.array_equal(g, w)
    for g, w in zip(hc.search_batch_host(hs, y, max_out=3), want):
        assert np.array_equal(g, w[:3])
    assert hc.search_batch_host_raw(hs, y.ctypes.data, len(y), None, None) == [len(w) for w in want]


def test_time_kernel_stats():
    """time_kernel = 2: the search kernel's own device time is reported and lies inside
    the call's device time."""
    y = to_dev(I.gen_text("dna", 4_000_000, 59))
    h = hc.prepare(y[1000:1032].cpu().numpy(), 6, 12)
    _, st = hc.search(h, y, stats=True, time_kernel=2)
    assert 0 < st["search_ms"] <= st["kernel_ms"]
    _, st = hc.search(h, y, stats=True, time_kernel=1)
    assert st["kernel_ms"] > 0 and st["search_ms"] == 0


def test_errors():
    h = hc.prepare(b"abcd", 2, 8)
    with pytest.raises(hc.HCError) as ei:
        hc.search_raw(h, 0, 100, None, 0, 0)
    assert ei.value.code == hc.HC_EINVAL
    assert hc.search_raw(h, 0, 0, None, 0, 0) == 0          # n = 0 -> 0
    # measurement-only modes are compiled out of the product library
    y = to_dev(np.frombuffer(b"xxabcdxx", np.uint8))
    for kw in ({"debug": 3}, {"trace": 8}):
        with pytest.raises(hc.HCError) as ei:
            hc.search(h, y, **kw)
        assert ei.value.code == hc.HC_EINVAL
    with pytest.raises(hc.HCError):
        hc.prepare(b"ab", 3, 8)


def test_c1_config_exact():
    cfg = I.CONFIGS["C1"]
    y, _ = I.config_text(cfg)
    yd = to_dev(y)
    q, a = cfg.qa[32]
    for o, x in I.patterns(cfg, y, 32):
        want = oracle.brute(x, y)
        assert o in want.tolist()
        for path in PATHS:
            assert np.array_equal(gpu(hc.prepare(x, q, a), yd, path=path), want)


@pytest.mark.parametrize("world", [2, 3, 7])
def test_text_shards_on_one_gpu(world):
    # the shards' searches (real kernels, sliced device text with the
    # (m-1)-byte halo), offset and concatenated in rank order, give the whole answer
    from paper_2310_15711_b200.shard import shard_bounds
    rng = np.random.default_rng(61 + world)
    y = I.gen_text("dna", 1_000_003, 61)
    for m, q in [(8, 4), (32, 6), (200, 6)]:
        x = y[777:777 + m].copy()
        yy = y.copy()
        cuts = [shard_bounds(len(y), m, world, r).end_lo for r in range(1, world)]
        for c in cuts:                       # occurrences straddling every cut
            for d in (0, 1, m // 2, m - 1):
                p = c - d
                if 0 <= p <= len(y) - m:
                    yy[p:p + m] = x
        for p in rng.integers(0, len(y) - m, 20):
            yy[p:p + m] = x
        want = oracle.brute(x, yy)
        h = hc.prepare(x, q, 12)
        yd = to_dev(yy, 5)
        parts = []
        for r in range(world):
            sh = shard_bounds(len(yy), m, world, r)
            if sh.size >= m:
                parts.append(gpu(h, yd[sh.text_lo:sh.text_hi]) + sh.text_lo)
        got = np.concatenate(parts)
        assert np.array_equal(got, want), (world, m)


def test_search_sharded_nccl_single_rank():
    # the exchange path over NCCL (world size 1 on the one GPU)
    import os
    import torch.distributed as dist
    from paper_2310_15711_b200.shard import search_sharded, shard_bounds
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        y = I.gen_text("dna", 300_000, 62)
        x = y[1000:1032].copy()
        sh = shard_bounds(len(y), 32, 1, 0)
        yd = to_dev(y)
        total, pos = search_sharded(hc.prepare(x, 6, 12), yd[sh.text_lo:sh.text_hi], sh)
        want = oracle.brute(x, y)
        assert total == len(want) and np.array_equal(pos.cpu().numpy(), want)
    finally:
        dist.destroy_process_group()


def test_search_batch_matches_single_searches():
    # hc_search_batch: every pattern's result is exactly hc_search's,
    # with mixed m / q / alpha / paths, zero and high occurrence counts (re-runs)
    rng = np.random.default_rng(71)
    y = I.gen_text("dna", 2_000_003, 71)
    yy = y.copy()
    specs = [(8, 4, 12), (16, 6, 12), (32, 6, 12), (33, 3, 11), (64, 6, 12), (200, 6, 12),
             (512, 6, 12), (1024, 8, 12), (5, 5, 10), (3, 2, 8)]
    pats = []
    for m, q, a in specs:
        o = int(rng.integers(0, len(y) - m))
        x = y[o:o + m].copy()
        for p in rng.integers(0, len(y) - m, 7):
            yy[p:p + m] = x
        pats.append((x, q, a))
    pats.append((np.frombuffer(b"ZZZZZZZZZZ", np.uint8), 3, 12))      # absent
    yd = to_dev(yy, 9)
    hs = [hc.prepare(x, q, a) for x, q, a in pats]
    want = [oracle.brute(x, yy) for x, _, _ in pats]
    got = hc.search_batch(hs, yd)
    torch.cuda.synchronize()
    for g, w in zip(got, want):
        assert np.array_equal(g.cpu().numpy(), w)
    # max_out truncation and counts; a tiny scratch forces the re-run path for m=3
    got, st = hc.search_batch(hs, yd, max_out=5, stats=True, time_kernel=1)
    for g, w in zip(got, want):
        assert np.array_equal(g.cpu().numpy(), w[:5])
    assert st["kernel_ms"] > 0
    cnts = hc.search_batch_raw(hs, yd.data_ptr(), yd.numel(), None, None, 0)
    assert cnts == [len(w) for w in want]


@pytest.mark.parametrize("path", [hc.PATH_STREAM, hc.PATH_GATHER, hc.PATH_SHC, hc.PATH_SCAN])
def test_ordering_paths(path):
    """Occurrence counts across every ordering branch of the finish kernel (rank count
    <= 256, bucket pass, skewed buckets -> block radix sort, > 8192 -> device sort),
    with the occurrences spread over the text or packed into one stretch."""
    rng = np.random.default_rng(57)
    n = 1 << 20
    for count, packed in [(2, False), (200, False), (300, False), (5000, False), (5000, True),
                          (8192, False), (8192, True), (8193, True), (20000, False)]:
        y = rng.integers(0, 4, n, dtype=np.uint8)           # bytes 0..3: "xy" never occurs
        x = np.frombuffer(b"xy", np.uint8)
        if packed:
            start = int(rng.integers(0, n - 2 * count - 2))
            ps = start + 2 * np.arange(count)
        else:
            ps = np.sort(rng.choice((n - 2) // 2, count, replace=False)) * 2
        for p in ps:
            y[p:p + 2] = x
        want = oracle.brute(x, y)
        assert len(want) == count
        got = gpu(hc.prepare(x, 2, 12), to_dev(y, 3), path=path)
        assert np.array_equal(got, want), (count, packed, len(got))


@pytest.mark.parametrize("no_multi", [0, 1, 2])
def test_search_batch_multi_pattern_groups(no_multi):
    """Multi-pattern launches (patterns sharing m, q, alpha filtered in one pass over the
    text; staged for shifts <= 32, gather access up to 256, single beyond): groups of
    1..4 and a partial last group, patterns with many occurrences (one
    over the scratch, one over the in-kernel ordering bound), absent patterns,
    overlapping occurrences, unaligned text; every result equals brute force."""
    rng = np.random.default_rng(73)
    y = I.gen_text("dna", 3_000_017, 73)
    yy = y.copy()
    pats = []
    for m, q, a, count in [(8, 4, 12, 9), (16, 6, 12, 6), (16, 3, 11, 5), (32, 6, 12, 3), (4, 2, 10, 2),
                           (24, 8, 12, 5), (64, 6, 12, 6), (100, 3, 11, 4), (250, 8, 12, 5),
                           (300, 6, 12, 2)]:
        for t in range(count):
            o = int(rng.integers(0, len(y) - m))
            x = y[o:o + m].copy()
            if t == 1:
                x = rng.permutation(x)                           # likely absent
            for p in rng.integers(0, len(y) - m, int(rng.integers(0, 9))):
                yy[p:p + m] = x
            pats.append((x, q, a))
    # very frequent patterns inside a group (count > 8192 and > the 65536 scratch)
    pats.insert(3, (np.frombuffer(b"AAAA", np.uint8), 2, 12))
    yy[1000:1000 + 300_000] = ord("A")
    pats.insert(5, (np.frombuffer(b"ACGT", np.uint8), 2, 12))
    yd = to_dev(yy, 5)
    hs = [hc.prepare(x, q, a) for x, q, a in pats]
    want = [oracle.brute(x, yy) for x, _, _ in pats]
    got = hc.search_batch(hs, yd, no_multi=no_multi)
    torch.cuda.synchronize()
    for k, (g, w) in enumerate(zip(got, want)):
        assert np.array_equal(g.cpu().numpy(), w), (k, len(g), len(w))
    got = hc.search_batch(hs, yd, max_out=3, no_multi=no_multi)
    for g, w in zip(got, want):
        assert np.array_equal(g.cpu().numpy(), w[:3])


def test_prepare_batch_equals_prepare():
    """hc_prepare_batch: same tables and H_v as hc_prepare for every pattern, the same
    search results, and handles usable and destroyable in any order."""
    rng = np.random.default_rng(75)
    y = I.gen_text("protein", 500_009, 75)
    for q, a in [(3, 11), (6, 12), (1, 8), (8, 15)]:
        xs = []
        for _ in range(7):
            m = int(rng.integers(q, 90))
            o = int(rng.integers(0, len(y) - m))
            xs.append(y[o:o + m].copy())
        hb = hc.prepare_batch(xs, q, a)
        yd = to_dev(y, 1)
        for x, h in zip(xs, hb):
            t1, t2 = h.table(), hc.prepare(x, q, a).table()
            assert np.array_equal(t1.F, t2.F) and t1.hv == t2.hv and t1.s == t2.s
            assert np.array_equal(gpu(h, yd), oracle.brute(x, y))
        got = hc.search_batch(hb, yd)
        for x, g in zip(xs, got):
            assert np.array_equal(g.cpu().numpy(), oracle.brute(x, y))
        for h in hb[::2]:
            h.close()
        assert np.array_equal(gpu(hb[1], yd), oracle.brute(xs[1], y))
        for h in hb[1::2]:
            h.close()
    with pytest.raises(hc.HCError):
        hc.prepare_batch([b"abc", b"a"], 2, 8)       # q > m for the second pattern


@pytest.mark.parametrize("path", [hc.PATH_AUTO, hc.PATH_STAGED, hc.PATH_GATHER, hc.PATH_STREAM, hc.PATH_SHC,
                                  hc.PATH_SCAN])
def test_largest_tables_every_path(path):
    """alpha = 15 (F = 128 KiB, the largest table) with short and long patterns on every
    path: each either fits its shared-memory layout or falls back (stream -> gather);
    SHC may refuse a layout it cannot fit (HC_EINVAL), never a failed launch."""
    rng = np.random.default_rng(77)
    y = I.gen_text("nl", 400_003, 77)
    for m, q in [(6, 3), (20, 5), (40, 8), (150, 6)]:
        o = int(rng.integers(0, len(y) - m))
        x = y[o:o + m].copy()
        want = oracle.brute(x, y)
        h = hc.prepare(x, q, 15)
        try:
            got = gpu(h, to_dev(y, 2), path=path)
        except hc.HCError as e:
            assert path in (hc.PATH_SHC, hc.PATH_SCAN) and e.code == -1, (m, q, e)
            continue
        assert np.array_equal(got, want), (m, q)


def _all_qs_builds():
    """Every (q, s) kernel build the ABI can reach: 1 <= q <= 8, 1 <= alpha <= 15,
    s = floor(alpha / q) (Eq. 4; s = 0 when q > alpha, reading R6).  For q = 1
    the hash is the byte itself (one build, s plays no role)."""
    builds = {}
    for q in range(1, 9):
        for alpha in range(1, 16):
            key = (q, 0 if q == 1 else alpha // q)
            builds.setdefault(key, []).append(alpha)
    return builds


@pytest.mark.parametrize("path", PATHS)
def test_every_kernel_build(path):
    """Every (q, s) instantiation, every alpha in 1..15 (the scalar F-load branch at
    alpha <= 1, s = 0 at q > alpha), short and long patterns (m = q, m < 2q for the
    while-else of R7, walks of several steps, m > 64 for the warp-wide verification),
    planted occurrences, unaligned text: element-wise equal to brute force (O1)."""
    builds = _all_qs_builds()
    assert len(builds) == 31
    rng = np.random.default_rng(81 + path)
    seen = set()
    for (q, s), alphas in sorted(builds.items()):
        for alpha in alphas:
            sigma = int(rng.choice([2, 4, 20, 256]))
            y = rng.integers(0, sigma, int(rng.integers(20_000, 40_000)), dtype=np.uint8)
            for m in sorted({q, q + 1, 2 * q - 1 if q > 1 else 1, 2 * q + 3, 37, 150}):
                if m < q:
                    continue
                o = int(rng.integers(0, len(y) - m))
                x = y[o:o + m].copy()
                yy = y.copy()
                for p in rng.integers(0, len(y) - m, 6):
                    yy[p:p + m] = x
                want = oracle.brute(x, yy)
                h = hc.prepare(x, q, alpha)
                t = h.table()
                assert t.s == (alpha // q)
                off = int(rng.integers(0, 16))
                try:
                    got = gpu(h, to_dev(yy, off), path=path)
                except hc.HCError as e:        # SHC may refuse a layout it cannot fit
                    assert path in (hc.PATH_SHC, hc.PATH_SCAN) and e.code == hc.HC_EINVAL, (q, alpha, m, e)
                    continue
                assert np.array_equal(got, want), (q, s, alpha, m, off, len(got), len(want))
                seen.add((q, s))
    assert seen == set(builds), sorted(set(builds) - seen)


@pytest.mark.parametrize("path", PATHS)
def test_long_patterns(path):
    """m in the thousands (warp-wide walks of hundreds of steps, 1 KiB verification
    rounds) and m = HC_MAX_PATTERN = 65536: the default path must search exactly; a
    forced path either searches exactly or refuses the layout with HC_EINVAL."""
    rng = np.random.default_rng(83)
    y = I.gen_text("protein", 600_011, 83)
    for m, q, alpha in [(4099, 4, 12), (8000, 6, 12), (12_345, 3, 11), (16_000, 8, 15), (65_536, 4, 12)]:
        o = int(rng.integers(0, len(y) - m))
        x = y[o:o + m].copy()
        yy = y.copy()
        for p in rng.integers(0, len(y) - m, 3):
            yy[p:p + m] = x
        yy[o + m // 2] ^= 1 if rng.random() < 0.5 else 0     # sometimes a near-miss at o
        want = oracle.brute(x, yy)
        h = hc.prepare(x, q, alpha)
        try:
            got = gpu(h, to_dev(yy, 7), path=path)
        except hc.HCError as e:
            assert path in (hc.PATH_SHC, hc.PATH_STAGED, hc.PATH_SCAN) and e.code == hc.HC_EINVAL, (m, e)
            continue
        assert np.array_equal(got, want), (m, q, alpha, len(got), len(want))
    with pytest.raises(hc.HCError) as ei:
        hc.prepare(bytes(65_537), 4, 12)
    assert ei.value.code == hc.HC_ETOOLONG


def test_stream_chunk_copies():
    """The stream path's chunk copies (one 1-D TMA bulk copy per chunk): unaligned texts,
    edge chunks (the first chunk, the last chunks, texts ending inside a 16-byte word),
    shifts below q (m < 2q), small chunks (many interior chunks per warp), few warps per
    CTA, both final drains, against brute force."""
    rng = np.random.default_rng(79)
    for n in (1000, 70_001, 1_000_003):
        y = I.gen_text("dna", n, 79 + n % 7)
        for m, q in [(8, 4), (16, 6), (32, 6), (13, 2), (4, 3), (9, 8)]:
            o = int(rng.integers(0, n - m))
            x = y[o:o + m].copy()
            want = oracle.brute(x, y)
            for off in (0, 5, 15):
                for bw, tile, spl in ((0, 0, 0), (8, 0, 0), (0, 700, 0), (3, 700, -1), (0, 0, -1)):
                    # seg_per_lane < 0: final drain on global text instead of private boxes
                    got = gpu(hc.prepare(x, q, 12), to_dev(y, off), path=hc.PATH_STREAM,
                              block_warps=bw, tile_bytes=tile, max_ctas=3 if tile else 0,
                              seg_per_lane=spl)
                    assert np.array_equal(got, want), (n, m, off, bw, tile, spl)


def test_epilogue_ordering_any_block_size():
    """The fused epilogue orders up to 8,192 positions in the last CTA, whatever its size:
    stream CTAs of 1..24 warps (the default is one 24-warp CTA per SM; fewer warps when
    alpha is large), counts from a few hundred (bucket pass) to just below and above the
    epilogue's capacity (host ordering)."""
    rng = np.random.default_rng(97)
    for n, m in ((40_000, 3), (200_000, 3), (450_000, 3), (700_000, 3)):
        y = rng.integers(0, 4, n, dtype=np.uint8)
        x = y[77:77 + m].copy()
        want = oracle.brute(x, y)
        for bw in (1, 3, 5, 8, 12, 20, 24):
            for alpha in (8, 12):
                got = gpu(hc.prepare(x, 2, alpha), to_dev(y, 3), path=hc.PATH_STREAM, block_warps=bw)
                assert np.array_equal(got, want), (n, bw, alpha, len(got), len(want))
