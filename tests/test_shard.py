"""Multi-rank text sharding (paper_2310_15711_b200/shard.py) on CPU:
gloo, world_size 2 and 3, with the oracle's brute force as the per-rank searcher
(test infrastructure only; the product path uses the CUDA search).  Checks that the
shards partition the window ends exactly (reading R11) and that the exchange
returns the whole-text answer, in order, on every rank, including occurrences that
straddle shard boundaries, empty shards and max_out truncation."""
import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2310_15711_b200 import inputs as I
from paper_2310_15711_b200.shard import Shard, search_sharded, shard_bounds


def test_shard_bounds_partition_window_ends():
    for n in [0, 1, 5, 17, 100, 1001]:
        for m in [1, 2, 7, 32]:
            for world in [1, 2, 3, 5, 8]:
                ends = []
                for r in range(world):
                    s = shard_bounds(n, m, world, r)
                    assert isinstance(s, Shard)
                    if s.size:
                        # the slice holds every window ending in [end_lo, end_hi)
                        assert s.text_lo == s.end_lo - m + 1 and s.text_hi == s.end_hi
                        assert s.text_lo >= 0 and s.text_hi <= n
                    ends.extend(range(s.end_lo, s.end_hi))
                assert ends == list(range(m - 1, n)), (n, m, world)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _brute_searcher(h, y_slice, max_out):
    pos = oracle.brute(h.x, y_slice.numpy())
    if max_out is not None:
        pos = pos[:max_out]
    return torch.from_numpy(np.asarray(pos, dtype=np.int64))


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = []
        for y, x, max_out in cases:
            h = SimpleNamespace(m=len(x), x=x)
            sh = shard_bounds(len(y), len(x), world, rank)
            y_slice = torch.from_numpy(y[sh.text_lo:sh.text_hi].copy())
            total, pos = search_sharded(h, y_slice, sh, max_out=max_out, searcher=_brute_searcher)
            res.append((total, pos.tolist()))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _cases():
    rng = np.random.default_rng(81)
    cases = []
    y = I.gen_text("dna", 5000, 81)
    x = y[1234:1234 + 12].copy()
    yy = y.copy()
    for p in [0, 1666 - 6, 2499 - 5, 2500 - 11, 3333 - 7, 4988]:   # around shard cuts
        yy[p:p + 12] = x
    cases.append((yy, x, None))
    cases.append((yy, x, 3))                                       # max_out truncation
    a = np.full(300, ord("a"), dtype=np.uint8)
    cases.append((a, a[:64].copy(), None))                        # every window matches
    cases.append((a[:5], a[:3].copy(), None))                     # n < world * m: empty shards
    cases.append((rng.integers(0, 4, 2000, dtype=np.uint8), np.array([1, 2], np.uint8), None))
    return cases


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_search_gloo(world):
    cases = _cases()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for i, (y, x, max_out) in enumerate(cases):
        want = oracle.brute(x, y).tolist()
        for r in range(world):
            total, pos = out[r][i]
            if max_out is None:
                assert total == len(want) and pos == want, (i, r)
            else:
                assert pos == want[:max_out], (i, r)
