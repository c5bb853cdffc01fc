#!/usr/bin/env python
"""GPU (q, alpha) sweep: for each m of a config, the search time of
every (q, alpha) on the paper's grid 1 <= q <= 8, 8 <= alpha <= 12, extended to
alpha <= 15 (F still fits in shared memory), median over a few patterns; the best
pair per m is reported beside the paper-prescribed one (Tables 1-3).  Every result
is checked against the count of the paper's (q, alpha) (the answer does not depend
on q and alpha).

    python tools/qa_sweep.py --config C2 --patterns 5 --out profiles/r01_qa_sweep_C2.json
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2310_15711_b200 import hc  # noqa: E402
from paper_2310_15711_b200 import inputs as I  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--patterns", type=int, default=5)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--alphas", type=int, nargs="+", default=[8, 9, 10, 11, 12, 13, 14, 15])
    ap.add_argument("--qs", type=int, nargs="+", default=[1, 2, 3, 4, 5, 6, 7, 8])
    ap.add_argument("--ms", type=int, nargs="+", default=None)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    cfg = I.CONFIGS[args.config]
    y_np, block = I.config_text(cfg)
    y = torch.from_numpy(y_np).cuda()
    n = len(y_np)
    flush = torch.ones(2 * torch.cuda.get_device_properties(0).L2_cache_size, dtype=torch.uint8,
                       device="cuda")
    res = {"config": cfg.name, "n": n, "patterns_per_point": args.patterns, "per_m": {}}
    for m in (args.ms or cfg.ms):
        pats = I.patterns(cfg, y_np, m, count=args.patterns, block=block)
        q0, a0 = cfg.qa[m]
        want = [hc.count(hc.prepare(x, q0, a0), y) for _, x in pats]
        grid = {}
        for q in args.qs:
            if q > m:
                continue
            for a in args.alphas:
                ts = []
                for (_, x), c in zip(pats, want):
                    h = hc.prepare(x, q, a)
                    for _ in range(args.reps):
                        flush.view(torch.int64).sum()
                        r, st = hc.search(h, y, max_out=0, stats=True, time_kernel=1)
                        ts.append(st["kernel_ms"])
                    got = hc.count(h, y)
                    assert got == c, (m, q, a, got, c)
                    h.close()
                grid[f"{q},{a}"] = round(statistics.median(ts) * 1e3, 2)
        best = min(grid, key=grid.get)
        res["per_m"][str(m)] = {
            "paper": {"q": q0, "alpha": a0, "us": grid.get(f"{q0},{a0}")},
            "best": {"q": int(best.split(",")[0]), "alpha": int(best.split(",")[1]),
                     "us": grid[best]},
            "speedup_vs_paper": round(grid[f"{q0},{a0}"] / grid[best], 3) if f"{q0},{a0}" in grid else None,
            "grid_us": grid}
        print(m, res["per_m"][str(m)]["paper"], res["per_m"][str(m)]["best"], flush=True)
    s = json.dumps(res, indent=1)
    if args.out:
        open(args.out, "w").write(s)
    else:
        print(s)


if __name__ == "__main__":
    main()
