#!/usr/bin/env python
"""Per-config, per-m single-call throughput (device time of hc_search: search kernel +
finish / ordering) on C2-C5, L2 flushed (read) before every call; patterns from the
config's seeded offsets.  Writes one JSON document (profiles/rNN_configs.json).

    python tools/config_bench.py --configs C3 C4 C5 --patterns 5 --reps 2 > out.json
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

NAMES = {1: "staged", 2: "gather", 3: "stream", 4: "shc"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["C2", "C3", "C4", "C5"])
    ap.add_argument("--patterns", type=int, default=5)
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    flush = torch.ones(2 * torch.cuda.get_device_properties(0).L2_cache_size, dtype=torch.uint8,
                       device="cuda")
    out = {"peak_gbs": peak, "patterns_per_m": args.patterns, "reps": args.reps,
           "timing": "device time per hc_search call (CUDA events recorded by the library: search "
                     "kernel + finish kernel + CUB ordering when count > 8192), median over "
                     "patterns x reps, L2 flushed before each call",
           "configs": {}}
    for key in args.configs:
        cfg = I.CONFIGS[key]
        y, block = I.config_text(cfg)
        yd = torch.from_numpy(y).cuda()
        n = len(y)
        res = {}
        for m in cfg.ms:
            q, a = cfg.qa[m]
            ts, counts, path = [], [], None
            for o, x in I.patterns(cfg, y, m, block=block)[:args.patterns]:
                h = hc.prepare(x, q, a)
                for r in range(args.reps + 1):
                    flush.view(torch.int64).sum()
                    torch.cuda.synchronize()
                    got, st = hc.search(h, yd, stats=True, time_kernel=1)
                    if r > 0:
                        ts.append(st["kernel_ms"])
                counts.append(int(got.numel()))
                path = NAMES[st["path"]]
            t = statistics.median(ts)
            gbps = n / (t / 1e3) / 1e9
            res[str(m)] = {"q": q, "alpha": a, "path": path, "device_us_median": round(t * 1e3, 2),
                           "GBps": round(gbps, 1), "pct_of_measured_hbm": round(100 * gbps / peak, 1),
                           "occ_per_pattern_mean": round(sum(counts) / len(counts), 1),
                           "occ_max": max(counts)}
            print(key, m, res[str(m)], file=sys.stderr, flush=True)
        out["configs"][cfg.name] = {"n": n, "per_m": res, "text_sha256": I.sha256(y)[:16]}
        del yd
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
