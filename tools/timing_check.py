#!/usr/bin/env python
"""Does the mid event of time_kernel = 2 (between the search kernel and the PDL-launched
finish kernel) change the call's device time?  Alternates time_kernel 1 and 2 on the
same C2 patterns (L2 flushed before each call) and prints the medians per m.

    python tools/timing_check.py [--per-m 5] [--reps 4]
"""
import argparse
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
    ap.add_argument("--per-m", type=int, default=5)
    ap.add_argument("--reps", type=int, default=4)
    args = ap.parse_args()
    cfg = I.CONFIGS[args.config]
    y_np, _ = I.config_text(cfg)
    y = torch.from_numpy(y_np).cuda()
    n = len(y_np)
    flush = torch.ones(2 * torch.cuda.get_device_properties(0).L2_cache_size, dtype=torch.uint8,
                       device="cuda")
    sp = int(torch.cuda.current_stream().cuda_stream)
    pos = torch.empty(1 << 20, dtype=torch.int64, device="cuda")
    st = hc.Stats()
    for m in cfg.ms:
        q, a = cfg.qa[m]
        hs = [hc.prepare(x, q, a) for _, x in I.patterns(cfg, y_np, m)[:args.per_m]]
        t = {1: [], 2: []}
        s2 = []
        for r in range(args.reps + 1):
            for tk in (1, 2):
                for h in hs:
                    flush.view(torch.int64).sum()
                    hc.search_raw(h, y.data_ptr(), n, pos.data_ptr(), pos.numel(), sp,
                                  hc.Opts(time_kernel=tk), st)
                    if r:
                        t[tk].append(st.kernel_ms * 1e3)
                        if tk == 2:
                            s2.append(st.search_ms * 1e3)
        print(f"m={m:5d} tk1 {statistics.median(t[1]):8.2f} us  tk2 {statistics.median(t[2]):8.2f} us"
              f"  search kernel {statistics.median(s2):8.2f} us  path {st.path}", flush=True)


if __name__ == "__main__":
    main()
