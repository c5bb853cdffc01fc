#!/usr/bin/env python
"""Per-pattern device time: single hc_search calls vs one hc_search_batch call.

    python tools/batch_bench.py --config C2 --patterns 20
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2310_15711_b200 import hc  # noqa: E402
from paper_2310_15711_b200 import inputs as I  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--patterns", type=int, default=20)
    ap.add_argument("--ms", type=int, nargs="+", default=None)
    args = ap.parse_args()
    cfg = I.CONFIGS[args.config]
    y_np, block = I.config_text(cfg)
    y = torch.from_numpy(y_np).cuda()
    n = len(y_np)
    flush = torch.ones(2 * torch.cuda.get_device_properties(0).L2_cache_size, dtype=torch.uint8,
                       device="cuda")
    sp = torch.cuda.current_stream().cuda_stream
    for m in (args.ms or cfg.ms):
        q, a = cfg.qa[m]
        hs = [hc.prepare(x, q, a) for _, x in I.patterns(cfg, y_np, m, count=args.patterns,
                                                           block=block)]
        cnt = [hc.count(h, y) for h in hs]
        cap = max(max(cnt), 1)
        pos = torch.empty(cap, dtype=torch.int64, device="cuda")
        o = hc.Opts(path=0, time_kernel=1)
        st = hc.Stats()
        single = 0.0
        for h in hs:
            flush.view(torch.int64).sum()
            hc.search_raw(h, y.data_ptr(), n, pos.data_ptr(), cap, sp, o, st)
            single += st.kernel_ms
        outs = [torch.empty(cap, dtype=torch.int64, device="cuda") for _ in hs]
        res = {}
        for nm in (0, 1):
            ob = hc.Opts(path=0, time_kernel=1, no_multi=nm)
            best = None
            for _ in range(3):
                flush.view(torch.int64).sum()
                got = hc.search_batch_raw(hs, y.data_ptr(), n, [t.data_ptr() for t in outs],
                                          [cap] * len(hs), sp, ob, st)
                assert got == cnt
                best = st.kernel_ms if best is None else min(best, st.kernel_ms)
            res[nm] = best / len(hs) * 1e3
        ps = single / len(hs) * 1e3
        print(f"m={m}: single {ps:.1f} us/pattern ({n / ps / 1e3:.0f} GB/s), batch multi "
              f"{res[0]:.1f} us/pattern ({n / res[0] / 1e3:.0f} GB/s), batch no-multi "
              f"{res[1]:.1f} us/pattern ({n / res[1] / 1e3:.0f} GB/s)", flush=True)


if __name__ == "__main__":
    main()
