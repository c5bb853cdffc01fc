#!/usr/bin/env python
"""Device time of hc_search with positions vs count-only (pos_out = NULL), per C2 m:
the difference is the cost of storing and ordering the positions."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2310_15711_b200 import hc  # noqa: E402
from paper_2310_15711_b200 import inputs as I  # noqa: E402

cfg = I.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
ms = [int(a) for a in sys.argv[2:]] or list(cfg.ms)
y_np, block = I.config_text(cfg)
y = torch.from_numpy(y_np).cuda()
n = len(y_np)
flush = torch.ones(2 * torch.cuda.get_device_properties(0).L2_cache_size, dtype=torch.uint8, device="cuda")
sp = int(torch.cuda.current_stream().cuda_stream)
pos = torch.empty(1 << 24, dtype=torch.int64, device="cuda")
st = hc.Stats()
for m in ms:
    q, a = cfg.qa[m]
    hs = [hc.prepare(x, q, a) for _, x in I.patterns(cfg, y_np, m, block=block)[:4]]
    t = {"pos": [], "count": []}
    for r in range(4):
        for h in hs:
            for mode in ("pos", "count"):
                flush.view(torch.int64).sum()
                c = hc.search_raw(h, y.data_ptr(), n, pos.data_ptr() if mode == "pos" else None,
                                  pos.numel() if mode == "pos" else 0, sp, hc.Opts(time_kernel=1), st)
                if r:
                    t[mode].append(st.kernel_ms * 1e3)
    print(f"m={m:5d} count={c:9d} with positions {statistics.median(t['pos']):9.2f} us  "
          f"count only {statistics.median(t['count']):9.2f} us  launches {st.launches}", flush=True)
