import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2310_15711_b200 import hc
rng = np.random.default_rng(1)
y = rng.integers(0, 4, 5000, dtype=np.uint8)
yd = torch.from_numpy(y).cuda()
for alpha in (13, 14, 15):
    for m, q in ((1, 1), (5, 2)):
        x = y[100:100 + m].copy()
        h = hc.prepare(x, q, alpha)
        try:
            res, st = hc.search(h, yd, stats=True, path=hc.PATH_STREAM)
            torch.cuda.synchronize()
            print(alpha, m, q, len(res), st["grid"], st["block"], st["smem_bytes"])
        except Exception as e:
            print(alpha, m, q, "ERR", e)
