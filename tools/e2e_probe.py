"""Wall-clock probe of the bench's e2e loop, per m (prepare + search_batch + D2H)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_15711_b200 import hc, inputs as I
cfg = I.CONFIGS["C2"]
y, block = I.config_text(cfg)
yd = torch.from_numpy(y).cuda()
sp = torch.cuda.current_stream().cuda_stream
cap = 1 << 16
for rep in range(3):
    for m in cfg.ms:
        q, a = cfg.qa[m]
        pats = I.patterns(cfg, y, m, block=block)
        bufs = [torch.empty(cap, dtype=torch.int64, device="cuda") for _ in pats]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hs = [hc.prepare(x, q, a) for o, x in pats]
        t1 = time.perf_counter()
        got = hc.search_batch_raw(hs, yd.data_ptr(), len(y), [b.data_ptr() for b in bufs], [cap] * len(hs), sp)
        t2 = time.perf_counter()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        for h in hs: h.close()
        print(f"rep {rep} m={m}: prepare {1e3*(t1-t0):.2f} ms, batch {1e3*(t2-t1):.2f} ms, sync {1e3*(t3-t2):.2f} ms, counts {sum(got)}", flush=True)
