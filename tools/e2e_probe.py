"""Wall-clock probe of the bench's e2e loop per m: prepare (single vs batch) +
search_batch + D2H, several repetitions in one process."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_15711_b200 import hc, inputs as I
cfg = I.CONFIGS["C2"]
y, block = I.config_text(cfg)
yd = torch.from_numpy(y).cuda()
sp = torch.cuda.current_stream().cuda_stream
cap = 1 << 16
pats = {m: I.patterns(cfg, y, m, block=block) for m in cfg.ms}
bufs = [torch.empty(cap, dtype=torch.int64, device="cuda") for _ in range(100)]
pin = torch.empty(cap, dtype=torch.int64).pin_memory()
for rep in range(4):
    for mode in ("single", "batch"):
        tp = tb = td = 0.0
        torch.cuda.synchronize()
        t00 = time.perf_counter()
        for m in cfg.ms:
            q, a = cfg.qa[m]
            t0 = time.perf_counter()
            hs = [hc.prepare(x, q, a) for o, x in pats[m]] if mode == "single" else \
                hc.prepare_batch([x for o, x in pats[m]], q, a)
            t1 = time.perf_counter()
            got = hc.search_batch_raw(hs, yd.data_ptr(), len(y), [b.data_ptr() for b in bufs], [cap] * len(hs), sp)
            t2 = time.perf_counter()
            for k, c in enumerate(got):
                pin[:c].copy_(bufs[k][:c], non_blocking=True)
            torch.cuda.synchronize()
            for h in hs: h.close()
            t3 = time.perf_counter()
            tp += t1 - t0; tb += t2 - t1; td += t3 - t2
        tot = time.perf_counter() - t00
        print(f"rep {rep} {mode}: total {1e3*tot:.1f} ms (prepare {1e3*tp:.1f}, batch call {1e3*tb:.1f}, d2h+close {1e3*td:.1f})", flush=True)
