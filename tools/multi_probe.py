"""One multi-pattern group (P patterns, one launch) vs the same patterns as separate
searches overlapped on the batch streams; per-pattern device time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_15711_b200 import hc, inputs as I
cfg = I.CONFIGS["C2"]
y_np, block = I.config_text(cfg)
y = torch.from_numpy(y_np).cuda(); n = len(y_np)
flush = torch.ones(2 * torch.cuda.get_device_properties(0).L2_cache_size, dtype=torch.uint8, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
for m in [8, 16, 32]:
    q, a = cfg.qa[m]
    for P in [1, 2, 4]:
        hs = [hc.prepare(x, q, a) for _, x in I.patterns(cfg, y_np, m, count=P, block=block)]
        outs = [torch.empty(1 << 16, dtype=torch.int64, device="cuda") for _ in hs]
        st = hc.Stats()
        res = {}
        for nm in (0, 1):
            ob = hc.Opts(path=0, time_kernel=1, no_multi=nm)
            ts = []
            for _ in range(4):
                flush.view(torch.int64).sum(); torch.cuda.synchronize()
                hc.search_batch_raw(hs, y.data_ptr(), n, [t.data_ptr() for t in outs], [1 << 16] * P, sp, ob, st)
                ts.append(st.kernel_ms)
            res[nm] = min(ts[1:]) * 1e3 / P
        print(f"m={m} P={P}: multi {res[0]:.1f} us/pattern, separate {res[1]:.1f} us/pattern", flush=True)
