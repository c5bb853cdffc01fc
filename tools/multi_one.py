"""One multi-pattern launch (C2, given m and P) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_15711_b200 import hc, inputs as I
m, P = int(sys.argv[1]), int(sys.argv[2])
cfg = I.CONFIGS["C2"]
y_np, block = I.config_text(cfg)
y = torch.from_numpy(y_np).cuda(); n = len(y_np)
sp = torch.cuda.current_stream().cuda_stream
q, a = cfg.qa[m]
hs = [hc.prepare(x, q, a) for _, x in I.patterns(cfg, y_np, m, count=P, block=block)]
outs = [torch.empty(1 << 16, dtype=torch.int64, device="cuda") for _ in hs]
st = hc.Stats()
for r in range(2):
    c = hc.search_batch_raw(hs, y.data_ptr(), n, [t.data_ptr() for t in outs], [1 << 16] * P, sp, hc.Opts(time_kernel=1), st)
    print(c, st.kernel_ms)
