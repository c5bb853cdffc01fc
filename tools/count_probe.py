"""Search with positions vs count only (device time), high-occurrence cases."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_15711_b200 import hc, inputs as I
for key, m in [("C5", 32), ("C4", 2), ("C2", 8)]:
    cfg = I.CONFIGS[key]
    y, block = I.config_text(cfg)
    yd = torch.from_numpy(y).cuda(); n = len(y)
    q, a = cfg.qa[m]
    o, x = I.patterns(cfg, y, m, block=block)[0]
    h = hc.prepare(x, q, a)
    sp = torch.cuda.current_stream().cuda_stream
    c = hc.count(h, yd)
    pos = torch.empty(max(c, 1), dtype=torch.int64, device="cuda")
    st = hc.Stats()
    for mode in ("positions", "count"):
        ts = []
        for r in range(3):
            if mode == "positions":
                hc.search_raw(h, yd.data_ptr(), n, pos.data_ptr(), c, sp, hc.Opts(time_kernel=1), st)
            else:
                hc.search_raw(h, yd.data_ptr(), n, None, 0, sp, hc.Opts(time_kernel=1), st)
            ts.append(st.kernel_ms * 1e3)
        print(f"{key} m={m} count={c} {mode}: {min(ts):.1f} us (launches {st.launches})", flush=True)
    del yd
    torch.cuda.empty_cache()
