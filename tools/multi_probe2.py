"""Multi-pattern group configurations (chunk bytes, buffers, warps) for P=4 on C2."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_15711_b200 import hc, inputs as I
cfg = I.CONFIGS["C2"]
y_np, block = I.config_text(cfg)
y = torch.from_numpy(y_np).cuda(); n = len(y_np)
flush = torch.ones(2 * torch.cuda.get_device_properties(0).L2_cache_size, dtype=torch.uint8, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
P = int(sys.argv[1]) if len(sys.argv) > 1 else 4
for tile, stages, bw in [(2048, 2, 16), (2560, 2, 16), (2048, 2, 12), (3072, 2, 12), (1536, 3, 16), (1536, 2, 16), (1024, 3, 16)]:
    line = []
    for m in [8, 16, 32]:
        q, a = cfg.qa[m]
        hs = [hc.prepare(x, q, a) for _, x in I.patterns(cfg, y_np, m, count=P, block=block)]
        outs = [torch.empty(1 << 16, dtype=torch.int64, device="cuda") for _ in hs]
        st = hc.Stats()
        ob = hc.Opts(path=0, time_kernel=1, tile_bytes=tile, stages=stages, block_warps=bw)
        ts = []
        for _ in range(4):
            flush.view(torch.int64).sum(); torch.cuda.synchronize()
            hc.search_batch_raw(hs, y.data_ptr(), n, [t.data_ptr() for t in outs], [1 << 16] * P, sp, ob, st)
            ts.append(st.kernel_ms)
        line.append(f"m={m} {min(ts[1:]) * 1e3 / P:.1f}")
    print(f"P={P} tile={tile} bufs={stages} warps={bw}: " + ", ".join(line) + " us/pattern", flush=True)
