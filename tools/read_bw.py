"""Read-only HBM bandwidth reference: torch reductions over a 256 MiB buffer (L2 flushed)."""
import torch
n = 256 << 20
y = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
flush = torch.ones(2 * torch.cuda.get_device_properties(0).L2_cache_size, dtype=torch.uint8, device="cuda")
for name, f in [("sum_i32", lambda: y.view(torch.int32).sum()), ("sum_i64", lambda: y.view(torch.int64).sum()),
                ("max_u8", lambda: y.max())]:
    ts = []
    for r in range(6):
        flush.view(torch.int64).sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    t = sorted(ts[1:])[len(ts[1:]) // 2]
    print(f"{name}: {t:.1f} us  {n / t / 1e3:.0f} GB/s")
