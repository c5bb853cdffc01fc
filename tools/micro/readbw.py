"""Read-only bandwidth probes on a 256 MiB buffer (L2 flushed before each): LDG.128 and
per-warp TMA bulk copies, several grid sizes / chunk sizes.  Prints GB/s per variant."""
import ctypes as C
import os
import statistics
import torch

lib = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libreadbw.so"))
n = 256 << 20
y = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
out = torch.zeros(4, dtype=torch.int32, device="cuda")
flush = torch.ones(2 * torch.cuda.get_device_properties(0).L2_cache_size, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
sp = C.c_void_p(st.cuda_stream)


def timeit(fn, reps=8):
    ts = []
    for r in range(reps + 1):
        flush.view(torch.int64).sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


for blocks in (148 * 4, 148 * 8, 148 * 16, 148 * 32):
    t = timeit(lambda: lib.probe_read_ldg(C.c_void_p(y.data_ptr()), C.c_size_t(n), C.c_void_p(out.data_ptr()), blocks, sp))
    print(f"ldg128 blocks={blocks}: {t*1e3:.1f} us  {n / t / 1e6:.0f} GB/s", flush=True)
for blocks, chunk in ((148 * 2, 4096), (148 * 3, 4096), (148 * 2, 8192), (148 * 1, 12288), (148 * 4, 2048), (148 * 6, 2048)):
    t = timeit(lambda: lib.probe_read_bulk(C.c_void_p(y.data_ptr()), C.c_size_t(n), C.c_void_p(out.data_ptr()), blocks, chunk, sp))
    print(f"bulk blocks={blocks} chunk={chunk}: {t*1e3:.1f} us  {n / t / 1e6:.0f} GB/s", flush=True)
t = timeit(lambda: y.view(torch.int64).sum())
print(f"torch int64 sum: {t*1e3:.1f} us  {n / t / 1e6:.0f} GB/s")
