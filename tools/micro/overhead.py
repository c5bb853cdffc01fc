"""Event-timed cost of launching one (nearly) empty kernel, as the bench times hc_search:
L2-flush kernel first, then events around the launch.  Variants: grid, dynamic shared
memory, last-CTA ticket, mapped-host write."""
import ctypes as C
import os
import statistics
import torch

lib = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "liboverhead.so"))
lib.probe_host_alloc.restype = C.c_void_p
dev = C.c_void_p()
lib.probe_host_alloc(C.byref(dev))
ctr = torch.zeros(8, dtype=torch.int32, device="cuda")
flush = torch.ones(2 * torch.cuda.get_device_properties(0).L2_cache_size, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
sp = C.c_void_p(st.cuda_stream)


def timeit(fn, do_flush=True, reps=12):
    ts = []
    for r in range(reps + 2):
        if do_flush:
            flush.view(torch.int64).sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts), min(ts)


for do_flush in (True, False):
    for blocks, smem in ((1, 0), (444, 0), (444, 72 * 1024), (296, 82 * 1024), (592, 24 * 1024)):
        for mode in (0, 1, 2):
            med, mn = timeit(lambda: lib.probe_launch(blocks, smem, mode, C.c_void_p(ctr.data_ptr()), dev, sp), do_flush)
            print(f"flush={int(do_flush)} blocks={blocks:4d} smem={smem:6d} mode={mode} "
                  f"(0 empty, 1 +ticket, 2 +host write): median {med:.2f} us  min {mn:.2f} us", flush=True)
