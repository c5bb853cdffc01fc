#!/usr/bin/env python
"""Interleaved A/B of two builds of libhc on the same patterns, in one process: calls
alternate A, B, A, B ... (L2 flushed before each), so clock and box drift hit both.

    python tools/ab.py LIB_A LIB_B [--config C2] [--m 8 16 32] [--per-m 4] [--reps 5]
"""
import argparse
import ctypes as C
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2310_15711_b200 import hc  # noqa: E402  (structs only)
from paper_2310_15711_b200 import inputs as I  # noqa: E402


def load(path):
    lib = C.CDLL(path)
    lib.hc_prepare.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int]
    lib.hc_prepare.restype = C.c_void_p
    lib.hc_search_ex.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t,
                                 C.c_void_p, C.POINTER(hc.Opts), C.POINTER(hc.Stats)]
    lib.hc_search_ex.restype = C.c_int64
    return lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs=2)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--m", type=int, nargs="+", default=None)
    ap.add_argument("--per-m", type=int, default=4)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--count-only", action="store_true")
    ap.add_argument("--b-spl", type=int, default=0, help="opts.seg_per_lane for library B")
    args = ap.parse_args()
    libs = [load(os.path.abspath(p)) for p in args.libs]
    cfg = I.CONFIGS[args.config]
    y_np, block = I.config_text(cfg)
    y = torch.from_numpy(y_np).cuda()
    n = len(y_np)
    flush = torch.ones(2 * torch.cuda.get_device_properties(0).L2_cache_size, dtype=torch.uint8,
                       device="cuda")
    pos = torch.empty(1 << 24, dtype=torch.int64, device="cuda")
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    st = hc.Stats()
    opts = hc.Opts(time_kernel=1)
    opts_b = hc.Opts(time_kernel=1, seg_per_lane=args.b_spl)
    tot = [0.0, 0.0]
    for m in args.m or cfg.ms:
        q, a = cfg.qa[m]
        xs = [x for _, x in I.patterns(cfg, y_np, m, block=block)[:args.per_m]]
        hs = [[lib.hc_prepare(x.ctypes.data, len(x), q, a) for x in xs] for lib in libs]
        t = [[], []]
        cnt = [None, None]
        for r in range(args.reps + 1):
            for i in range(len(xs)):
                for k in (0, 1):
                    flush.view(torch.int64).sum()
                    c = libs[k].hc_search_ex(hs[k][i], C.c_void_p(y.data_ptr()), n,
                                             None if args.count_only else C.c_void_p(pos.data_ptr()),
                                             0 if args.count_only else pos.numel(), sp,
                                             C.byref(opts_b if k else opts), C.byref(st))
                    assert c >= 0
                    if cnt[k] is None:
                        cnt[k] = c
                    if r:
                        t[k].append(st.kernel_ms * 1e3)
        ma, mb = statistics.median(t[0]), statistics.median(t[1])
        tot[0] += ma
        tot[1] += mb
        print(f"m={m:5d}  A {ma:8.2f} us  B {mb:8.2f} us  B/A {mb / ma:6.3f}", flush=True)
    print(f"sum   A {tot[0]:8.2f} us  B {tot[1]:8.2f} us  B/A {tot[1] / tot[0]:6.3f}")


if __name__ == "__main__":
    main()
