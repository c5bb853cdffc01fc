#!/usr/bin/env python
"""Small searches on every kernel of libhc, for compute-sanitizer (memcheck, racecheck,
synccheck) and for the fault-injection check.  Each case is compared with brute force
(oracle O1); the script exits 1 on any mismatch.

    compute-sanitizer --tool memcheck python tools/sanitize_case.py
    HC_LIB=paper_2310_15711_b200/libhc_instr.so python tools/sanitize_case.py --inject

Texts are 16-byte multiples at 256-aligned cudaMalloc addresses (run with
PYTORCH_NO_CUDA_MEMORY_CACHING=1 so that every tensor is its own exact-size
allocation): the kernels' aligned 8/16-byte word reads then stay inside the text
(hc_device.cuh, end8).  --inject sets the instrumented build's fault hook (debug =
9: the finish kernel shifts the first ordered position by one) and expects the
comparison to FAIL.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2310_15711_b200 import hc  # noqa: E402
from paper_2310_15711_b200 import inputs as I  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--inject", action="store_true", help="fault hook on (instrumented build)")
    ap.add_argument("--small", action="store_true", help="fewer cases (racecheck is slow)")
    ap.add_argument("--unaligned", action="store_true",
                    help="also texts at odd offsets / odd lengths and small chunks (edge chunks): "
                         "with the instrumented build every text access is bounds-checked "
                         "against [y, y + n) and traps outside it")
    args = ap.parse_args()
    dbg = 9 if args.inject else 0
    rng = np.random.default_rng(91)
    n = 1 << 17 if args.small else 1 << 19
    y = I.gen_text("dna", n, 91)
    cases = []
    for m, q, a in [(8, 4, 12), (16, 6, 12), (33, 3, 11), (200, 6, 12), (3, 2, 8), (1100, 8, 15)]:
        o = int(rng.integers(0, n - m))
        x = y[o:o + m].copy()
        yy = y.copy()
        for p in rng.integers(0, n - m, 9):
            yy[p:p + m] = x
        cases.append((x, q, a, yy))
    # many occurrences: the finish kernel's bucket and radix branches and the large ordering
    ya = np.full(n, ord("A"), np.uint8)
    cases.append((np.frombuffer(b"AAAA", np.uint8).copy(), 2, 10, ya))
    bad = 0
    paths = [hc.PATH_STREAM, hc.PATH_GATHER, hc.PATH_STAGED, hc.PATH_SHC, hc.PATH_SCAN]
    for x, q, a, yy in cases:
        want = oracle.brute(x, yy)
        yd = torch.from_numpy(yy).cuda()
        h = hc.prepare(x, q, a)
        for path in paths:
            try:
                got = hc.search(h, yd, path=path, debug=dbg).cpu().numpy()
            except hc.HCError as e:
                if e.code == hc.HC_EINVAL and path in (hc.PATH_SHC, hc.PATH_STAGED, hc.PATH_SCAN):
                    continue
                raise
            if not np.array_equal(got, want):
                bad += 1
                print(f"MISMATCH m={len(x)} path={path}: {len(got)} vs {len(want)}", flush=True)
    if args.unaligned:
        big = torch.zeros(n + 64, dtype=torch.uint8, device="cuda")
        for x, q, a, yy in cases[:5]:
            for off, cut in ((1, 0), (13, 5), (16, 11)):
                yv = yy[:len(yy) - cut]
                want = oracle.brute(x, yv)
                big[off:off + len(yv)] = torch.from_numpy(yv).cuda()
                yd = big[off:off + len(yv)]
                h = hc.prepare(x, q, a)
                for path, kw in ((hc.PATH_AUTO, {}), (hc.PATH_STREAM, {"tile_bytes": 700, "max_ctas": 3}),
                                 (hc.PATH_STREAM, {"seg_per_lane": -1, "block_warps": 3}),
                                 (hc.PATH_GATHER, {"max_ctas": 2}), (hc.PATH_SCAN, {}), (hc.PATH_SHC, {}),
                                 (hc.PATH_STAGED, {})):
                    try:
                        got = hc.search(h, yd, path=path, **kw).cpu().numpy()
                    except hc.HCError as e:
                        if e.code == hc.HC_EINVAL and path in (hc.PATH_SHC, hc.PATH_STAGED, hc.PATH_SCAN, hc.PATH_STREAM):
                            continue
                        raise
                    if not np.array_equal(got, want):
                        bad += 1
                        print(f"MISMATCH unaligned m={len(x)} off={off} cut={cut} path={path}", flush=True)
    # multi-pattern launches (hc_search_batch)
    xs = [y[o:o + 16].copy() for o in rng.integers(0, n - 16, 4)]
    hb = [hc.prepare(x, 6, 12) for x in xs]
    got = hc.search_batch(hb, torch.from_numpy(y).cuda(), debug=dbg)
    for x, g in zip(xs, got):
        if not np.array_equal(g.cpu().numpy(), oracle.brute(x, y)):
            bad += 1
            print("MISMATCH batch", flush=True)
    torch.cuda.synchronize()
    print(f"sanitize_case: {bad} mismatches", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
