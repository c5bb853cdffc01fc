#!/usr/bin/env python
"""Run a few hc_search calls of one config / m (for ncu captures and quick timing).

    python tools/profile_search.py --config C2 --m 16 32 1024 --reps 3 [--path 0|1|2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

if any(a.startswith("--debug") for a in sys.argv) or "--trace" in sys.argv:
    # measurement-only modes exist in the instrumented build only (HC_INSTRUMENT=1)
    from paper_2310_15711_b200 import build as _b
    os.environ["HC_LIB"] = _b.build(instrument=True)
from paper_2310_15711_b200 import hc  # noqa: E402
from paper_2310_15711_b200 import inputs as I  # noqa: E402


def analyze_trace(tr, grid, T, stages):
    import numpy as np
    a = tr[:grid * T * 4].view(grid, T, 4).cpu().numpy().astype(np.float64)
    ce0 = tr[grid * T * 4: grid * T * 4 + 2 * grid].view(grid, 2).cpu().numpy().astype(np.float64)
    t0 = a[a > 0].min() if (a > 0).any() else ce0[ce0 > 0].min()
    a = np.where(a > 0, a - t0, np.nan) / 1e3   # us since first event
    fs, fe, se, ss = a[..., 0], a[..., 1], a[..., 2], a[..., 3]
    med = lambda v: float(np.nanmedian(v)) if np.isfinite(v).any() else float("nan")
    print(f"  trace (median, us): first data {med(fs[:, 0]):.2f}; filter {med(fe - fs):.2f}; "
          f"filter end -> surv start {med(ss - fe):.2f}; surv {med(se - ss):.2f}; "
          f"surv end -> refilled data {med(fs[:, stages:] - se[:, :-stages]):.2f}; "
          f"tile period {med(fs[:, 1:] - fs[:, :-1]):.2f}")
    ce = tr[grid * T * 4: grid * T * 4 + 2 * grid].view(grid, 2).cpu().numpy().astype(np.float64)
    ce = (ce - t0) / 1e3
    print(f"  CTA entry min {ce[:, 0].min():.2f} p50 {np.median(ce[:, 0]):.2f} max {ce[:, 0].max():.2f}; "
          f"exit p50 {np.median(ce[:, 1]):.2f} max {ce[:, 1].max():.2f} (us vs first tile event)")
    fz = tr[grid * T * 4 + 2 * grid: grid * T * 4 + 2 * grid + 2].cpu().numpy().astype(np.float64)
    fz = (fz - t0) / 1e3
    print(f"  finish kernel: start {fz[0]:.2f}, after griddepcontrol.wait {fz[1]:.2f}; "
          f"grid span (first entry -> finish wait) {fz[1] - ce[:, 0].min():.2f} us")
    last = np.nanmax(np.where(np.isfinite(fe), fe, np.nan), axis=1)   # per CTA, last traced filter end
    print(f"  span: first event 0, CTA last-traced-filter-end p50 {np.nanpercentile(last, 50):.2f} "
          f"p90 {np.nanpercentile(last, 90):.2f} max {np.nanmax(last):.2f} us; "
          f"CTA first data p50 {np.nanpercentile(fs[:, 0], 50):.2f} max {np.nanmax(fs[:, 0]):.2f}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--m", type=int, nargs="+", default=[16])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--path", type=int, default=0)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--spl", type=int, default=0)
    ap.add_argument("--cps", type=int, default=0)
    ap.add_argument("--debug", type=int, default=0)
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--absent", action="store_true", help="random pattern (likely absent)")
    ap.add_argument("--trace", type=int, default=0, help="trace N tiles per CTA (staged)")
    ap.add_argument("--sw", type=int, default=0, help="survivor warps (staged)")
    ap.add_argument("--bw", type=int, default=0, help="warps per CTA (stream)")
    ap.add_argument("--noflush", action="store_true", help="no L2 flush between calls")
    args = ap.parse_args()
    cfg = I.CONFIGS[args.config]
    y, block = I.config_text(cfg, args.n)
    yd = torch.from_numpy(y).cuda()
    flush = torch.ones(2 * torch.cuda.get_device_properties(0).L2_cache_size, dtype=torch.uint8,
                       device="cuda")
    torch.cuda.synchronize()

    def flush_l2():
        # read-only flush: evicts the text with CLEAN lines (a write flush would leave
        # dirty lines whose write-back then competes with the timed search)
        flush.view(torch.int64).sum()
    for m in args.m:
        q, a = cfg.qa[m] if m in cfg.qa else cfg.qa[min(cfg.qa, key=lambda k: abs(k - m))]
        o, x = I.patterns(cfg, y, m, count=1, block=block)[0]
        if args.absent:
            import numpy as np
            x = np.random.default_rng(m).permutation(x)
        h = hc.prepare(x, q, a)
        tr = torch.zeros(2048 * max(args.trace, 1) * 4 + 4096 + 2048 * 32, dtype=torch.int64, device="cuda")
        for r in range(args.reps):
            if not args.noflush:
                flush_l2()
            tr.zero_()
            res, st = hc.search(h, yd, stats=True, path=args.path, tile_bytes=args.tile,
                                stages=args.stages, seg_per_lane=args.spl, time_kernel=1,
                                ctas_per_sm=args.cps, debug=args.debug,
                                tma_chunk=args.chunk, trace=tr.data_ptr() if args.trace else 0,
                                trace_tiles=args.trace, surv_warps=args.sw, block_warps=args.bw)
            torch.cuda.synchronize()
            print(f"m={m} q={q} a={a} rep={r} count={len(res)} kernel_us={st['kernel_ms']*1e3:.1f} "
                  f"GBps={len(y)/(st['kernel_ms']/1e3)/1e9:.0f} grid={st['grid']} smem={st['smem_bytes']}"
                  + (f" phaseB iters={st['dbg'][0]} calls={st['dbg'][1]}" if args.debug == 5 else "")
                  + (f" epilogue ordering {st['dbg'][0] / 1e3:.2f} us for {st['dbg'][1]} positions"
                     if args.debug == 10 else ""),
                  flush=True)
            if args.trace and args.debug == 12:
                # latest passage of each critical-path point over all warps, us after the
                # earliest CTA entry
                g, T = st["grid"], args.trace
                ts = tr[g * (T * 4 + 2) + 8: g * (T * 4 + 2) + 8 + 16].cpu().numpy().astype("uint64")
                cn = tr[g * (T * 4 + 2) + 24: g * (T * 4 + 2) + 24 + 4].cpu().numpy()
                print(f"  phase B: iterations {cn[0]}, warp-wide walks {cn[1]}, warp-wide verifications {cn[2]}")
                t0 = int(~ts[0])
                names = ["entry", "table", "-", "loop done", "q1 drained", "phase B done", "flushed",
                         "ticket", "published"] + [f"B it{k}" for k in range(7)]
                print("  path (us after first CTA entry): " + ", ".join(
                    f"{nm} {(int(t) - t0) / 1e3:.2f}" for nm, t in zip(names[1:], ts[1:]) if int(t)))
            elif args.trace and r == args.reps - 1 and st["path"] == 2:
                # gather: per-warp events (trace_tiles >= 8): table loaded, filtered, drained, flushed
                import numpy as np
                g, T = st["grid"], args.trace
                a = tr[:g * T * 4].view(g, T, 4)[:, :8, :].cpu().numpy().astype(np.float64)
                ce = tr[g * T * 4: g * T * 4 + 2 * g].view(g, 2).cpu().numpy().astype(np.float64)
                t0 = ce[:, 0].min()
                rel = lambda v: (v - t0) / 1e3
                for k_, nm in enumerate(["table loaded", "filtered", "drained", "flushed"]):
                    r_ = rel(a[:, :, k_]).ravel()
                    print(f"  gather warps {nm}: p10 {np.percentile(r_, 10):.2f} p50 {np.median(r_):.2f} "
                          f"p90 {np.percentile(r_, 90):.2f} p99 {np.percentile(r_, 99):.2f} max {r_.max():.2f} us")
                d = rel(a[:, :, 2]) - rel(a[:, :, 1])
                print(f"  drain time per warp: p50 {np.median(d):.2f} p99 {np.percentile(d, 99):.2f} max {d.max():.2f}")
                r_ = rel(ce[:, 1])
                print(f"  CTA exit: p50 {np.median(r_):.2f} p90 {np.percentile(r_, 90):.2f} max {r_.max():.2f} us")
                worst = np.unravel_index(np.argmax(a[:, :, 3]), a[:, :, 3].shape)
                print(f"  slowest warp (cta {worst[0]}, warp {worst[1]}):", np.round(rel(a[worst[0], worst[1]]), 2))
            elif args.trace and r == args.reps - 1:
                analyze_trace(tr, st["grid"], args.trace, args.stages or 3)
                if args.debug == 11:
                    import numpy as np
                    g = st["grid"]
                    b0 = g * args.trace * 4 + 2 * g
                    pr = tr[b0:b0 + g * 8 * 4].view(g, 8, 4).cpu().numpy().astype(np.float64) / 1965.0
                    print("  per-warp us (wait, filter, tail, release): mean",
                          np.round(pr.mean(axis=(0, 1)), 2), "max-over-warps mean",
                          np.round(pr.max(axis=1).mean(axis=0), 2))


if __name__ == "__main__":
    main()
