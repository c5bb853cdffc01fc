#!/usr/bin/env python
"""Benchmark of the B200 Hash Chain search (BASELINE.json metric: text GB/s
searched per pattern vs m on 1 B200, % of HBM peak; bit-exact).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl hc|reference]

Workload (N=1): BASELINE.json configs[1] = C2, DNA-like i.i.d. text of 256 MiB,
m in {8,...,1024}, 100 patterns per m copied from seeded text offsets, (q, alpha)
per m from the paper's Table 1 (inputs.py).  One STEP searches every (m, pattern)
of the config once (the whole hot path: search kernel, count read-back, ordering of
the positions into the caller's int64 buffer), i.e. 800 searches of 256 MiB, twice:
as one hc_search_batch call per m (the 100 searches overlap on library streams;
`value`) and as 800 single hc_search calls (per_m single numbers, roofline).  L2 is
flushed (2 x L2 bytes read) before every single search and every batch call,
outside the timed intervals; the device time comes from CUDA events the library
records on the caller's stream.  value = bytes searched / summed device time.

Under torchrun (N>1), --mode replicas (default): every rank searches the same text
with its own seeded patterns (weak scaling; no data-path collective);
value = bytes searched by all ranks / max over ranks of the search time.
--mode shard: the ranks search every pattern together, each over its share of the
window ends (an (m-1)-byte halo on the left), and all-gather counts and positions
over NCCL (paper_2310_15711_b200/shard.py; strong scaling); a search's
time is its kernel time plus the exchange, value = n x searches / max over ranks.

--impl reference times the oracle (oracle/, plain C HC of Fig. 5 run over the
host cores) on a bounded sample of the same workload: the base contract's
reference arm for this tier.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
PATH_NAMES = {1: "staged", 2: "gather", 3: "stream", 4: "shc"}
sys.path.insert(0, ROOT)

from paper_2310_15711_b200 import inputs as I  # noqa: E402

METRIC = "text GB/s searched per pattern vs m (1 B200), % of HBM peak; bit-exact"
# fraction of 32-B sectors HC touches, SURVEY.md 8(d) (simulated, DNA/protein/NL within 15%)
F32 = {8: 1.0, 16: 1.0, 32: 1.0, 64: 0.63, 128: 0.29, 256: 0.145, 512: 0.075, 1024: 0.039,
       2048: 0.019, 4096: 0.011, 2: 1.0, 4: 1.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def __exit__(self, *a):
        self.samples = []
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                self.samples.append(f)

    def summary(self):
        if not getattr(self, "samples", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if s[5 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def gen_workload(cfg, rank: int, per_m: int | None):
    y, block = I.config_text(cfg)
    work = []
    for m in cfg.ms:
        q, a = cfg.qa[m]
        pats = I.patterns(cfg, y, m, count=per_m, salt=rank, block=block)
        for o, x in pats:
            work.append((m, q, a, o, x))
    return y, work


def reference_arm(args, cfg, ws, rank):
    """Oracle (O2, Fig. 5 HC in plain C) over the host cores on a bounded sample."""
    if rank != 0:
        return
    import oracle
    y, work = gen_workload(cfg, 0, args.per_m)
    T = os.cpu_count() or 1
    budget = args.ref_seconds
    by_m = {}
    for item in work:
        by_m.setdefault(item[0], []).append(item)
    sample = [lst[k] for k in range(max(len(v) for v in by_m.values())) for lst in by_m.values()
              if k < len(lst)]
    # warm-up: one search
    oracle.hc_threaded(sample[0][4], y, sample[0][1], sample[0][2], threads=T)
    step_vals = []
    done_total = 0
    t_total = 0.0
    per_step = max(1, budget / max(1, args.steps))
    idx = 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        nb = 0
        while True:
            m, q, a, o, x = sample[idx % len(sample)]
            idx += 1
            oracle.hc_threaded(x, y, q, a, threads=T)
            nb += len(y)
            if time.perf_counter() - t0 > per_step:
                break
        dt = time.perf_counter() - t0
        step_vals.append(nb / dt / 1e9)
        done_total += nb
        t_total += dt
    v = done_total / t_total / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "GB/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1000 * t_total / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": cfg.name, "n": cfg.n, "ms": list(cfg.ms),
                       "patterns_per_m": cfg.patterns_per_m if args.per_m is None else args.per_m},
            "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": T, "kind": "oracle",
                             "sample": f"{idx} searches of {len(y)} B (patterns round-robin over m), "
                                       f"O2 HC (oracle/hc_oracle.c) split over {T} threads by "
                                       "window-end ranges"},
            "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, y, work, seconds: float):
    import oracle
    T = os.cpu_count() or 1
    by_m = {}
    for item in work:
        by_m.setdefault(item[0], []).append(item)
    order = [lst[k] for k in range(max(len(v) for v in by_m.values())) for lst in by_m.values()
             if k < len(lst)]
    t0 = time.perf_counter()
    nb = 0
    cnt = 0
    while time.perf_counter() - t0 < seconds and cnt < len(order):
        m, q, a, o, x = order[cnt]
        oracle.hc_threaded(x, y, q, a, threads=T)
        nb += len(y)
        cnt += 1
    dt = time.perf_counter() - t0
    return {"value": round(nb / dt / 1e9, 3), "unit": "GB/s", "cores": T, "kind": "oracle",
            "sample": f"{cnt} searches of {len(y)} B (one pattern per m in turn, from the first), "
                      f"O2 HC (oracle/hc_oracle.c) over {T} threads by window-end ranges"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="hc", choices=["hc", "reference"])
    ap.add_argument("--per-m", type=int, default=None, help="patterns per m (default: config's)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=60.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--out", default=None, help="also append the JSON line to this file")
    ap.add_argument("--mode", default="replicas", choices=["replicas", "shard"])
    ap.add_argument("--api", default="batch", choices=["batch", "single"],
                    help="value from one hc_search_batch call per m (default) or from single "
                         "hc_search calls; both are always measured and reported per m")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    ws, rank, local = dist_init()
    cfg = I.CONFIGS[args.config]
    if args.impl == "reference":
        reference_arm(args, cfg, ws, rank)
        return

    import torch
    from paper_2310_15711_b200 import hc

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    sp = int(stream.cuda_stream)
    shard_mode = args.mode == "shard"
    # replicas: per-rank patterns (salt = rank); shard: every rank takes part in every search
    y_np, work = gen_workload(cfg, 0 if shard_mode else rank, args.per_m)
    n = len(y_np)
    y = torch.from_numpy(y_np).to(dev)
    handles = [hc.prepare(x, q, a) for (m, q, a, o, x) in work]
    # Preprocessing time per pattern (host Fig. 3 + upload; the paper times it with every
    # search): hc_prepare alone, and amortised by hc_prepare_batch, per m
    prep_us = {}
    for m_ in cfg.ms:
        xs_ = [x for (mm, q, a, o, x) in work if mm == m_]
        qa_ = next((q, a) for (mm, q, a, o, x) in work if mm == m_)
        t0 = time.perf_counter()
        hs_ = [hc.prepare(x, *qa_) for x in xs_]
        t1 = time.perf_counter()
        hb_ = hc.prepare_batch(xs_, *qa_)
        t2 = time.perf_counter()
        for h_ in hs_ + hb_:
            h_.close()
        prep_us[m_] = (1e6 * (t1 - t0) / len(xs_), 1e6 * (t2 - t1) / len(xs_))
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush_buf = torch.ones(2 * l2, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize(dev)

    def flush_l2():
        # read-only L2 flush: reading 2 x L2 bytes evicts the text with CLEAN lines (a
        # write flush leaves dirty lines whose write-back competes with the timed search)
        flush_buf.view(torch.int64).sum()

    # exact per-pattern counts (warm-up also sizes the position buffer)
    counts = [hc.search_raw(h, y.data_ptr(), n, None, 0, sp) for h in handles]
    cap = max(1, max(counts))
    pos = torch.empty(cap, dtype=torch.int64, device=dev)
    opts = hc.Opts(path=0, time_kernel=1)
    st = hc.Stats()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in work]
    if shard_mode:
        from paper_2310_15711_b200.shard import shard_bounds
        shards = {m: shard_bounds(n, m, ws, rank) for m in cfg.ms}
        xev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in work]
        cnt_t = torch.zeros(1, dtype=torch.int64, device=dev)
        pad = torch.full((cap,), -1, dtype=torch.int64, device=dev)
        g_cnt = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(ws)]
        g_pos = [torch.empty(cap, dtype=torch.int64, device=dev) for _ in range(ws)]

    def step(timed: bool):
        per = []
        launches = 0
        for k, h in enumerate(handles):
            flush_l2()
            e0, e1 = ev[k]
            e0.record(stream)
            if shard_mode:
                sh = shards[work[k][0]]
                c = hc.search_raw(h, y.data_ptr() + sh.text_lo, sh.size, pos.data_ptr(), cap, sp,
                                  opts, st) if sh.size >= work[k][0] else 0
                x0, x1 = xev[k]
                x0.record(stream)
                # exchange: counts, then the positions padded to cap
                torch.add(pos[:c], sh.text_lo, out=pad[:c])   # global positions
                if dist:
                    cnt_t.fill_(c)
                    dist.all_gather(g_cnt, cnt_t)
                    dist.all_gather(g_pos, pad)
                x1.record(stream)
            else:
                c = hc.search_raw(h, y.data_ptr(), n, pos.data_ptr(), cap, sp, opts, st)
                assert c == counts[k]
            e1.record(stream)
            launches += st.launches
            per.append((st.kernel_ms, st.path))
            if shard_mode and not timed:
                total = int(sum(t.item() for t in g_cnt)) if dist else c
                assert total == counts[k], (k, total, counts[k])
        torch.cuda.synchronize(dev)
        calls = [e0.elapsed_time(e1) for (e0, e1) in ev]
        # value uses the library's device time of each call's work (search launch to the
        # end of its last kernel, CUDA events on the launching stream); the event pair
        # around the Python call (host API overhead included) is reported as call time
        times = [kms for (kms, _) in per]
        if shard_mode:
            times = [t + x0.elapsed_time(x1) for t, (x0, x1) in zip(times, xev)]
        return times, per, launches, calls

    # hc_search_batch per m (all of its patterns in one call; replicas mode only)
    use_batch = not shard_mode
    by_m = {}
    for k, (m, q, a, o, x) in enumerate(work):
        by_m.setdefault(m, []).append(k)
    if use_batch:
        bufs = [torch.empty(cap, dtype=torch.int64, device=dev) for _ in work]
        bst = hc.Stats()

    def batch_step(timed: bool):
        tms = {}
        nl = 0
        for m, idx in by_m.items():
            flush_l2()
            got = hc.search_batch_raw([handles[k] for k in idx], y.data_ptr(), n,
                                      [bufs[k].data_ptr() for k in idx], [cap] * len(idx), sp,
                                      opts, bst)
            assert got == [counts[k] for k in idx], m
            tms[m] = bst.kernel_ms
            nl += bst.launches          # search (single or multi-pattern) + finish kernels
        return tms, nl

    for _ in range(args.warmup):
        step(False)
        if use_batch:
            batch_step(False)

    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    all_times = []
    all_kernel = []
    all_calls = []
    all_batch = []
    launches_total = 0
    launches_batch = 0
    with Clocks(local) as clk:
        t_wall0 = time.perf_counter()
        for _ in range(args.steps):
            times, per, launches, calls = step(True)
            all_times.append(times)
            all_kernel.append(per)
            all_calls.append(calls)
            launches_total += launches
            if use_batch:
                bt, bl = batch_step(True)
                all_batch.append(bt)
                launches_batch += bl
        torch.cuda.synchronize(dev)
        t_wall = time.perf_counter() - t_wall0
    if dist:
        dist.barrier()
    clocks = clk.summary()

    search_ms = sum(sum(t) for t in all_times)          # device time of all timed searches
    value_api = "single"
    if use_batch and args.api == "batch":
        search_ms = sum(sum(bt.values()) for bt in all_batch)
        value_api = "batch"
        launches_total = launches_batch
    bytes_done = n * len(work) * args.steps
    if shard_mode:
        bytes_done /= ws                                 # each rank covers 1/ws of every search
    if dist:
        tt = torch.tensor([search_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        search_ms_max = float(tt.item())
        bb = torch.tensor([bytes_done], dtype=torch.float64, device=dev)
        dist.all_reduce(bb, op=dist.ReduceOp.SUM)
        bytes_all = float(bb.item())
    else:
        search_ms_max, bytes_all = search_ms, float(bytes_done)
    value = bytes_all / (search_ms_max / 1e3) / 1e9

    peak, peak_src = load_peaks()
    # per-m breakdown (median over patterns and steps)
    per_m = {}
    for k, (m, q, a, o, x) in enumerate(work):
        d = per_m.setdefault(m, {"t": [], "kt": [], "ct": [], "path": None, "q": q, "alpha": a,
                                 "occ": 0})
        for s in range(args.steps):
            d["t"].append(all_times[s][k])
            d["kt"].append(all_kernel[s][k][0])
            d["ct"].append(all_calls[s][k])
        d["path"] = PATH_NAMES[all_kernel[0][k][1]]
        d["occ"] += counts[k]
    per_m_out = {}
    for m, d in per_m.items():
        med = statistics.median(d["t"])
        kmed = statistics.median(d["kt"])
        per_m_out[str(m)] = {
            "GBps_median": round(n / (med / 1e3) / 1e9, 1),
            "GBps_min": round(n / (max(d["t"]) / 1e3) / 1e9, 1),
            "GBps_max": round(n / (min(d["t"]) / 1e3) / 1e9, 1),
            "device_us_median": round(med * 1e3, 2),
            "call_us_median": round(statistics.median(d["ct"]) * 1e3, 2),
            "call_GBps_median": round(n / (statistics.median(d["ct"]) / 1e3) / 1e9, 1),
            "pct_of_measured_hbm": round(100 * n / (med / 1e3) / 1e9 / peak, 1),
            "pct_of_8TBps": round(100 * n / (med / 1e3) / 1e9 / 8000, 1),
            "q": d["q"], "alpha": d["alpha"], "path": d["path"],
            "occ_per_pattern": round(d["occ"] / len(d["t"]) * args.steps, 2),
            "prepare_us": round(prep_us[m][0], 2),
            "prepare_batch_us_per_pattern": round(prep_us[m][1], 2),
            "GBps_incl_prepare": round(n / ((med + prep_us[m][0] / 1e3) / 1e3) / 1e9, 1),
        }
        if use_batch:
            bms = [bt[m] for bt in all_batch]
            npat = len(by_m[m])
            bmed = statistics.median(bms) / npat          # ms per pattern
            per_m_out[str(m)]["batch_us_per_pattern"] = round(bmed * 1e3, 2)
            per_m_out[str(m)]["batch_GBps"] = round(n / (bmed / 1e3) / 1e9, 1)
            per_m_out[str(m)]["batch_pct_of_measured_hbm"] = round(100 * n / (bmed / 1e3) / 1e9 / peak, 1)

    # roofline of the dominant kernel: the search kernel whose launches take the largest
    # share of the step (the stream kernel on C2: m <= 32).  Algorithmic bytes per launch = f(m) * n +
    # 4 B per position written.
    shares = {}
    for m, d in per_m.items():
        shares[(d["path"])] = shares.get(d["path"], 0.0) + sum(d["kt"])
    dom = max(shares, key=shares.get)
    alg_bytes = 0.0
    kt = 0.0
    for k, (m, q, a, o, x) in enumerate(work):
        path = PATH_NAMES[all_kernel[0][k][1]]
        if path != dom:
            continue
        for s in range(args.steps):
            alg_bytes += F32.get(m, 1.0) * n + 4 * counts[k]
            kt += all_kernel[s][k][0] / 1e3
    achieved = alg_bytes / kt / 1e9 if kt > 0 else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(dom)
    roofline = {"bound": "hbm", "kernel": f"{dom}_kernel (search)", "achieved": round(achieved, 1),
                "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": traffic, "peak_source": peak_src,
                "share_of_step": round(shares[dom] / sum(shares.values()), 3),
                "algorithmic_bytes": "f(m) * n per launch (SURVEY 8(d) sector fractions) + 4 B/position"}

    line = {"metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(search_ms / args.steps, 3), "higher_is_better": True,
            "scaling": "strong" if shard_mode else "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic",
            "config": {"workload": cfg.name, "n": n, "ms": list(cfg.ms),
                       "parallelism": (f"text sharded over {ws} GPUs + NCCL all-gather" if shard_mode
                                       else f"{ws} replica(s), patterns split by rank"),
                       "patterns_per_m": len(work) // len(cfg.ms), "searches_per_step": len(work),
                       "qa": {str(m): list(cfg.qa[m]) for m in cfg.ms},
                       "l2": "flushed (2 x L2 bytes read, clean eviction) before every single search and before every batch call, outside the timed intervals",
                       "api": value_api,
                       "timing": ("value: sum over m of the device time (CUDA events on the caller's "
                                  "stream, recorded by the library) of one hc_search_batch call with "
                                  "all of that m's patterns (the searches overlap on library streams; "
                                  "each returns exactly its hc_search result); per_m also gives the "
                                  "single hc_search calls (device time per call: search + finish "
                                  "kernels) and the event time around each whole Python call")
                                 if value_api == "batch" else
                                 ("sum over searches of the library's CUDA-event device time per "
                                  "hc_search call (search kernel with fused count publication, plus "
                                  "the ordering kernels when they run); per_m also gives the event "
                                  "time around the whole Python call (host API overhead included)"),
                       "wall_ms_per_step_incl_flush": round(1000 * t_wall / args.steps, 2),
                       "text_sha256": I.sha256(y_np)[:16]},
            "pct_of_measured_hbm": round(100 * value / peak, 1),
            "pct_of_8TBps": round(100 * value / 8000, 1),
            "per_m": per_m_out, "roofline": roofline, "clocks": clocks,
            "gpu_launches": launches_total}

    # ---------------------------------------------------------------- end to end
    if not args.no_e2e:
        y_pin = torch.from_numpy(y_np).pin_memory()
        ydev = torch.empty(n, dtype=torch.uint8, device=dev)
        pos_pin = torch.empty(cap, dtype=torch.int64).pin_memory()
        h2d = n + sum(len(x) for (_, _, _, _, x) in work)
        d2h = 0
        e2e_steps = max(1, min(args.steps, 2))
        if shard_mode:
            # this rank's text: the union of its slices over the m values
            lo = min(sh.text_lo for sh in shards.values())
            hi = max(sh.text_hi for sh in shards.values())
            h2d = (hi - lo) + sum(len(x) for (_, _, _, _, x) in work)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            d2h = 0
            if shard_mode:
                ydev[lo:hi].copy_(y_pin[lo:hi], non_blocking=True)
            else:
                ydev.copy_(y_pin, non_blocking=True)
            if use_batch and args.api == "batch":
                for m, idx in by_m.items():
                    t_m = time.perf_counter()
                    hs = hc.prepare_batch([work[k][4] for k in idx], work[idx[0]][1],
                                          work[idx[0]][2])
                    got = hc.search_batch_raw(hs, ydev.data_ptr(), n,
                                              [bufs[k].data_ptr() for k in idx], [cap] * len(idx), sp)
                    for k, c in zip(idx, got):
                        pos_pin[:c].copy_(bufs[k][:c], non_blocking=True)
                        d2h += 8 + 8 * c
                    for h in hs:
                        h.close()
                    torch.cuda.synchronize(dev)   # this m's positions are on the host
                    if os.environ.get("HC_BENCH_DEBUG"):
                        print(f"e2e m={m}: {1e3 * (time.perf_counter() - t_m):.2f} ms", file=sys.stderr)
                continue
            for (m, q, a, o, x), c in zip(work, counts):
                h = hc.prepare(x, q, a)                       # host table + upload
                if shard_mode:
                    sh = shards[m]
                    got = hc.search_raw(h, ydev.data_ptr() + sh.text_lo, sh.size, pos.data_ptr(),
                                        cap, sp) if sh.size >= m else 0
                    cnt_t.fill_(got)
                    pad[:got] = pos[:got] + sh.text_lo
                    if dist:
                        dist.all_gather(g_cnt, cnt_t)
                        dist.all_gather(g_pos, pad)
                    if rank == 0:
                        cs = [int(t.item()) for t in g_cnt] if dist else [got]
                        parts = [g[:k] for g, k in zip(g_pos, cs)] if dist else [pad[:got]]
                        res = torch.cat(parts)
                        pos_pin[:res.numel()].copy_(res, non_blocking=True)
                        d2h += 8 * len(cs) + 8 * res.numel()
                else:
                    got = hc.search_raw(h, ydev.data_ptr(), n, pos.data_ptr(), cap, sp)
                    pos_pin[:got].copy_(pos[:got], non_blocking=True)
                    d2h += 8 + 8 * got
                h.close()
            torch.cuda.synchronize(dev)
        t_e2e = time.perf_counter() - t0
        if dist:
            tt = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e2e = float(tt.item())
        e2e_bytes = n * len(work) * e2e_steps * (1 if shard_mode else ws)
        line["e2e"] = {"value": round(e2e_bytes / t_e2e / 1e9, 1), "unit": "GB/s",
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                       "includes": "pinned H2D of the text, hc_prepare(_batch) of every pattern, "
                                   + ("hc_search_batch per m" if (use_batch and args.api == "batch")
                                      else "hc_search per pattern")
                                   + ", D2H of counts and positions; wall clock"}

    if rank == 0 and ws == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg, y_np, work, args.cpu_seconds)
    if rank == 0:
        s = json.dumps(line)
        print(s, flush=True)
        if args.out:
            with open(args.out, "a") as f:
                f.write(s + "\n")
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
