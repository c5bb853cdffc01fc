#!/usr/bin/env python
"""Per-source-line hot spots of one kernel in an ncu report (--print-source cuda,sass).

    python tools/ncu_lines.py REPORT.ncu-rep 'stream_kernel<(int)4' [top]

Aggregates, per (file, line), the warp-level instructions executed and the warp-stall
samples, over the first function block whose name contains the pattern, and prints the
top lines with their source text.
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    rep, pat = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    blocks = []
    cur = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = {"file": r[1], "fn": None, "rows": [], "hdr": None}
            blocks.append(cur)
        elif r[0] == "Function Name" and cur is not None:
            cur["fn"] = r[1]
        elif r[0] == "Line No" and cur is not None:
            cur["hdr"] = r
        elif cur is not None and cur["hdr"] is not None:
            cur["rows"].append(r)
    # the function blocks of the first matching kernel (one per source file)
    fn = next((b["fn"] for b in blocks if b["fn"] and pat in b["fn"]), None)
    if fn is None:
        print("no match")
        return
    agg = defaultdict(lambda: [0.0, 0.0, ""])
    tot_i = tot_s = 0.0
    seen = set()
    for b in blocks:
        if b["fn"] != fn or b["file"] in seen:
            continue
        seen.add(b["file"])
        h = b["hdr"]
        ii = h.index("Instructions Executed")
        si = h.index("Warp Stall Sampling (All Samples)")
        line = None
        src = ""
        for r in b["rows"]:
            if r[0]:
                line, src = r[0], r[1]
            try:
                ins = float(r[ii] or 0)
                smp = float(r[si] or 0)
            except (ValueError, IndexError):
                continue
            key = (b["file"].split("/")[-1], line)
            a = agg[key]
            a[0] += ins
            a[1] += smp
            a[2] = src
            tot_i += ins
            tot_s += smp
    print(f"{fn}: {tot_i:.0f} warp instructions, {tot_s:.0f} stall samples")
    for (f, ln), (ins, smp, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{f}:{ln:>5} inst {100 * ins / max(tot_i, 1):5.1f}%  samples {100 * smp / max(tot_s, 1):5.1f}%  {src.strip()[:90]}")


if __name__ == "__main__":
    main()
