#!/usr/bin/env python
"""Summarise an ncu --set full report (per kernel launch) and a launch-list csv.

    python tools/ncu_summary.py REPORT.ncu-rep [LAUNCHES.csv] > summary.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg",
    "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers",
]
STALL = "smsp__pcsamp_warps_issue_stalled_"


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def main():
    hdr, units, data = raw(sys.argv[1])
    res = []
    for r in data:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        e = {"kernel": d.get("Kernel Name", ""), "id": d.get("ID", "")}
        for m in METRICS:
            if m in d:
                e[m] = f"{d[m]} {u.get(m, '')}".strip()
        st = {k[len(STALL):]: float((d[k] or "0").replace(",", ""))
              for k in d if k.startswith(STALL) and not k.endswith("_not_issued")}
        tot = sum(st.values()) or 1.0
        e["top_stalls_pct"] = {k: round(100 * v / tot, 1)
                               for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:6]}
        res.append(e)
    out = {"report": sys.argv[1], "launches": res}
    if len(sys.argv) > 2:
        txt = open(sys.argv[2]).read().splitlines()
        i = [k for k, l in enumerate(txt) if l.startswith('"ID"')][0]
        rows = list(csv.DictReader(io.StringIO("\n".join(txt[i:]))))
        share = {}
        for r in rows:
            name = r["Kernel Name"].split("(")[0].replace("void ", "")
            name = "torch L2 flush" if name.startswith("at::") else name.split("<")[0]
            share[name] = share.get(name, 0.0) + float(r["Metric Value"])
        tot = sum(v for k, v in share.items() if k != "torch L2 flush")
        out["launch_list_share_excl_flush"] = {k: round(v / tot, 3) for k, v in share.items()
                                               if k != "torch L2 flush"}
        out["launch_list_ns"] = {k: v for k, v in share.items()}
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main()
