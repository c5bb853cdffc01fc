#!/usr/bin/env python
"""Copy the outputs of tools/round_profile.sh (gpurun_out/) into profiles/r02/ under a tag
and refresh profiles/traffic.json (mean DRAM bytes per launch of the stream and gather
kernels, from the ncu --set full summary of the C2 searches).

    python tools/store_evidence.py r2g [old_tag_to_remove]
"""
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
DST = os.path.join(ROOT, "profiles", "r02")


def num(s):
    v, u = s.split()[:2]
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]


def main():
    tag = sys.argv[1]
    old = sys.argv[2] if len(sys.argv) > 2 else None
    if old:
        for f in os.listdir(DST):
            if f"_{old}" in f:
                os.remove(os.path.join(DST, f))
    shutil.copy(os.path.join(OUT, "bench.json"), os.path.join(DST, f"bench_{tag}.json"))
    shutil.copy(os.path.join(OUT, "launches.csv"), os.path.join(DST, f"launches_bench_step_{tag}.csv"))
    shutil.copy(os.path.join(OUT, "parity.txt"), os.path.join(DST, f"gputest_{tag}.txt"))
    for c in ("c2", "c3", "c4", "c5"):
        shutil.copy(os.path.join(OUT, f"ncu_summary_{c}.json"),
                    os.path.join(DST, f"ncu_full_summary_{tag}_{c}.json"))
    for f in ("ncu_lines_stream_m16.txt", "ncu_lines_gather_m1024.txt"):
        shutil.copy(os.path.join(OUT, f), os.path.join(DST, f))
    d = json.load(open(os.path.join(OUT, "ncu_summary_c2.json")))["launches"]
    tot = lambda l: num(l["dram__bytes_read.sum"]) + num(l["dram__bytes_write.sum"])
    st = [tot(l) for l in d if "stream" in l["kernel"]]
    ga = [tot(l) for l in d if "gather" in l["kernel"]]
    json.dump({"stream": sum(st) / len(st), "gather": sum(ga) / len(ga),
               "source": f"profiles/r02/ncu_full_summary_{tag}_c2.json: dram__bytes_read.sum + "
                         "dram__bytes_write.sum per launch, mean over the captured launches (stream: "
                         "C2 m=8/16/32; gather: C2 m=64/128/256/512/1024)"},
              open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
    b = json.load(open(os.path.join(OUT, "bench.json")))
    print("value", b["value"], "frac", b["roofline"]["frac"], "batch", b["batch"]["value"], "e2e",
          b["e2e"]["value"], {m: v["device_us_median"] for m, v in b["per_m"].items()})


if __name__ == "__main__":
    main()
