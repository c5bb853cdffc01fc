#!/bin/bash
# bench + ncu evidence for profiles/ (run on the GPU box)
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1 > gpurun_out/parity.txt
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
# launch list of one bench step (reduced: 5 patterns per m) -- cold-cache, serialised
python bench.py --steps 1 --warmup 3 --per-m 5 --no-e2e --no-cpu > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --per-m 5 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
# full capture of the stream kernel (m=8, m=16, m=32) and the gather kernel (m=128)
python tools/profile_search.py --m 8 16 32 128 --reps 1 > gpurun_out/pf_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stream_kernel|gather_kernel" -c 4 \
    -o gpurun_out/prof_round python tools/profile_search.py --m 8 16 32 128 --reps 1 > gpurun_out/ncu_full.log 2>&1
echo done
