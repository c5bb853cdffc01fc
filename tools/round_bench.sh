#!/bin/bash
# GPU tests, bench line and ncu launch list (small outputs only)
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1 > gpurun_out/parity.txt
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --steps 1 --warmup 3 --per-m 5 --no-e2e --no-cpu > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --per-m 5 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo done
