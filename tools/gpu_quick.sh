#!/bin/bash
# parity (fast GPU tests) + per-m timing of single calls + gather traces
python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/tq.log 2>&1; echo rc=$? >> gpurun_out/tq.log
python tools/timing_check.py > gpurun_out/tkq.log 2>&1
python tools/profile_search.py --config C2 --m 128 1024 --path 2 --trace 1 --reps 3 > gpurun_out/traceq.log 2>&1
echo done
