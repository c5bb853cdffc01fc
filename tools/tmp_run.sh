timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tq.log 2>&1; echo rc=$? >> gpurun_out/tq.log
python tools/batch_bench.py --config C2 --ms 8 16 2>&1 | tail -2
python tools/batch_bench.py --config C4 --ms 4 8 2>&1 | tail -2
