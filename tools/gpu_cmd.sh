python -m pytest tests -m gpu -x -q > gpurun_out/tq.log 2>&1; echo rc=$? >> gpurun_out/tq.log
python tools/timing_check.py > gpurun_out/tkq.log 2>&1
