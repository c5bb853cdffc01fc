python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/tq.log 2>&1; echo rc=$? >> gpurun_out/tq.log
python tools/profile_search.py --config C5 --m 32 256 --reps 2 --path 5 > gpurun_out/c5scan.log 2>&1
python tools/profile_search.py --config C2 --m 8 32 256 --reps 2 --path 5 > gpurun_out/c2scan.log 2>&1
