timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/parity.txt
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
