python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo rc=$? >> gpurun_out/bench_r2b.err
