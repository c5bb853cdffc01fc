set -x
python tools/profile_search.py --config C2 --m 1024 128 64 --path 2 --trace 1 --reps 3 > gpurun_out/trace_gather.log 2>&1
python tools/profile_search.py --config C2 --m 8 16 1024 128 --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stream_kernel|gather_kernel" -c 8 -o gpurun_out/prof_r2a python tools/profile_search.py --config C2 --m 8 16 1024 128 --reps 2 > gpurun_out/ncu_r2a.log 2>&1
echo done
