timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -4 > gpurun_out/parity.txt
for path in 3 4; do echo "== path $path"; python tools/profile_search.py --m 8 16 32 64 --reps 3 --path $path 2>&1 | grep -v "rep=0" | awk '{print $1, $5, $6, $7, $8}'; done > gpurun_out/exp.txt 2>&1
echo "== C5 shc" >> gpurun_out/exp.txt; timeout 300 python tools/profile_search.py --config C5 --m 32 256 --reps 2 --path 4 2>&1 | tail -4 >> gpurun_out/exp.txt
