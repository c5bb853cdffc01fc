timeout 400 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/parity.txt
python tools/profile_search.py --m 8 16 --reps 3 --path 3 2>&1 | grep -v "rep=0" | awk '{print $1, $5, $6}' > gpurun_out/exp.txt
python tools/profile_search.py --config C3 --m 4 --reps 3 2>&1 | grep -v "rep=0" | awk '{print $1, $5, $6}' >> gpurun_out/exp.txt
