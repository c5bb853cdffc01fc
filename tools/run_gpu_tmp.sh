timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/parity.txt
for t in 0 8192; do echo "== shc tile=$t"; python tools/profile_search.py --m 8 16 32 64 --reps 3 --path 4 --tile $t 2>&1 | grep "rep=2" | awk "{print \$1, \$6, \$8, \$9}"; done > gpurun_out/exp.txt 2>&1
