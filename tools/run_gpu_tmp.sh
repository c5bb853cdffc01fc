timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/parity.txt
for r in 1 2; do for v in base new; do for spl in 2 4; do echo "== $v spl=$spl"; HC_LIB=build_obj/libhc_$v.so python tools/profile_search.py --m 64 128 256 512 1024 --reps 3 --path 2 --spl $spl 2>&1 | grep "rep=2" | awk "{print \$1, \$6}"; done; done; done > gpurun_out/exp.txt 2>&1
