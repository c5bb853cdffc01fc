HC_LIB=build_obj/libhc_new.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/parity.txt
for r in 1 2; do for v in base new; do echo "== $v"; HC_LIB=build_obj/libhc_$v.so python tools/profile_search.py --m 8 16 32 64 1024 --reps 4 2>&1 | grep -v "rep=0" | awk "{print \$1, \$6}"; done; done > gpurun_out/exp.txt 2>&1
