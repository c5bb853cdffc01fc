HC_LIB=build_obj/libhc_pm32.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/parity.txt
for r in 1 2; do for v in 0 8 32; do echo "== pm$v"; HC_LIB=build_obj/libhc_pm$v.so python tools/profile_search.py --m 8 16 32 --reps 3 --path 3 2>&1 | grep -v "rep=0" | awk "{print \$1, \$6}"; done; done > gpurun_out/exp.txt 2>&1
