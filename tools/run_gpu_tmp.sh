HC_LIB=build_obj/libhc_p8.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "batch" 2>&1 | tail -2 > gpurun_out/parity.txt
for r in 1; do for v in p4 p8; do echo "== $v"; HC_LIB=build_obj/libhc_$v.so python tools/batch_bench.py --patterns 24 --ms 8 16 32 64 128 256 2>&1; done; done > gpurun_out/exp.txt
