for r in 1 2; do for v in base new; do echo "== $v"; HC_LIB=build_obj/libhc_$v.so python tools/batch_bench.py --patterns 20 --ms 8 16 32 64 256 2>&1; done; done > gpurun_out/exp.txt
