python tools/ab.py paper_2310_15711_b200/libhc_base.so paper_2310_15711_b200/libhc.so --m 8 16 32 64 128 --per-m 4 --reps 4 > gpurun_out/ab1.log 2>&1
