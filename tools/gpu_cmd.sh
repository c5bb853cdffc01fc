python tools/ab.py paper_2310_15711_b200/libhc_base.so paper_2310_15711_b200/libhc_noab.so --m 64 128 256 512 1024 --per-m 3 --reps 4 > gpurun_out/ab_noab.log 2>&1
python tools/ab.py paper_2310_15711_b200/libhc_noab.so paper_2310_15711_b200/libhc.so --m 64 128 256 512 1024 --per-m 3 --reps 4 > gpurun_out/ab_noab2.log 2>&1
