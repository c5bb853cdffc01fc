#!/bin/bash
# fused-epilogue correctness + load-qualifier A/B on the gather path (C2, m = 64..1024)
python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
python tools/timing_check.py > gpurun_out/tk3.log 2>&1
for v in "" _ld1 _ld2; do
  echo "== variant libhc$v" >> gpurun_out/ab_ld.log
  HC_LIB=paper_2310_15711_b200/libhc$v.so python tools/profile_search.py --config C2 --m 64 128 256 1024 --reps 4 >> gpurun_out/ab_ld.log 2>&1
done
for v in "" _ld1 _ld2; do
  HC_LIB=paper_2310_15711_b200/libhc$v.so ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum -k regex:gather_kernel --csv \
    python tools/profile_search.py --config C2 --m 128 1024 --reps 2 > gpurun_out/ncu_ld$v.csv 2>&1
done
echo done
