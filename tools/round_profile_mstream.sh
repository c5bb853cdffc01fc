#!/bin/bash
# ncu --set full of the multi-pattern kernel (one group of 4 C2 patterns, m = 16)
python tools/multi_one.py 16 4 > gpurun_out/m1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"mstream_kernel" -c 1 \
    -o gpurun_out/prof_mstream python tools/multi_one.py 16 4 > gpurun_out/ncu_mstream.log 2>&1
echo done
