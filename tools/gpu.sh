#!/bin/bash
# build libhc.so (fail fast), then run the given command on the GPU box
set -e
cd /root/repo
python -m paper_2310_15711_b200.build > /tmp/build.log 2>&1 || { grep -E "error" -A3 /tmp/build.log | head -20; exit 1; }
timeout 3000 /usr/local/graft/bin/gpurun --timeout ${GPU_TIMEOUT:-1200} -- "$1" 2>&1 | grep -v "^\[gpurun\] send"
