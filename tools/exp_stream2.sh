#!/bin/bash
# stream path (per-warp cp.async chunks) vs staged: chunk bytes x buffers sweep
echo "== staged"
python tools/profile_search.py --m 8 16 32 64 --reps 3 --path 1 2>&1 | grep -v "rep=0" | awk '{print $1, $5, $6, $7, $8}'
for cfgs in "2048 3" "1024 4" "2048 2" "4096 2" "4096 3" "1024 3" "3072 3"; do
  set -- $cfgs
  echo "== stream chunk=$1 bufs=$2"
  python tools/profile_search.py --m 8 16 32 64 --reps 3 --path 3 --tile $1 --stages $2 2>&1 | grep -v "rep=0" | awk '{print $1, $5, $6, $7, $8}'
done
