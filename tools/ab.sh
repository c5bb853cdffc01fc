#!/bin/bash
# A/B: run profile_search.py with build_obj/libhc_base.so and libhc_new.so, interleaved.
#   tools/ab.sh "<profile_search args>" [rounds]
for r in $(seq ${2:-2}); do
  for v in base new; do
    echo "== $v"
    HC_LIB=build_obj/libhc_$v.so python tools/profile_search.py $1 2>&1 | grep -v "rep=0"
  done
done
