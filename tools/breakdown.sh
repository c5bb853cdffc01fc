#!/bin/bash
# per-phase breakdown of the stream path on C2 (instrumented build): full search, copy
# pipeline alone (debug 1), copy + phase A (debug 3), epilogue ordering stamps (debug 10)
for d in 0 1 3 10; do
  echo "== debug $d"
  python tools/profile_search.py --config C2 --m ${MS:-8 16 32} --reps 4 --debug $d 2>&1 | grep -v "rep=0"
done
