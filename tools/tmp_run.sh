timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tq.log 2>&1; echo rc=$? >> gpurun_out/tq.log
P=paper_2310_15711_b200
echo "== prev vs new (C2)"; python tools/ab.py $P/libhc_prev.so $P/libhc.so --config C2 --m 8 16 32 --per-m 5 --reps 6
echo "== prev vs new (C3)"; python tools/ab.py $P/libhc_prev.so $P/libhc.so --config C3 --m 4 8 16 --per-m 4 --reps 4
echo "== prev vs new (C4)"; python tools/ab.py $P/libhc_prev.so $P/libhc.so --config C4 --m 2 4 8 16 --per-m 3 --reps 4
