P=paper_2310_15711_b200
echo "== base vs oldverify"; python tools/ab.py $P/libhc_base.so $P/libhc_oldv.so --config C2 --m 16 32 64 128 1024 --per-m 4 --reps 4
echo "== new vs oldverify"; python tools/ab.py $P/libhc.so $P/libhc_oldv.so --config C2 --m 16 32 64 128 1024 --per-m 4 --reps 4
