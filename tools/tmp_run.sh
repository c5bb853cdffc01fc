P=paper_2310_15711_b200
echo "== new vs nobox (C2)"; python tools/ab.py $P/libhc.so $P/libhc_nobox.so --config C2 --m 8 16 32 --per-m 5 --reps 6
echo "== new vs nobox (C3)"; python tools/ab.py $P/libhc.so $P/libhc_nobox.so --config C3 --m 4 8 16 32 --per-m 4 --reps 4
echo "== new vs nobox (C4)"; python tools/ab.py $P/libhc.so $P/libhc_nobox.so --config C4 --m 2 4 8 16 32 --per-m 3 --reps 4
