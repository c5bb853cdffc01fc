for g in 0 32 128; do
echo "== HC_L2_FETCH=$g"
if [ $g = 0 ]; then unset HC_L2_FETCH; else export HC_L2_FETCH=$g; fi
python tools/profile_search.py --config C2 --m 32 64 128 256 512 1024 --reps 6 2>&1 | grep "rep=[345]\|libhc" | awk '{print $1, $6}' | paste -sd' '
done
