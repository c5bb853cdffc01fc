# stage ring sweep on the current kernel (full search)
for cfgs in "24576 2" "16384 3" "12288 4" "10240 4" "8192 6" "16384 2" "20480 2"; do
  set -- $cfgs
  echo "== tile=$1 stages=$2"
  python tools/profile_search.py --m 8 16 32 64 --reps 3 --tile $1 --stages $2 2>&1 | grep "rep=2" | awk '{print $1, $5, $6, $7, $8}'
done
