for cfgs in "16384 2 0" "16384 3 0" "16384 4 0" "32768 2 0" "32768 3 0" "8192 4 0" "8192 8 0" "15360 2 0"; do
  set -- $cfgs
  echo "== tile=$1 stages=$2 cps=$3"
  python tools/profile_search.py --m 16 64 --reps 3 --tile $1 --stages $2 --cps $3 --debug 1 2>&1 | grep "rep=2" | sed 's/^/DEBUG /'
  python tools/profile_search.py --m 8 16 32 64 --reps 3 --tile $1 --stages $2 --cps $3 2>&1 | grep "rep=2"
done
