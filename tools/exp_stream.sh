for cfgs in "16384 2 0 1 0" "16384 2 0 2 0" "32768 2 0 1 0" "16384 3 0 1 0" "15360 2 0 0 0" "16384 2 0 0 0" "32768 2 0 0 0" "8192 3 0 0 0"; do
  set -- $cfgs
  echo "== tile=$1 stages=$2 cps=$3 debug=$4 chunk=$5"
  python tools/profile_search.py --m 8 16 32 64 --reps 3 --tile $1 --stages $2 --cps $3 --debug $4 --chunk $5 2>&1 | grep "rep=2"
done
