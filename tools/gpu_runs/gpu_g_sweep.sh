# TMA stages / tile sweep (lanes-per-row divisor 4): C3, 60 iterations, 2 rounds
for r in 1 2; do
for cfg in "2 1024" "3 1024" "3 512" "4 512" "2 512"; do
  set -- $cfg
  echo "STAGES=$1 TILE=$2 $(BF_TMA_STAGES=$1 BF_TMA_TILE=$2 timeout 300 python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1 | cut -c1-60)"
done
done
