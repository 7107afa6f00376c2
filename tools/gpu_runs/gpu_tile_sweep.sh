# TMA tile / CTAs-per-SM sweep: C3, 60 GMRES iterations
for cfg in "1024 8" "1024 7" "1024 6" "1024 5" "1024 4" "1536 5" "1536 4" "1024 6"; do
  set -- $cfg
  echo "TILE=$1 CTAS=$2"; BF_TMA_TILE=$1 BF_TMA_CTAS=$2 timeout 300 python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1 | cut -c1-80
done
