set -x
for cfg in "" "BF_TMA_STAGES=3" "BF_TMA_CTAS=6" "BF_TMA_CTAS=8" "BF_TMA_STAGES=3 BF_TMA_CTAS=6"; do for rep in 1 2; do env $cfg python tools/profile_step.py --config 3 --maxit 60 --warm 1 2>&1 | tail -1 | cut -c1-60 | sed "s/^/[$cfg] /"; done; done
