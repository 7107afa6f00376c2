#!/bin/bash
# A/B of one environment setting on C3 / C4 full solves: ab_env.sh <tag> "<VAR=VALUE ...>"
O=gpurun_out/${1:-ab_env}
mkdir -p $O
for cfg in 3 4; do
  python tools/profile_step.py --config $cfg --maxit 1000 --warm 2 > $O/base_c$cfg.log 2>&1
  env $2 python tools/profile_step.py --config $cfg --maxit 1000 --warm 2 > $O/alt_c$cfg.log 2>&1
  echo "C$cfg default:"; grep "^run [12]" $O/base_c$cfg.log | cut -c1-100; echo "C$cfg $2:"; grep "^run [12]" $O/alt_c$cfg.log | cut -c1-100
done
