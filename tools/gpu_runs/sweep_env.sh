#!/bin/bash
# sweep of environment settings on C3 / C4 full solves: sweep_env.sh <tag> "<VAR=V ...>" "<VAR=V ...>" ...
O=gpurun_out/$1
mkdir -p $O
shift
i=0
for e in "BF_NOP=1" "$@"; do
  for cfg in 3 4; do
    env $e python tools/profile_step.py --config $cfg --maxit 1000 --warm 2 > $O/s${i}_c$cfg.log 2>&1
    echo "C$cfg [$e]: $(grep '^run 2' $O/s${i}_c$cfg.log | cut -c8-52)"
  done
  i=$((i+1))
done
