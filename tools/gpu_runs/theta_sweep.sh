#!/bin/bash
# strength-threshold sweep with the R22 default smoothers: theta x PMIS seed (C2, C3, C4)
O=gpurun_out/${1:-theta}
mkdir -p $O
S=""
for th in 0.25 0.2 0.18 0.22; do for seed in 5649 1 2 3; do S="$S;theta=$th,seed=$seed"; done; done
S=${S#;}
for c in 3 4 2; do
python tools/option_sweep.py --config $c --opts "$S" >> $O/sweep.txt 2>&1
done
python tools/option_sweep.py --config 5 --restart 200 --maxit 2000 --opts "theta=0.25;theta=0.2" >> $O/sweep.txt 2>&1
cat $O/sweep.txt
