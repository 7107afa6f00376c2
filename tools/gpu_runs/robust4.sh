#!/bin/bash
# sign-preserving l1 diagonal (R23): PMIS seed sweep on C2 (8 seeds), C3, C4 (3 seeds), C5
O=gpurun_out/${1:-rob4}
mkdir -p $O
for base in "theta=0.25" "smoother=0" "theta=0.18" "cheb_lo=0.3"; do
S=""
for seed in 5649 1 2 3 4 5 6 7; do S="$S;$base,seed=$seed"; done
S=${S#;}
python tools/option_sweep.py --config 2 --opts "$S" >> $O/sweep.txt 2>&1
done
for c in 3 4; do
for base in "theta=0.25" "theta=0.18"; do
S=""
for seed in 5649 1 2; do S="$S;$base,seed=$seed"; done
S=${S#;}
python tools/option_sweep.py --config $c --opts "$S" >> $O/sweep.txt 2>&1
done
done
python tools/option_sweep.py --config 5 --restart 200 --maxit 2000 --opts "theta=0.25;theta=0.18" >> $O/sweep.txt 2>&1
cat $O/sweep.txt
