#!/bin/bash
# C2 (64^3) convergence vs PMIS seed for several smoother settings
O=gpurun_out/${1:-c2r}
mkdir -p $O
for base in "smoother=0" "smoother=1,smoother_p=-1" "smoother=1,smoother_p=-1,cheb_lo=0.05,cheb_degree=3" "nu_pre=2,nu_post=2" "smoother=0,nu_pre=2,nu_post=2" "theta=0.18,smoother=1,smoother_p=-1" "theta=0.18,smoother=0" "cheb_lo=0.3" "cheb_lo=0.05"; do
S=""
for seed in 5649 1 2 3; do S="$S;$base,seed=$seed"; done
S=${S#;}
python tools/option_sweep.py --config 2 --opts "$S" >> $O/sweep.txt 2>&1
done
python tools/option_sweep.py --config 2 --restart 60 --opts "seed=5649;seed=1;seed=2;seed=3" >> $O/sweep.txt 2>&1
cat $O/sweep.txt
