#!/bin/bash
# theta x smoother x PMIS seed on C3 / C4 (the robust-on-C2 candidates)
O=gpurun_out/${1:-rob2}
mkdir -p $O
for c in 3 4; do
for base in "theta=0.18,smoother=0" "theta=0.18,smoother=0,nu_pre=2,nu_post=2" "theta=0.2,smoother=0" "theta=0.2,smoother=0,nu_pre=2,nu_post=2" "theta=0.18,smoother=0,nu_pre=1,nu_post=2" "theta=0.18,cheb_lo=0.3"; do
S=""
for seed in 5649 1 2; do S="$S;$base,seed=$seed"; done
S=${S#;}
python tools/option_sweep.py --config $c --opts "$S" >> $O/sweep.txt 2>&1
done
done
for base in "theta=0.18,smoother=0,nu_pre=2,nu_post=2" "theta=0.2,smoother=0" "theta=0.2,smoother=0,nu_pre=2,nu_post=2" "theta=0.18,smoother=0,nu_pre=1,nu_post=2" "theta=0.18,cheb_lo=0.3" "theta=0.2,cheb_lo=0.3"; do
S=""
for seed in 5649 1 2 3; do S="$S;$base,seed=$seed"; done
S=${S#;}
python tools/option_sweep.py --config 2 --opts "$S" >> $O/sweep.txt 2>&1
done
cat $O/sweep.txt
