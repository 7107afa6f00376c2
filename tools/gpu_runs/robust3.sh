#!/bin/bash
# theta = 0.18 neighbourhood: Chebyshev lower end x PMIS seed (C2, C3, C4), the theta cliff, C5
O=gpurun_out/${1:-rob3}
mkdir -p $O
for base in "theta=0.18,cheb_lo=0.1" "theta=0.18,cheb_lo=0.2" "theta=0.18,cheb_lo=0.3" "theta=0.18,cheb_lo=0.4" "theta=0.25,cheb_lo=0.3"; do
S=""
for seed in 5649 1 2 3 4 5 6 7; do S="$S;$base,seed=$seed"; done
S=${S#;}
python tools/option_sweep.py --config 2 --opts "$S" >> $O/sweep.txt 2>&1
done
for c in 3 4; do
for base in "theta=0.18,cheb_lo=0.2" "theta=0.16" "theta=0.17" "theta=0.17,cheb_lo=0.3"; do
S=""
for seed in 5649 1 2; do S="$S;$base,seed=$seed"; done
S=${S#;}
python tools/option_sweep.py --config $c --opts "$S" >> $O/sweep.txt 2>&1
done
done
python tools/option_sweep.py --config 5 --restart 200 --maxit 2000 --opts "theta=0.18;theta=0.18,cheb_lo=0.3" >> $O/sweep.txt 2>&1
cat $O/sweep.txt
