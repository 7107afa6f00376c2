#!/bin/bash
# R23 (coarsening stops before a Galerkin level with a non-positive diagonal): PMIS seed sweep
O=gpurun_out/${1:-rob5}
mkdir -p $O
for base in "diag_stop=1" "diag_stop=1,smoother=0" "diag_stop=0"; do
S=""
for seed in 5649 1 2 3 4 5 6 7; do S="$S;$base,seed=$seed"; done
S=${S#;}
python tools/option_sweep.py --config 2 --opts "$S" >> $O/sweep.txt 2>&1
done
for c in 3 4; do
S=""
for seed in 5649 1 2; do S="$S;diag_stop=1,seed=$seed"; done
S=${S#;}
python tools/option_sweep.py --config $c --opts "$S" >> $O/sweep.txt 2>&1
done
python tools/option_sweep.py --config 5 --restart 200 --maxit 2000 --opts "diag_stop=1;diag_stop=0" >> $O/sweep.txt 2>&1
python tools/option_sweep.py --config 5 --restart 30 --maxit 3000 --opts "diag_stop=1" >> $O/sweep.txt 2>&1
python tools/option_sweep.py --config 1 --opts "diag_stop=1;diag_stop=0" >> $O/sweep.txt 2>&1
cat $O/sweep.txt
