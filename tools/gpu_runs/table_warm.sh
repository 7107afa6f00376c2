#!/bin/bash
# ncu full-set table of one BF apply with the caches left as the previous kernel left them (--cache-control none):
# per-kernel rates closer to the in-graph ones than the default cold-cache capture
O=gpurun_out/${1:-table_warm}
mkdir -p $O
K='k_csr|k_wjds|k_dia|k_bsr2|k_dots|k_axpy|k_split|k_merge|k_dense_tail|k_vcycle_tail|k_coarse_inv'
ncu --set full --clock-control none --cache-control none -k regex:"$K" -s 76 -c 70 -o $O/t python tools/profile_step.py --config 3 --maxit 30 > $O/ncu.log 2>&1
python tools/ncu_table.py $O/t.ncu-rep 150 > $O/table.txt 2>&1
rm -f $O/t.ncu-rep
