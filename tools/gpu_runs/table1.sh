#!/bin/bash
O=gpurun_out/${1:-table1}
mkdir -p $O
K='k_csr|k_wjds|k_dia|k_bsr2|k_split|k_merge|k_dense_tail|k_vcycle_tail|k_coarse_inv'
ncu --set full --clock-control none -k regex:"$K" -s ${2:-75} -c ${3:-60} -o $O/t python tools/profile_step.py --config 3 --maxit 30 > $O/ncu.log 2>&1
python tools/ncu_table.py $O/t.ncu-rep 150 > $O/table.txt 2>&1
rm -f $O/t.ncu-rep
grep -E "k_wjds|kernel" $O/table.txt
