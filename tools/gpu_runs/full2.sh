#!/bin/bash
# ncu --set full tables of one BF apply with and without the window kernels
O=gpurun_out/${1:-full2}
mkdir -p $O
K='k_csr|k_dia|k_bsr2|k_dots|k_axpy|k_split|k_merge|k_dense_tail|k_vcycle_tail|k_coarse_inv'
ncu --set full --clock-control none -k regex:"$K" -s 80 -c 110 -o $O/win python tools/profile_step.py --config 3 --maxit 30 > $O/ncu_win.log 2>&1
python tools/ncu_table.py $O/win.ncu-rep 150 > $O/win_table.txt 2>&1
rm -f $O/win.ncu-rep
BF_NO_WIN=1 ncu --set full --clock-control none -k regex:"$K" -s 80 -c 110 -o $O/nowin python tools/profile_step.py --config 3 --maxit 30 > $O/ncu_nowin.log 2>&1
python tools/ncu_table.py $O/nowin.ncu-rep 150 > $O/nowin_table.txt 2>&1
rm -f $O/nowin.ncu-rep
du -sh gpurun_out
