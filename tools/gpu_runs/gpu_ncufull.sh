set -x
python tools/profile_step.py --config 3 --maxit 30 > gpurun_out/plain_nf.log 2>&1 && \
timeout 1200 ncu -f --set full --clock-control none -k regex:"k_csr|k_dia|k_bsr2|k_dots|k_axpy|k_split_vec|k_merge_vec|k_dense_tail|k_dia_smooth_merge" -s 70 -c 45 -o /tmp/prof_bf_final python tools/profile_step.py --config 3 --maxit 30 > gpurun_out/ncu_bf_final.log 2>&1
tail -1 gpurun_out/ncu_bf_final.log
python tools/ncu_table.py /tmp/prof_bf_final.ncu-rep > gpurun_out/ncu_bf_final_table.txt 2>&1
ncu -i /tmp/prof_bf_final.ncu-rep --page raw --csv > gpurun_out/ncu_bf_final_raw.csv 2>/dev/null
ls -la gpurun_out/
