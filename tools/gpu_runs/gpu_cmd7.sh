timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python tools/profile_step.py --config 3 --maxit 30 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_v2.csv python tools/profile_step.py --config 3 --maxit 30 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csr -c 16 -o gpurun_out/prof_csr python tools/profile_step.py --config 3 --maxit 30 > gpurun_out/ncu_csr.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dots|k_axpy_dots|k_axpy_norm|k_bsr2" -s 80 -c 4 -o gpurun_out/prof_gm python tools/profile_step.py --config 3 --maxit 30 > gpurun_out/ncu_gm.log 2>&1
tail -2 gpurun_out/prof_plain.log; tail -2 gpurun_out/ncu_csr.log; tail -2 gpurun_out/ncu_gm.log
