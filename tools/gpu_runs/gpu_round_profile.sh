# round-end evidence: tests, bench line, ncu launch list of one step, ncu --set full of the top kernels
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python tools/profile_step.py --config 3 --maxit 30 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python tools/profile_step.py --config 3 --maxit 30 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_csr_tma|k_dia|k_bsr2|k_dots|k_axpy" -s 60 -c 40 -o gpurun_out/prof_final python tools/profile_step.py --config 3 --maxit 30 > gpurun_out/ncu_final.log 2>&1
tail -1 gpurun_out/ncu_final.log
