# quick GPU check: parity tests, one profiled step (plain), launch list
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
BF_VERBOSE=1 python tools/profile_step.py --config 3 --maxit 30 --warm 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_quick.csv python tools/profile_step.py --config 3 --maxit 30 > /dev/null 2>&1
tail -2 gpurun_out/prof_plain.log
if [ "$FULL" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_csr|k_bsr2|k_dots|k_axpy" -s 40 -c 40 -o gpurun_out/prof_full python tools/profile_step.py --config 3 --maxit 30 > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
fi
