set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "long_rows" 2>&1 | tail -3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_csr_short|k_ilu_pencil|k_cpr_resid|k_cpr_merge" -s 8 -c 8 -o gpurun_out/prof_cpr_short python tools/profile_step.py --config 3 --maxit 4 --opts precond=2 > gpurun_out/ncu_cpr_short.log 2>&1
tail -1 gpurun_out/ncu_cpr_short.log
