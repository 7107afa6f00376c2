# CPR parity (fixed graph patching), suite durations per file, CPR timing + launch list, spectra
set -x
timeout 900 python -m pytest tests/test_gpu_cpr.py -q -x > gpurun_out/t_cpr.txt 2>&1; tail -15 gpurun_out/t_cpr.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_assemble.py -q --durations=15 --timeout=600 > gpurun_out/t_parity.txt 2>&1; tail -22 gpurun_out/t_parity.txt
timeout 600 python tools/precond_compare.py --configs 1,2,3,4 > gpurun_out/precond_compare.jsonl 2> gpurun_out/precond_compare.err
BF_ILU_FLAGS=1 timeout 300 python tools/precond_compare.py --configs 3 --preconds 2 > gpurun_out/cpr_flags.jsonl 2>&1
grep config gpurun_out/precond_compare.jsonl gpurun_out/cpr_flags.jsonl | cut -c1-400
python tools/profile_step.py --config 3 --maxit 30 --opts precond=2 > gpurun_out/cpr_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cpr.csv python tools/profile_step.py --config 3 --maxit 30 --opts precond=2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_cpr.csv 2>&1 | head -25
