# CPR / coupled AMG on the GPU: parity tests, comparison table, then the whole GPU suite timed
set -x
timeout 900 python -m pytest tests/test_gpu_cpr.py -q -x 2>&1 | tail -25
timeout 900 python tools/precond_compare.py --configs 1,2,3,4 > gpurun_out/precond_compare.jsonl 2> gpurun_out/precond_compare.err
tail -c 4000 gpurun_out/precond_compare.jsonl
tail -5 gpurun_out/precond_compare.err
timeout 2000 python -m pytest tests -m gpu -q --durations=30 > gpurun_out/pytest_gpu_durations.txt 2>&1
tail -45 gpurun_out/pytest_gpu_durations.txt
