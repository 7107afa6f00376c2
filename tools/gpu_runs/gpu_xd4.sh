set -x
timeout 900 python -m pytest tests/test_gpu_cpr.py -q -x 2>&1 | tail -2
for rep in 1 2; do timeout 300 python tools/ilu_bench.py --reps 10; done
