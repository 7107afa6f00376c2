set -x
timeout 900 python -m pytest tests/test_gpu_cpr.py -q -x > gpurun_out/t_cpr4.txt 2>&1; tail -3 gpurun_out/t_cpr4.txt
for t in "16 8" "8 8" "32 4"; do set -- $t; BF_PENCIL_TJ=$1 BF_PENCIL_TK=$2 timeout 300 python tools/ilu_bench.py --reps 10 | sed "s/^/TJ=$1 TK=$2 /"; done
