set -x
bash tools/gpu_runs/gpu_c5setup.sh
for sl in 0 100 200 500; do BF_PENCIL_SLEEP=$sl timeout 300 python tools/ilu_bench.py --reps 10 | sed "s/^/SLEEP=$sl /"; done
