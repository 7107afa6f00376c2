set -x
free -g; nproc
for t in "16 8" "32 4" "8 16" "8 8" "4 32" "16 4" "128 1"; do set -- $t; BF_PENCIL_TJ=$1 BF_PENCIL_TK=$2 timeout 300 python tools/ilu_bench.py --reps 10 | sed "s/^/TJ=$1 TK=$2 /" >> gpurun_out/tiles.txt 2>&1; done
cat gpurun_out/tiles.txt
