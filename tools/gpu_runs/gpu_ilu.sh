# ILU sweep knobs, ncu of the two sweeps, full-size test durations
set -x
for c in 4 2 1 8; do for s in 0 64 256; do BF_ILU_CTAS=$c BF_ILU_SLEEP=$s timeout 300 python tools/ilu_bench.py >> gpurun_out/ilu_sweep.jsonl 2>&1; done; done
BF_ILU_FLAGS=1 timeout 300 python tools/ilu_bench.py >> gpurun_out/ilu_sweep.jsonl 2>&1
cat gpurun_out/ilu_sweep.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ilu_(fwd|bwd)_v" -s 6 -c 2 -o gpurun_out/prof_ilu python tools/ilu_bench.py --reps 2 > gpurun_out/ncu_ilu.log 2>&1
tail -2 gpurun_out/ncu_ilu.log
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q --durations=10 --timeout=2000 > gpurun_out/t_full.txt 2>&1; tail -15 gpurun_out/t_full.txt
