set -x
for l in 0 2 4 8 16; do BF_PENCIL_LAG=$l timeout 300 python tools/ilu_bench.py --reps 10 | sed "s/^/LAG=$l /"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ilu_pencil" -s 2 -c 1 -o gpurun_out/prof_pencil2 python tools/ilu_bench.py --reps 2 > gpurun_out/ncu_pencil2.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -s -k c5 --timeout=1400 > gpurun_out/t_c5.txt 2>&1; tail -20 gpurun_out/t_c5.txt
