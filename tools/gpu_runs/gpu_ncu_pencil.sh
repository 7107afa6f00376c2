set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ilu_pencil" -s 2 -c 2 -o gpurun_out/prof_pencil python tools/ilu_bench.py --reps 2 > gpurun_out/ncu_pencil.log 2>&1
tail -2 gpurun_out/ncu_pencil.log
