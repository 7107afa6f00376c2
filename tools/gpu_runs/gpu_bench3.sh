set -x
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_final3.json 2> gpurun_out/bench_final3.err
tail -c 600 gpurun_out/bench_final3.json
tail -3 gpurun_out/bench_final3.err
