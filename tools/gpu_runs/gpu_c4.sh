set -x
timeout 1200 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
tail -c 300 gpurun_out/bench_c4.json; tail -2 gpurun_out/bench_c4.err
