set -x
timeout 1200 python bench.py > gpurun_out/bench_final6.json 2> gpurun_out/bench_final6.err
tail -c 200 gpurun_out/bench_final6.json; tail -2 gpurun_out/bench_final6.err
timeout 600 python bench.py --impl reference > gpurun_out/ref_final6.json 2> gpurun_out/ref_final6.err
tail -c 300 gpurun_out/ref_final6.json
