set -x
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_final4.json 2> gpurun_out/bench_final4.err
tail -c 300 gpurun_out/bench_final4.json; tail -2 gpurun_out/bench_final4.err
timeout 600 python -m pytest tests -m gpu -q -x --timeout=900 > gpurun_out/t_suite3.txt 2>&1; tail -2 gpurun_out/t_suite3.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
