set -x
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_final5.json 2> gpurun_out/bench_final5.err
tail -c 200 gpurun_out/bench_final5.json; tail -2 gpurun_out/bench_final5.err
python tools/profile_step.py --config 3 --maxit 30 > gpurun_out/plain_final5.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_final5.csv python tools/profile_step.py --config 3 --maxit 30 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_final5.csv | head -5
