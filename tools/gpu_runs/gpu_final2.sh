set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "long_rows or gmres or apply" 2>&1 | tail -3
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err
tail -c 800 gpurun_out/bench_final2.json
python tools/profile_step.py --config 3 --maxit 30 > gpurun_out/plain_final2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_final2.csv python tools/profile_step.py --config 3 --maxit 30 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_final2.csv | head -8
