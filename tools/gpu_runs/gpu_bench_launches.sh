# bench line + ncu launch list (time + DRAM bytes) of one GMRES(30) cycle at C3
timeout 600 python -m pytest tests -m "gpu and not slow" -q -x 2>&1 | tail -1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_now.json 2> gpurun_out/bench_now.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_now.csv python tools/profile_step.py --config 3 --maxit 30 > /dev/null 2>&1
echo done
