# round evidence: bench line, launch list (time + DRAM bytes) of one BF step, CPR comparison
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
tail -c 1500 gpurun_out/bench_final.json
python tools/profile_step.py --config 3 --maxit 30 > gpurun_out/plain_final.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python tools/profile_step.py --config 3 --maxit 30 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_final.csv | head -12
timeout 900 python tools/precond_compare.py --configs 1,2,3,4 > gpurun_out/precond_compare_final.jsonl 2> gpurun_out/precond_compare_final.err
grep config gpurun_out/precond_compare_final.jsonl | cut -c1-250
