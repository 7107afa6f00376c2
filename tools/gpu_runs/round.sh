#!/bin/bash
# GPU-box pass, results under gpurun_out/<tag>/.  Stages (second argument, default "bench launches full"):
#   tests    the GPU test suite
#   bench    the default bench line
#   launches ncu launch list of the bench command (first 7000 launches: warm-up step setup + its solve)
#            and of one setup + GMRES(30) cycle (tools/profile_step.py), with per-kernel DRAM bytes
#   full     ncu --set full capture of one BF apply + J SpMV + CGS2 passes
set -x
O=gpurun_out/${1:-round}
STAGES=${2:-"bench launches full"}
mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for s in $STAGES; do
case $s in
tests)
  python -m pytest tests -m gpu -x -q --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
  tail -5 $O/pytest_gpu.log;;
bench)
  python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
  tail -c 300 $O/bench.json;;
launches)
  ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 7000 --log-file $O/launches_bench.csv \
      python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_bench.log 2>&1
  python tools/launch_summary.py $O/launches_bench.csv > $O/launches_bench.txt 2>&1
  ncu --metrics $M --clock-control none --csv --log-file $O/launches_step.csv \
      python tools/profile_step.py --config 3 --maxit 30 > $O/ncu_step.log 2>&1
  python tools/launch_summary.py $O/launches_step.csv > $O/launches_step.txt 2>&1
  python tools/traffic_summary.py $O/launches_step.csv > $O/traffic.json 2> $O/traffic.err;;
full)
  ncu --set full --clock-control none --import-source on \
      -k regex:'k_csr|k_wjds|k_dia|k_bsr2|k_dots|k_axpy|k_split|k_merge|k_dense_tail|k_vcycle_tail|k_coarse_inv' \
      -s 70 -c 150 -o $O/full_apply python tools/profile_step.py --config 3 --maxit 30 > $O/ncu_full.log 2>&1
  python tools/ncu_table.py $O/full_apply.ncu-rep 150 > $O/full_apply_table.txt 2>&1
  # gpurun_out/ is capped at 64 MiB: keep the report only if it is small
  if [ $(stat -c %s $O/full_apply.ncu-rep) -gt 30000000 ]; then rm -f $O/full_apply.ncu-rep; fi;;
esac
done
rm -f $O/*.csv.tmp; du -sh gpurun_out; ls -la $O
