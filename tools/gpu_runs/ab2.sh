#!/bin/bash
O=gpurun_out/${1:-ab2}
mkdir -p $O
for cfg in 3 4; do
  BF_VERBOSE=1 python tools/profile_step.py --config $cfg --maxit 1000 --warm 2 > $O/win_c$cfg.log 2> $O/win_c$cfg.err
  BF_NO_WIN=1 python tools/profile_step.py --config $cfg --maxit 1000 --warm 2 > $O/nowin_c$cfg.log 2>&1
  grep "^run [12]" $O/win_c$cfg.log | cut -c1-100; grep "^run [12]" $O/nowin_c$cfg.log | cut -c1-100
done
grep "wjds" $O/win_c3.err | sort | uniq | head -20
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file $O/launches_step.csv python tools/profile_step.py --config 3 --maxit 30 > $O/ncu_step.log 2>&1
python tools/launch_summary.py $O/launches_step.csv > $O/launches_step.txt 2>&1
python tools/traffic_summary.py $O/launches_step.csv > $O/traffic.json 2> $O/traffic.err
head -40 $O/launches_step.txt
