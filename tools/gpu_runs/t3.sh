#!/bin/bash
O=gpurun_out/${1:-t3}
mkdir -p $O
python -m pytest tests/test_gpu_parity.py tests/test_gpu_checked.py -x -q > $O/pytest_a.log 2>&1; tail -4 $O/pytest_a.log
for cfg in 3 4; do
  BF_VERBOSE=1 python tools/profile_step.py --config $cfg --maxit 1000 --warm 2 > $O/win_c$cfg.log 2> $O/win_c$cfg.err
  grep "^run [12]" $O/win_c$cfg.log | cut -c1-100
done
python -m pytest tests/test_gpu_fullsize.py -x -q > $O/pytest_full.log 2>&1; tail -3 $O/pytest_full.log
