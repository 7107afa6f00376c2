#!/bin/bash
# A/B of the shared-memory window kernels (k_csr_win.cuh) on C3 / C4 full solves + the parity tests that cover them
O=gpurun_out/${1:-ab_win}
mkdir -p $O
python -m pytest tests/test_gpu_parity.py -x -q -k "variants" > $O/pytest_variants.log 2>&1; tail -3 $O/pytest_variants.log
for cfg in 3 4; do
  BF_VERBOSE=1 python tools/profile_step.py --config $cfg --maxit 1000 --warm 2 > $O/win_c$cfg.log 2> $O/win_c$cfg.err
  BF_NO_WIN=1 python tools/profile_step.py --config $cfg --maxit 1000 --warm 2 > $O/nowin_c$cfg.log 2>&1
  grep "^run" $O/win_c$cfg.log | cut -c1-120; grep "^run" $O/nowin_c$cfg.log | cut -c1-120
done
grep "window" $O/win_c3.err | sort | uniq | head -20
python -m pytest tests/test_gpu_fullsize.py -x -q -k "c3_hierarchy or c3_gmres_forced or c4_full" > $O/pytest_full.log 2>&1; tail -3 $O/pytest_full.log
