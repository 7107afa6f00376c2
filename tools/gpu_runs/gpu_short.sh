set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for rep in 1 2; do for s in 0 4 8; do BF_SHORT=$s python tools/profile_step.py --config 3 --maxit 60 --warm 1 2>&1 | tail -1 | sed "s/^/SHORT=$s /" | cut -c1-120; done; done
