set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for rep in 1 2 3; do python tools/profile_step.py --config 3 --maxit 60 --warm 1 2>&1 | tail -1 | cut -c1-80; done
