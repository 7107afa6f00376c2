set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cpr.py -q -x 2>&1 | tail -2
for rep in 1 2; do python tools/profile_step.py --config 3 --maxit 60 --warm 1 2>&1 | tail -1 | cut -c1-80; BF_NO_MERGE_FUSE=1 python tools/profile_step.py --config 3 --maxit 60 --warm 1 2>&1 | tail -1 | sed 's/^/nofuse /' | cut -c1-86; done
