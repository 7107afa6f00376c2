set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cpr.py -q -x 2>&1 | tail -2
BF_VERBOSE=1 python tools/profile_step.py --config 3 --maxit 2 --warm 2 2>&1 | grep -E "amg|run 2" | tail -3 | cut -c1-120
BF_SERIAL_SETUP=1 python tools/profile_step.py --config 3 --maxit 2 --warm 2 2>&1 | grep -E "run 2" | cut -c1-80
python tools/profile_step.py --config 3 --maxit 2 --warm 2 2>&1 | grep -E "run 2" | cut -c1-80
