set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "hierarchy or split" 2>&1 | tail -2
REPS=8 python tools/setup_repeat.py 3 2>&1 | grep -o "setup [0-9.]* ms" | tr '\n' ' '; echo
BF_VERBOSE=1 REPS=3 python tools/setup_repeat.py 3 2>&1 | grep "amg" | tail -2
