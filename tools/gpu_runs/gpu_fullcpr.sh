set -x
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -k "c3" --durations=5 2>&1 | tail -8
