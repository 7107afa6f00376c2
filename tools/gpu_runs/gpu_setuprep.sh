set -x
REPS=12 python tools/setup_repeat.py 3 solve 2>&1 | tail -12 | cut -c1-40
REPS=12 BF_SERIAL_SETUP=1 python tools/setup_repeat.py 3 solve 2>&1 | tail -12 | cut -c1-40
