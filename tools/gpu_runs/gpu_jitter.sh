set -x
for rep in 1 2 3; do python tools/profile_step.py --config 3 --maxit 10 --warm 2 2>&1 | grep -o "setup [0-9.]* ms" | tr '\n' ' '; echo; done
REPS=10 python tools/setup_repeat.py 3 solve 2>&1 | grep -o "setup [0-9.]* ms, device bytes [0-9.]*" | tr '\n' ';'
