set -x
BF_VERBOSE=1 python tools/profile_step.py --config 3 --maxit 2 --warm 2 2>&1 | grep -v "^\[bf_setup\]   " | tail -24
