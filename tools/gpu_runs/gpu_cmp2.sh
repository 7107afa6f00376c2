timeout 600 python -m pytest tests -m "gpu and not slow" -q -x 2>&1 | tail -3
python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1 | cut -c1-80
BF_NO_TAIL=1 python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1 | cut -c1-80
