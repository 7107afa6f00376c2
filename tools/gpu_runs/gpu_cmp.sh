timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python tools/profile_step.py --config 3 --maxit 30 --warm 2 2>&1 | tail -1 | cut -c1-80
BF_NO_TMA=1 python tools/profile_step.py --config 3 --maxit 30 --warm 2 2>&1 | tail -1 | cut -c1-80
