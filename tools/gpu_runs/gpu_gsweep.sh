timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for g in 100 6 3 1.5 0.75; do echo "BF_TMA_G=$g"; BF_TMA_G=$g python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1 | cut -c1-80; done
