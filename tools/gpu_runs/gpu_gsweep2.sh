for g in 3 1.5 0.75 0.4; do echo "BF_TMA_G=$g"; BF_TMA_G=$g python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1 | cut -c1-60; done
