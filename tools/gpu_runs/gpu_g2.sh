for lim in 8 100; do echo "lim=$lim"; BF_STENCIL_G2=$lim python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1 | cut -c1-60; done
