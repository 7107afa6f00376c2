for gp in 0 1 2 4; do for gr in 0 1 4 8; do echo "P=$gp R=$gr"; BF_TMA_G_P=$gp BF_TMA_G_R=$gr python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1 | cut -c1-60; done; done
