for t in 0 1000 3000 8000 30000; do echo "BF_TAIL_NNZ=$t"; BF_TAIL_NNZ=$t python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1 | cut -c1-80; done
