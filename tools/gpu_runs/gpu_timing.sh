set -x
for rep in 1 2; do for t in 0 1 4 8; do python tools/profile_step.py --config 3 --maxit 60 --warm 1 --opts timing=$t 2>&1 | tail -1 | sed "s/^/timing=$t /" | cut -c1-100; done; done
