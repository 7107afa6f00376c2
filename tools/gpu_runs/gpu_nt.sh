# quick check: parity subset + C3 60 iterations x2
timeout 600 python -m pytest tests -m "gpu and not slow" -q -x 2>&1 | tail -1
for r in 1 2; do echo "$(timeout 300 python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1 | cut -c1-70)"; done
