# dense tail operator check: parity subset, C3 60 iterations, 2 rounds
timeout 600 python -m pytest tests -m "gpu and not slow" -q -x 2>&1 | tail -3
for r in 1 2; do
  echo "dtail    $(timeout 300 python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1 | cut -c1-70)"
  echo "no dtail $(BF_NO_DTAIL=1 timeout 300 python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1 | cut -c1-70)"
done
