# PDL on the GMRES step kernels: parity subset, C3 60 iterations, 2 rounds
timeout 600 python -m pytest tests -m "gpu and not slow" -q -x 2>&1 | tail -2
for r in 1 2; do
  echo "pdl    $(timeout 300 python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1 | cut -c1-70)"
  echo "no pdl $(BF_NO_PDL=1 timeout 300 python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1 | cut -c1-70)"
done
