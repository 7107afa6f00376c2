# fused-restriction check: parity tests, then C3 60 iterations with/without, interleaved
timeout 600 python -m pytest tests -m "gpu and not slow" -q -x 2>&1 | tail -3
for i in 1 2; do
  echo "rfuse";    timeout 300 python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1 | cut -c1-80
  echo "rfuse+L0"; BF_RFUSE_L0=1 timeout 300 python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1 | cut -c1-80
  echo "no rfuse"; BF_NO_RFUSE=1 timeout 300 python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1 | cut -c1-80
done
BF_VERBOSE=1 timeout 300 python tools/profile_step.py --config 3 --maxit 60 --warm 0 2>&1 | grep -i "setup\|rfuse" | tail -5
