# tail-threshold sweep: C3, 60 GMRES iterations, per-iteration time
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for t in 0 3000 30000 400000 2000000; do
  for bps in 1 2; do
    echo "TAIL_NNZ=$t BPS=$bps"; BF_TAIL_NNZ=$t BF_TAIL_BPS=$bps timeout 300 python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1
  done
done
BF_NO_TAIL=1 timeout 300 python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1
