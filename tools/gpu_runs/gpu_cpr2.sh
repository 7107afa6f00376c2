# CPR with value-flag sweeps: parity, timing vs flag-array sweeps, launch list of one CPR step, spectra
set -x
timeout 900 python -m pytest tests/test_gpu_cpr.py -q -x 2>&1 | tail -15
timeout 600 python tools/precond_compare.py --configs 3,4 --preconds 1,2 > gpurun_out/cpr_vflag.jsonl 2>&1
BF_ILU_FLAGS=1 timeout 600 python tools/precond_compare.py --configs 3 --preconds 2 > gpurun_out/cpr_flags.jsonl 2>&1
cat gpurun_out/cpr_vflag.jsonl gpurun_out/cpr_flags.jsonl | grep config
python tools/profile_step.py --config 3 --maxit 30 --opts precond=2 > gpurun_out/cpr_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cpr.csv python tools/profile_step.py --config 3 --maxit 30 --opts precond=2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_cpr.csv 2>&1 | head -30
timeout 1200 python tools/spectrum.py --dims 100,20 --save gpurun_out/spectrum.npz > gpurun_out/spectrum.json 2> gpurun_out/spectrum.err
tail -12 gpurun_out/spectrum.err
