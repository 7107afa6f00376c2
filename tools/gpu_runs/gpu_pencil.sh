# pencil ILU sweeps: parity, timing, CPR comparison at C3/C4, smoke
set -x
timeout 900 python -m pytest tests/test_gpu_cpr.py -q -x > gpurun_out/t_cpr2.txt 2>&1; tail -15 gpurun_out/t_cpr2.txt
timeout 300 python tools/ilu_bench.py > gpurun_out/ilu_pencil.jsonl 2>&1
BF_ILU_PENCIL=0 timeout 300 python tools/ilu_bench.py >> gpurun_out/ilu_pencil.jsonl 2>&1
cat gpurun_out/ilu_pencil.jsonl
timeout 600 python tools/precond_compare.py --configs 3,4 --preconds 1,2 > gpurun_out/cpr_pencil.jsonl 2>&1; grep config gpurun_out/cpr_pencil.jsonl | cut -c1-330
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
