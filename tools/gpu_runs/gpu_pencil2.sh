set -x
timeout 900 python -m pytest tests/test_gpu_cpr.py -q -x > gpurun_out/t_cpr3.txt 2>&1; tail -5 gpurun_out/t_cpr3.txt
timeout 300 python tools/ilu_bench.py > gpurun_out/ilu_pencil2.jsonl 2>&1; cat gpurun_out/ilu_pencil2.jsonl
timeout 600 python tools/precond_compare.py --configs 3,4 --preconds 2 > gpurun_out/cpr_pencil2.jsonl 2>&1; grep config gpurun_out/cpr_pencil2.jsonl | cut -c1-330
timeout 1500 python tools/spectrum.py --dims 100,20 --save gpurun_out/spectrum.npz > gpurun_out/spectrum.json 2> gpurun_out/spectrum.err; tail -9 gpurun_out/spectrum.err
