set -x
timeout 2400 python -m pytest tests -m gpu -q --durations=25 --timeout=1500 > gpurun_out/t_suite.txt 2>&1; tail -35 gpurun_out/t_suite.txt
bash tools/gpu_runs/gpu_mesh.sh
