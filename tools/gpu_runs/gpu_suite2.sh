set -x
timeout 1800 python -m pytest tests -m gpu -q --durations=8 --timeout=1200 > gpurun_out/t_suite2.txt 2>&1; tail -14 gpurun_out/t_suite2.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
