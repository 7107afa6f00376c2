set -x
timeout 1200 python -m pytest tests -m gpu -q --durations=5 --timeout=900 > gpurun_out/t_suite4.txt 2>&1; tail -9 gpurun_out/t_suite4.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
