set -x
timeout 1200 python tools/newton_c5.py > gpurun_out/newton_c5.json 2> gpurun_out/newton_c5.err
tail -c 1200 gpurun_out/newton_c5.json; tail -3 gpurun_out/newton_c5.err
