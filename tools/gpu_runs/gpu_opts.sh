set -x
timeout 900 python tools/option_sweep.py --config 3 > gpurun_out/opts_c3.txt 2>&1; cat gpurun_out/opts_c3.txt
timeout 900 python tools/option_sweep.py --config 4 > gpurun_out/opts_c4.txt 2>&1; cat gpurun_out/opts_c4.txt
