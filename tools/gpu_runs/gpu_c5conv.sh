set -x
timeout 1500 python tools/precond_compare.py --configs 5 --preconds 0,2 --maxit 1500 > gpurun_out/c5conv.jsonl 2> gpurun_out/c5conv.err
grep config gpurun_out/c5conv.jsonl | cut -c1-300
timeout 900 python tools/precond_compare.py --configs 5 --preconds 0 --smoother 1 --maxit 1500 >> gpurun_out/c5conv.jsonl 2>> gpurun_out/c5conv.err
tail -1 gpurun_out/c5conv.jsonl | cut -c1-300
