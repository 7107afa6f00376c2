# mesh independence (C3 and C4 recipes at 32^3, 64^3, 128^3) for BF and CPR-AMG(2)
set -x
timeout 1200 python tools/precond_compare.py --configs 3,4 --preconds 0,2 --grids "32,32,32;64,64,64;128,128,128" > gpurun_out/mesh.jsonl 2> gpurun_out/mesh.err
grep config gpurun_out/mesh.jsonl | cut -c1-260
