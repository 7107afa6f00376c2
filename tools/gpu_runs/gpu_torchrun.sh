set -x
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --steps 2 --warmup 3 > gpurun_out/bench_torchrun.json 2> gpurun_out/bench_torchrun.err
tail -c 400 gpurun_out/bench_torchrun.json; tail -3 gpurun_out/bench_torchrun.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29612 bench.py --impl reference --gpus 1 --steps 2 --warmup 3 > gpurun_out/ref_torchrun.json 2> gpurun_out/ref_torchrun.err
tail -c 300 gpurun_out/ref_torchrun.json; tail -3 gpurun_out/ref_torchrun.err
