# exercise the multi-rank bench path (NCCL init, barrier, max-over-ranks) with one rank
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline 2>gpurun_out/tr1.err | tail -1
tail -3 gpurun_out/tr1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 2>>gpurun_out/tr1.err | tail -1
