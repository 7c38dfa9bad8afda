export HGS_DIST_BACKEND=gloo HGS_FORCE_DEVICE=0
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/mr.out 2>gpurun_out/mr.err; echo rc=$?
wc -c gpurun_out/mr.out; tail -c 600 gpurun_out/mr.out; grep -i "error\|Traceback" -A5 gpurun_out/mr.err | head -30
