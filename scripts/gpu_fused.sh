#!/bin/bash
# fused-exchange validation: full GPU suite + 2-process bench on one GPU (both modes)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for F in 1 0; do
TG_FUSED_EXCHANGE=$F TG_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --scale 24 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_2proc_fused$F.log 2>&1; echo "rc=$?" >> gpurun_out/bench_2proc_fused$F.log
done
tail -3 gpurun_out/pytest_gpu.log
