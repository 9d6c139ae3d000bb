#!/bin/bash
# Multi-process bench path on the final head: 2 and 4 ranks sharing one GPU (gloo plumbing), RMAT-24.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for N in 2 4; do
  TG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N --scale 24 --steps 3 --warmup 3 --out gpurun_out/r3aj_bench_${N}proc.json > gpurun_out/r3aj_bench_${N}proc.log 2>&1
  echo "N=$N rc=$?"; tail -c 300 gpurun_out/r3aj_bench_${N}proc.log
done
