#!/bin/bash
# multi-process bench path (2 and 4 ranks sharing the one GPU, gloo for the torch side)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for N in 2 4; do
TG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $N --scale 24 --steps 3 --warmup 3 --out gpurun_out/r2ap_bench_${N}proc.json > gpurun_out/r2ap_bench_${N}proc.log 2>&1
echo "N=$N rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2ap_bench_${N}proc.json')); print(d['value'], d['n_gpus'], d['per_algorithm_ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['config']['parallelism'])"
done
