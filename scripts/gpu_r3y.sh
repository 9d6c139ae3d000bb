#!/bin/bash
# Final bench line + ncu launch list of the same command + PageRank per-round DRAM traffic (a non-final round).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r3y_bench.json 2> gpurun_out/r3y_bench.err; echo "bench rc=$?" >> gpurun_out/r3y_bench.err
timeout 1200 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r3y_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r3y_ncu_launch.log 2>&1
echo "launches rc=$?" >> gpurun_out/r3y_ncu_launch.log
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_pull -c 6 --csv --log-file gpurun_out/r3y_pr_rounds.csv python -c "
import sys; sys.path.insert(0, '.')
import paper_1312_3018_b200 as tg
eng = tg.Engine.rmat(28)
print(eng.pagerank(5)[1])
" > gpurun_out/r3y_pr.log 2>&1
tail -c 400 gpurun_out/r3y_bench.json; tail -2 gpurun_out/r3y_ncu_launch.log
