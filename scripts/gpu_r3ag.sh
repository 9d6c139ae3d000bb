#!/bin/bash
# Final-head evidence: bench line, ncu launch list of the same command, PageRank DRAM traffic over all 5 rounds.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r3ag_bench.json 2> gpurun_out/r3ag_bench.err; echo "bench rc=$?" >> gpurun_out/r3ag_bench.err
timeout 1200 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r3ag_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r3ag_ncu_launch.log 2>&1
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_pull -s 15 -c 15 --csv --log-file gpurun_out/r3ag_pr_rounds.csv python -c "
import sys; sys.path.insert(0, '.')
import paper_1312_3018_b200 as tg
eng = tg.Engine.rmat(28)
eng.pagerank(5)
print(eng.pagerank(5)[1])
" > gpurun_out/r3ag_pr.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/r3ag_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['per_algorithm_gteps'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['clocks'])"
