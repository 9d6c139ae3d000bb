#!/bin/bash
# Final head: bench line + ncu launch list of the same command.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r3aq_bench.json 2> gpurun_out/r3aq_bench.err
timeout 1200 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r3aq_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r3aq_ncu_launch.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/r3aq_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['per_algorithm_gteps'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['share_of_kernel_time'], d['clocks'])"
