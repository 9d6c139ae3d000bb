#!/bin/bash
# Validation of the session-3 head: smoke, full GPU suite, default bench line, reference arm.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3i_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r3i_smoke.log
timeout 1300 python -m pytest tests -x -q -m gpu > gpurun_out/r3i_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r3i_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r3i_bench.json 2> gpurun_out/r3i_bench.err; echo "bench rc=$?" >> gpurun_out/r3i_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r3i_bench_ref.json 2> gpurun_out/r3i_bench_ref.err
tail -2 gpurun_out/r3i_smoke.log; tail -3 gpurun_out/r3i_pytest_gpu.log; tail -c 600 gpurun_out/r3i_bench.json
