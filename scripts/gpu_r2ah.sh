#!/bin/bash
# full GPU suite (as the driver runs it) + smoke, on the current head
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ah_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2ah_smoke.log
timeout 1800 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/r2ah_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2ah_pytest_gpu.log
tail -3 gpurun_out/r2ah_smoke.log; tail -22 gpurun_out/r2ah_pytest_gpu.log
