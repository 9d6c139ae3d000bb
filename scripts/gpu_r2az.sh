#!/bin/bash
# walker window pre-scan: parity, then A/B against the previous library (build/libtgraph_base.so)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cc.py tests/test_multiproc.py -m gpu -q -x > gpurun_out/r2az_tests.log 2>&1; tail -3 gpurun_out/r2az_tests.log
O=gpurun_out/r2az_ab.txt
echo "# new (32-bit edge offsets)" > $O
timeout 900 python scripts/sweep_env.py 28 "TG_X=1;2" >> $O 2>&1
cp paper_1312_3018_b200/libtgraph.so /tmp/new.so; cp build/libtgraph_base.so paper_1312_3018_b200/libtgraph.so
echo "# base" >> $O
timeout 900 python scripts/sweep_env.py 28 "TG_X=1;2" >> $O 2>&1
cp /tmp/new.so paper_1312_3018_b200/libtgraph.so
echo "# new again" >> $O
timeout 900 python scripts/sweep_env.py 28 "TG_X=1" >> $O 2>&1
cat $O
TG_TRACE=1 timeout 600 python scripts/trace_all.py 28 sssp,bc > gpurun_out/r2az_trace.txt 2>&1; grep "step=[3-9] \|L=[2-5]" gpurun_out/r2az_trace.txt
