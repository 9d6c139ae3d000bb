#!/bin/bash
# compute-sanitizer on C1 with P = 1, 2, 3 (per-partition streams at P > 1), all five algorithms.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t python scripts/sanitize_c1.py > gpurun_out/r3p_$t.txt 2>&1
  echo "$t rc=$?" >> gpurun_out/r3p_$t.txt
  tail -3 gpurun_out/r3p_$t.txt
done
