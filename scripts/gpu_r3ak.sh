#!/bin/bash
# --set full captures of the final PageRank class pulls (a non-final round) and the dense SSSP walker launch.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/final_pr.ncu-rep gpurun_out/final_sssp.ncu-rep
F="--set full --import-source on --kernel-name-base demangled --clock-control none"
timeout 900 ncu $F -k regex:k_pull -s 3 -c 3 -o gpurun_out/final_pr python -c "
import sys; sys.path.insert(0, '.')
import paper_1312_3018_b200 as tg
eng = tg.Engine.rmat(28)
print(eng.pagerank(5)[1])
" > gpurun_out/final_pr.log 2>&1
timeout 900 ncu $F -k regex:SsspOp -s 4 -c 1 -o gpurun_out/final_sssp python scripts/prof_driver.py 28 sssp > gpurun_out/final_sssp.log 2>&1
for r in final_pr final_sssp; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null
done
ls -la gpurun_out/final_*
