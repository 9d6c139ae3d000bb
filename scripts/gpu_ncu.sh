#!/bin/bash
# ncu evidence: launch list of the bench command + --set full of the hot kernels.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
S=${S:-28}
NCU="ncu --clock-control none"
rm -f gpurun_out/*.ncu-rep
timeout 1200 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/launches.csv python bench.py --scale $S --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_bench.log 2>&1
echo "launches rc=$?" >> gpurun_out/ncu_launch_bench.log
F="--set full --import-source on --kernel-name-base demangled"
timeout 900 $NCU $F -k regex:k_pull -c 3 -o gpurun_out/prof_pr python scripts/prof_driver.py $S pr > gpurun_out/ncu_pr.log 2>&1
timeout 900 $NCU $F -k regex:"BfsOp|k_bfs_bottom_up" -c 4 -o gpurun_out/prof_bfs python scripts/prof_driver.py $S bfs > gpurun_out/ncu_bfs.log 2>&1
timeout 900 $NCU $F -k regex:SsspOp -s 3 -c 2 -o gpurun_out/prof_sssp python scripts/prof_driver.py $S sssp > gpurun_out/ncu_sssp.log 2>&1
timeout 900 $NCU $F -k regex:"BcFwdOp|k_bc_pull" -s 1 -c 3 -o gpurun_out/prof_bcf python scripts/prof_driver.py $S bc > gpurun_out/ncu_bcf.log 2>&1
timeout 900 $NCU $F -k regex:"BcBwd" -s 1 -c 3 -o gpurun_out/prof_bcb python scripts/prof_driver.py $S bc > gpurun_out/ncu_bcb.log 2>&1
ls -la gpurun_out/
