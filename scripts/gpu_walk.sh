#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for cfg in "0 4" "5 4" "6 4" "0 3" "5 2"; do set -- $cfg
  TG_WALK_MINB=$1 TG_UNROLL=$2 timeout 300 python scripts/time_algs.py 28 "minb=$1 U=$2" >> gpurun_out/walk.txt 2>&1
done
