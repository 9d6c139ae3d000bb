#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
if grep -q "pytest rc=0" gpurun_out/pytest_gpu.log; then
timeout 1500 python bench.py --scale ${S:-28} --steps 3 --warmup 2 ${BENCH_ARGS} --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
python - <<'PY'
import json
d=json.load(open("gpurun_out/bench.json"))
print("value",d["value"],"ms/step",d["ms_per_step"],"e2e",d["e2e"] and d["e2e"]["value"])
print("per_alg",{k:round(v,2) for k,v in d["per_algorithm_gteps"].items()})
print("ms",{k:round(v,2) for k,v in d["per_algorithm_ms_per_step"].items()})
print("roof",{k:d["roofline"][k] for k in ("kernel","achieved","frac","share_of_kernel_time")})
for k,v in d["kernels"].items(): print("  ",k,v)
print("build_s",d["config"]["build_s"],"clocks",d["clocks"],"cpu",d["cpu_baseline"] and d["cpu_baseline"]["value"])
PY
fi
