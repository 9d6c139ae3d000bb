"""bench.py's driver contract on CPU: the reference arm (the CPU oracle on a
bounded sample) prints one JSON line with the keys the driver reads, on our
arm's metric / unit, its config naming the sample it actually runs."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                         cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GTEPS"
    # the config names what this arm runs (a bounded RMAT-20 sample of RMAT-28)
    assert d["config"]["scale"] == 20 and "RMAT-20" in d["config"]["workload"]
    assert "RMAT-28" in d["config"]["sample_of"]
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["cpu_baseline"]["nproc"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_gather_probe_ceiling_parses_the_committed_table():
    sys.path.insert(0, ROOT)
    import bench

    c = bench.gather_probe_ceiling()
    assert c is not None and 1e11 < c < 1e12
