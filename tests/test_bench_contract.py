"""bench.py's reference arm (CPU) prints one JSON line with the keys the
driver reads; the GPU arm's line is exercised on the B200 (-m gpu)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["config"]["workload"] == "cfg3"
    # the GPU arm prints the same workload-defining config (driver: same_config)
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == json.loads(json.dumps(bench.product_config(bench.workload("cfg3"))))


@pytest.mark.gpu
def test_gpu_arm_line():
    d = _run(["--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-fit"])
    for k in ("roofline", "e2e", "gpu_launches", "clocks", "e2e_numpy_f64"):
        assert k in d, k
    r = d["roofline"]
    assert 0 < r["frac"] <= 1 and r["peak"] > 0 and r["unit"] == "TFLOP/s"
    ex = r["executed"]
    assert 0 < ex["tensor"]["frac"] <= 1 and 0 < ex["mufu"]["frac"] <= 1
    assert r["frac_executed"] == max(ex["tensor"]["frac"], ex["mufu"]["frac"])
    assert d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
