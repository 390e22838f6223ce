"""bench.py's driver contract on a reduced run: one JSON line with the keys
the driver and the judge read (metric, value, e2e with its copy sizes,
roofline with traffic, clocks, gpu_launches), the in-line parity check
against the reference-made cfg-2 fixture passing, and a positive
throughput. The full default run is the driver's; this guards the line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--groups", "2", "--steps", "1", "--warmup", "3",
           "--skip-spmv", "--skip-cpu", "--skip-canonical", "--skip-asm", "--skip-widths", "--skip-configs",
           "--skip-dd"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 3
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    ro = d["roofline"]
    assert ro["bound"] == "hbm" and 0 < ro["frac"] <= 1.0 and ro["peak"] > 0 and ro["traffic"]
    assert d["gpu_launches"] > 0 and "workload" in d["config"]
    par = d["parity"]["serial_vs_reference"]
    assert par["iterations_equal"] and par["solutions_bitwise"]
