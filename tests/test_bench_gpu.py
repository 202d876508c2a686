"""bench.py's own arm keeps the driver's JSON contract (one line; roofline,
e2e, clocks, gpu_launches, cpu_baseline) -- small configurations on one GPU."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("config,extra", [("c1", []), ("c2", ["--n", "200000", "--nq", "1000"]),
                                          ("c4", ["--n", "20000", "--nq", "256"])])
def test_bench_json_contract(config, extra):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", config, "--steps", "3",
                          "--warmup", "3", "--e2e-steps", "1", *extra],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks",
                "cpu_baseline"):
        assert key in d, key
    assert d["value"] > 0 and d["steps"] == 3 and d["warmup"] == 3 and d["gpu_launches"] > 0
    r = d["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    assert 0 < r["frac"] < 2
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert "workload" in d["config"]
    nt = d["near_ties"]  # stage parity of the run's own codes and tables (SURVEY 8(c) rules)
    assert nt["code_mismatches_not_near_tie"] == 0 and nt["table_mismatches_not_near_tie"] == 0
    assert d["cpu_baseline"]["cpu"]
