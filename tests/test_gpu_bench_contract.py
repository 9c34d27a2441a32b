"""bench.py keeps the driver's JSON-line contract (task statement, DESIGN.md
§6): one JSON line with the metric, value, timing, config, roofline,
cpu_baseline, e2e, gpu_launches and clocks keys; the reference arm prints
its own line with impl = reference."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_has_every_contract_key():
    d = _run(["--steps", "4", "--warmup", "3", "--n", str(1 << 24), "--no-extras",
              "--cpu-n", str(1 << 18)])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
              "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] == 3
    assert d["higher_is_better"] is True and d["value"] > 0
    assert "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.2
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 2 * 4 * (1 << 24) and e["d2h_bytes_per_step"] > 0
    assert 0 < e["value"] <= d["value"] * 1.01
    assert d["gpu_launches"] == 4                    # one fused update per timed step
    c = d["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in c
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


def test_reference_arm_line_same_config():
    n = 1 << 18
    ours = _run(["--steps", "4", "--warmup", "3", "--n", str(n), "--no-extras", "--cpu-n", str(n)])
    d = _run(["--impl", "reference", "--steps", "3", "--warmup", "1", "--n", str(n)])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "pairs/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert ours["impl"] == "ours" and d["config"] == ours["config"]
    assert d["metric"] == ours["metric"] and d["higher_is_better"] == ours["higher_is_better"]
