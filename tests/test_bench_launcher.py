"""bench.py's launcher and reference arm on the CPU (no GPU needed):
`--gpus 2` forms a 2-rank group by itself (re-exec under
torch.distributed.run, gloo here), `--gpus 1` stays one process, a launcher
whose rank count disagrees with --gpus fails loudly, and the reference arm
prints the contract line on the same `config` object as our arm."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _run(args, env=None, rc=0):
    e = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                         capture_output=True, text=True, timeout=300, env=e)
    assert out.returncode == rc, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    return [json.loads(ln) for ln in lines], out


def test_gpus_2_spawns_two_ranks():
    lines, _ = _run(["--gpus", "2", "--dry-run"])
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["ranks"] == [0, 1] and d["local_ranks"] == [0, 1]
    assert d["distinct_pids"] == 2


def test_gpus_1_is_one_process():
    lines, _ = _run(["--dry-run"])
    assert lines == [{"dry_run": True, "impl": "ours", "n_gpus": 1, "ranks": [0],
                      "local_ranks": [0], "distinct_pids": 1}]


def test_rank_count_mismatch_fails_loudly():
    _, out = _run(["--gpus", "4", "--dry-run"],
                  env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"}, rc=2)
    assert "--gpus 4" in out.stderr


def test_reference_arm_contract_on_cpu():
    import bench
    n = 1 << 16
    lines, _ = _run(["--impl", "reference", "--n", str(n), "--steps", "2", "--warmup", "1"])
    assert len(lines) == 1
    d = lines[0]
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "pairs/s"
    assert d["metric"] == bench.METRIC and d["config"] == bench.workload_config(n, 1)
    assert d["steps"] == 2 and d["warmup"] == 1 and d["n_gpus"] == 1
    assert d["e2e"] == {"value": d["value"], "unit": "pairs/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    c = d["cpu_baseline"]
    assert c["kind"] == "reference" and c["cores"] >= 1 and c["value"] == d["value"]
    # under a 2-rank launcher only rank 0 prints, on the 2-GPU config
    lines, _ = _run(["--impl", "reference", "--gpus", "2", "--n", str(n), "--steps", "1",
                     "--warmup", "1"])
    assert len(lines) == 1 and lines[0]["config"] == bench.workload_config(n, 2)
