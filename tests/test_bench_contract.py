"""bench.py's JSON contract on the CPU: the reference arm (the fp64 oracle timed on the host
cores) prints one line with the base contract's keys, and our arm refuses to run without a GPU
(no CPU fallback on the product path)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=600, cwd=ROOT, env=dict(os.environ, CUDA_VISIBLE_DEVICES=""))


def test_reference_arm_line_keys():
    res = _bench("--impl", "reference", "--workload", "T", "--steps", "2", "--warmup", "1")
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in j, k
    assert j["impl"] == "reference" and j["steps"] == 2 and j["warmup"] == 1 and j["n_gpus"] == 1
    assert j["value"] > 0 and j["higher_is_better"] is True and j["vs_baseline"] is None
    assert j["config"]["workload"].startswith("T:")
    assert j["cpu_baseline"]["kind"] == "oracle" and j["cpu_baseline"]["cores"] >= 1
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["d2h_bytes_per_step"] == 0
    assert j["e2e"]["value"] == pytest.approx(j["value"])


def test_our_arm_fails_loudly_without_a_gpu():
    res = _bench("--workload", "T", "--steps", "1", "--warmup", "0", "--no-cpu-baseline", "--no-e2e")
    assert res.returncode != 0
    assert not [ln for ln in res.stdout.splitlines() if ln.startswith("{")]   # no bench line


@pytest.mark.parametrize("n", [2, 3])
def test_gpus_n_self_launches_n_ranks(n):
    """`bench.py --gpus N` without a launcher starts N ranks itself (torchrun, 127.0.0.1); the
    dry run brings them up on gloo and rank 0 reports every rank (no GPU needed)."""
    res = _bench("--gpus", str(n), "--dry-run")
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    assert j["dry_run"] is True and j["n_gpus"] == n
    assert sorted(r["rank"] for r in j["ranks"]) == list(range(n))
    assert len({r["pid"] for r in j["ranks"]}) == n          # one process per rank
