"""bench.py end to end on the B200 (the driver's contract): one JSON line with the base keys, the
roofline of the dominant kernel (measured live), the CPU oracle baseline, the end-to-end number
through the public API with host buffers, clocks and the kernel-launch count -- on the small preset
T (seconds) and on the default L8 line's M7 north_star sub-record fields."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def _bench(*args, timeout=600):
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract_preset_t():
    j = _bench("--workload", "T", "--steps", "3", "--warmup", "3", "--no-target-point", "--cpu-budget-s", "1")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert k in j, k
    assert j["n_gpus"] == 1 and j["steps"] == 3 and j["warmup"] == 3 and j["value"] > 0
    assert j["config"]["workload"].startswith("T:")
    r = j["roofline"]
    assert r["bound"] in ("host-link", "tensor") and r["achieved"] > 0 and 0 < r["frac"] < 1.2 and r["peak"] > 0
    assert j["cpu_baseline"]["kind"] == "oracle" and j["cpu_baseline"]["cores"] >= 1 and j["cpu_baseline"]["value"] > 0
    e = j["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert j["gpu_launches"] > 0
    assert j["clocks"]["sm_max_mhz"] and j["clocks"]["samples"] >= 0


def test_bench_north_star_subrecord_m7():
    """The default line carries the M7 r=0.5 north_star point: load and attention as fractions of
    their peaks, hidden-load %, TTFT / T* (shortened run; values are sanity-checked only)."""
    j = _bench("--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu-baseline", "--profile-steps", "1", timeout=900)
    ns = j["north_star_point"]
    assert ns["workload"].startswith("M7:")
    assert 0.5 < ns["load_frac_of_h2d_peak"] < 1.1
    assert 0.2 < ns["attn_frac_of_bf16_peak"] < 1.0
    assert ns["t_star_ms"] > 0 and ns["ttft_over_t_star"] >= 0.95
    assert j["roofline"]["bound"] == "host-link" and 0.7 < j["roofline"]["frac"] < 1.05
