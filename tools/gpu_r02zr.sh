#!/bin/bash
# SURVEY-defined device TTFT beside the step time
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02zr_bench.jsonl 2> gpurun_out/r02zr_bench.err; echo rc=$?
python - <<'PY'
import json
j = json.loads(open("gpurun_out/r02zr_bench.jsonl").read().strip().splitlines()[-1])
ns = j["north_star_point"]
print("L8 ttft", round(j["ttft_ms"], 3), "device", round(j["ttft_device_ms"], 3), "T*", round(j["ttft_over_t_star"], 3), round(j["ttft_device_over_t_star"], 3), "match us", round(j["match_prefix_us"]), "e2e", round(j["e2e"]["value"]), j["e2e"].get("host_hugepage_frac"))
print("M7 ttft", round(ns["ttft_ms"], 3), "device", round(ns["ttft_device_ms"], 3))
PY
timeout 300 python -m pytest tests/test_bench_gpu.py -q 2>&1 | tail -1
