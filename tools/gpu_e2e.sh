#!/bin/bash
# host_io (e2e) path: its parity tests, then the L8 and M7 r=0.5 bench lines with e2e.
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -q -x -k "host_io or offload or overlap_sync" 2>&1 | tail -2
: > gpurun_out/e2e.jsonl
timeout 300 python bench.py --no-cpu-baseline >> gpurun_out/e2e.jsonl 2>> gpurun_out/e2e.err
timeout 300 python bench.py --no-cpu-baseline --load-mode sm >> gpurun_out/e2e.jsonl 2>> gpurun_out/e2e.err
timeout 300 python bench.py --workload M7 --ratio 0.5 --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/e2e.jsonl 2>> gpurun_out/e2e.err
python - <<'PY'
import json
for l in open("gpurun_out/e2e.jsonl"):
    j=json.loads(l)
    print(j["config"]["workload"][:3], j.get("pipeline"), "val %.0f ttft %.3f e2e %.0f"%(j["value"], j["ttft_ms"], j["e2e"]["value"]), j["clocks"]["reasons"])
PY
