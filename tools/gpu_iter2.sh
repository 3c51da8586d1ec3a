#!/bin/bash
# v3 attention: parity, then a short perf sweep; then the workloads that failed last time.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; rc=$?; echo "pytest rc=$rc" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
if [ $rc -ne 0 ]; then grep -E "Error|assert|FAILED" gpurun_out/gpu_tests.log | head -20; exit 1; fi
OUT=gpurun_out/sweep.jsonl; : > $OUT
timeout 200 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline >> $OUT 2> gpurun_out/e1.err || tail -5 gpurun_out/e1.err
timeout 200 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --mode sync >> $OUT 2> gpurun_out/e2.err || tail -5 gpurun_out/e2.err
for r in 0.0 0.5; do
  timeout 300 python bench.py --workload M7 --ratio $r --steps 10 --warmup 2 --no-e2e --no-cpu-baseline >> $OUT 2> gpurun_out/e3.err || tail -5 gpurun_out/e3.err
done
timeout 300 python bench.py --workload M7 --ratio 0.5 --steps 10 --warmup 2 --no-e2e --no-cpu-baseline --layer-body >> $OUT 2> gpurun_out/e4.err || tail -20 gpurun_out/e4.err
timeout 300 python bench.py --workload T --steps 20 --warmup 3 --no-e2e --no-cpu-baseline >> $OUT 2> gpurun_out/e5.err || tail -20 gpurun_out/e5.err
python - <<'PY'
import json
for l in open("gpurun_out/sweep.jsonl"):
    j=json.loads(l)
    ra=j.get("roofline_attn") or {}
    print(j["config"]["workload"][:60], j["config"]["workload"][-30:], "ttft %.2f"%j["ttft_ms"], "gather/layer %.1fus"%(j["gather_ms_per_layer"]*1e3), "attn/layer", j.get("attn_ms_per_layer"), "TF/s", ra.get("achieved"), ra.get("frac"))
PY
