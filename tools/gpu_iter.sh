#!/bin/bash
# One iteration: parity tests, then a short perf sweep (L8, L8 sync, M7 r in {0, 0.5, 1}).
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; rc=$?; echo "pytest rc=$rc" >> gpurun_out/gpu_tests.log
tail -4 gpurun_out/gpu_tests.log
if [ $rc -ne 0 ]; then grep -E "Error|assert|FAILED" gpurun_out/gpu_tests.log | head -20; exit 1; fi
OUT=gpurun_out/sweep.jsonl; : > $OUT
timeout 200 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline >> $OUT 2>> gpurun_out/sweep.err
timeout 200 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --mode sync >> $OUT 2>> gpurun_out/sweep.err
for r in 0.0 0.5 0.75 1.0; do
  timeout 300 python bench.py --workload M7 --ratio $r --steps 10 --warmup 2 --no-e2e --no-cpu-baseline >> $OUT 2>> gpurun_out/sweep.err
done
python - <<'PY'
import json
for l in open("gpurun_out/sweep.jsonl"):
    j=json.loads(l)
    print(j["config"]["workload"][:60], j["config"]["workload"][-13:], "ttft %.2f"%j["ttft_ms"], "gather/layer %.1fus"%(j["gather_ms_per_layer"]*1e3), "attn/layer %.1fus %.0f TF/s (%.1f%%)"%(j["attn_ms_per_layer"]*1e3, j["roofline_attn"]["achieved"], 100*j["roofline_attn"]["frac"]), "clk", j["clocks"].get("sm_mhz"))
PY
tail -3 gpurun_out/sweep.err
