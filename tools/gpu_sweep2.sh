#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
OUT=gpurun_out/sweep.jsonl; : > $OUT
for g in 8 16 32; do
  timeout 200 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --gather-ctas $g >> $OUT 2>> gpurun_out/sweep.err
done
timeout 200 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --mode sync >> $OUT 2>> gpurun_out/sweep.err
for r in 0.0 0.5 1.0; do
  timeout 300 python bench.py --workload M7 --ratio $r --steps 10 --warmup 2 --no-e2e --no-cpu-baseline >> $OUT 2>> gpurun_out/sweep.err
done
python - <<'PY'
import json
for l in open("gpurun_out/sweep.jsonl"):
    j=json.loads(l)
    print(j["config"]["workload"][:90], "ctas", j["gather_ctas"], "ttft %.2f"%j["ttft_ms"], "gather/layer %.1fus (%.1f GB/s, evented %.1fus)"%(j["gather_ms_per_layer"]*1e3, j["roofline"]["achieved"] if j["roofline"]["unit"]=="GB/s" else -1, j["gather_ms_per_layer_evented"]*1e3), "attn/layer %.1fus %.0f TF/s"%(j["attn_ms_per_layer"]*1e3, j["roofline_attn"]["achieved"]), "peak h2d", round(j["roofline"]["peak"],1))
PY
tail -3 gpurun_out/sweep.err
