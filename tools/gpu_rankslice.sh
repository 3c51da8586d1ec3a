#!/bin/bash
# Per-rank work of a P-GPU KV-head-sharded run, emulated on one GPU (bench.py --rank-slice P),
# for each a2 mover.
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
OUT=gpurun_out/rankslice.jsonl; : > $OUT
for P in 2 4 8; do for m in sm ce_runs; do
  timeout 200 python bench.py --rank-slice $P --load-mode $m --steps 30 --warmup 5 --no-e2e --no-cpu-baseline >> $OUT 2>> gpurun_out/rankslice.err
done; done
python - <<'PY'
import json
for l in open("gpurun_out/rankslice.jsonl"):
    j=json.loads(l)
    print(j["config"]["parallelism"][:28], j.get("pipeline"), "ttft %.3f ms"%j["ttft_ms"], "ms/step %.3f"%j["ms_per_step"], "load %.1fus %.1f GB/s (%.3f)"%(j["gather_ms_per_layer"]*1e3, j["roofline"]["achieved"] if j["roofline"]["unit"]=="GB/s" else -1, j["roofline"]["frac"]), "attn %.1fus"%(j["attn_ms_per_layer"]*1e3), j["load_path"])
PY
