#!/bin/bash
# Per-rank work of KV-head sharding vs the context-split variant (bench.py --rank-slice P
# --shard heads|context) at P = 2 / 4 / 8, L8 and M7 r=0.5; plus the default bench line.
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
OUT=gpurun_out/ctxsplit.jsonl; : > $OUT
timeout 300 python bench.py --no-cpu-baseline >> $OUT 2>> gpurun_out/ctxsplit.err
for P in 2 4 8; do for sh in heads context; do
  timeout 200 python bench.py --rank-slice $P --shard $sh --steps 20 --warmup 3 --no-e2e --no-cpu-baseline >> $OUT 2>> gpurun_out/ctxsplit.err
  timeout 200 python bench.py --workload M7 --ratio 0.5 --rank-slice $P --shard $sh --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> $OUT 2>> gpurun_out/ctxsplit.err
done; done
python - <<'PY'
import json
for l in open("gpurun_out/ctxsplit.jsonl"):
    j=json.loads(l)
    ra=j["roofline_attn"] or {}
    print(j["config"]["workload"][:3], j["config"]["parallelism"][:32], "ttft %.3f"%j["ttft_ms"], "load %.1fus"%(j["gather_ms_per_layer"]*1e3), "%.3f"%j["roofline"]["frac"] if j["roofline"]["unit"]=="GB/s" else "", "attn %.1fus %.0f TF/s"%(j["attn_ms_per_layer"]*1e3, ra.get("achieved", 0)), j["load_path"])
PY
tail -3 gpurun_out/ctxsplit.err
