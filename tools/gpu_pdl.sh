#!/bin/bash
# A/B of programmatic dependent launch (PCR_PDL=1 default vs 0) on the latency-bound short-suffix
# attention (append -> attention -> split-KV combine) and on the pipelines it sits in.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; rc=$?; echo "pytest rc=$rc" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
OUT=gpurun_out/pdl.jsonl; : > $OUT
for rep in 1 2; do
for pdl in 1 0; do
  export PCR_PDL=$pdl
  timeout 300 python tools/attn_bench.py --small | sed "s/^{/{\"pdl\": $pdl, /" >> $OUT 2>> gpurun_out/pdl.err
  for P in 1 8; do
    timeout 200 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --rank-slice $P | sed "s/^{/{\"pdl\": $pdl, /" >> $OUT 2>> gpurun_out/pdl.err
  done
  timeout 300 python bench.py --workload M7 --ratio 0.5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | sed "s/^{/{\"pdl\": $pdl, /" >> $OUT 2>> gpurun_out/pdl.err
done
done
python - <<'PY'
import json
for l in open("gpurun_out/pdl.jsonl"):
    try: j=json.loads(l)
    except Exception: continue
    if "ttft_ms" in j:
        print("pdl", j["pdl"], j["config"]["workload"][:60], "ttft %.3f"%j["ttft_ms"], "attn/layer %.1fus"%(j["attn_ms_per_layer"]*1e3), "iso %.1fus"%(j["roofline_attn"]["isolated"]["avg_launch_ms"]*1e3))
    else:
        print("pdl", j["pdl"], {k: v for k, v in j.items() if k in ("ms_per_layer", "tflops", "hq", "hkv", "n1", "n2", "sm_mhz")})
PY
