#!/bin/bash
# Parity with the default build, then attention throughput vs. the number of poly-exp2 pairs.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; rc=$?; echo "pytest rc=$rc" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
if [ $rc -ne 0 ]; then grep -E "Error|assert|FAILED" gpurun_out/gpu_tests.log | head -20; exit 1; fi
OUT=gpurun_out/poly.jsonl; : > $OUT
for P in 0 2 4; do
  PCR_NVCC_EXTRA="-DPCR_POLY_PAIRS=$P" python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
  for r in 0.0 0.5; do
    timeout 300 python bench.py --workload M7 --ratio $r --steps 10 --warmup 2 --no-e2e --no-cpu-baseline | python -c "import json,sys; j=json.loads(sys.stdin.read()); j['poly_pairs']=$P; print(json.dumps(j))" >> $OUT 2>> gpurun_out/poly.err
  done
done
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/poly.jsonl"):
    j=json.loads(l)
    print("poly", j["poly_pairs"], j["config"]["workload"][:52], "ttft %.2f"%j["ttft_ms"], "gather/layer %.1fus"%(j["gather_ms_per_layer"]*1e3), "attn/layer %.1fus %.0f TF/s (%.1f%%)"%(j["attn_ms_per_layer"]*1e3, j["roofline_attn"]["achieved"], 100*j["roofline_attn"]["frac"]))
PY
