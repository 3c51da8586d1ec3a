#!/bin/bash
# E12 analogue (fig:breakdown): base / Only-Up / Only-Down / Up-Down on M7 with the new
# chunks offloaded layer by layer (f1), plus the offload parity tests in every mode.
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -q -x -k "offload" 2>&1 | tail -2
OUT=gpurun_out/breakdown.jsonl; : > $OUT
for r in 0.25 0.5 0.75; do for m in sync only-up only-down overlap; do
  timeout 300 python bench.py --workload M7 --ratio $r --offload --mode $m --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> $OUT 2>> gpurun_out/breakdown.err
done; done
python - <<'PY'
import json
for l in open("gpurun_out/breakdown.jsonl"):
    j=json.loads(l)
    print("N1", j["config"]["N1"], j["pipeline"]["mode"], "ttft %.2f ms"%j["ttft_ms"], "load %.0f us"%(j["gather_ms_per_layer"]*1e3), "attn %.0f us"%(j["attn_ms_per_layer"]*1e3), "offload %.0f us (%.1f MiB)"%((j["offload_ms_per_layer"] or 0)*1e3, (j["offload_bytes_per_layer"] or 0)/2**20), j["clocks"]["reasons"])
PY
tail -3 gpurun_out/breakdown.err
