#!/bin/bash
# M7 r=0.5 pipeline interference: gather CTAs 2/4/8/16, the gather on its own SMs (PCR_GATHER_SMEM),
# and the attention alone on the same box
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
OUT=gpurun_out/r02za.jsonl; : > $OUT
timeout 300 python tools/attn_bench.py --shape 4096,4224,32,8 2>&1 | tail -1
for G in 8 4 2 16 8; do
  timeout 300 python bench.py --workload M7 --ratio 0.5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --gather-ctas $G >> $OUT 2>/dev/null
done
PCR_GATHER_SMEM=200000 timeout 300 python bench.py --workload M7 --ratio 0.5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> $OUT 2>/dev/null
PCR_PDL=0 timeout 300 python bench.py --workload M7 --ratio 0.5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> $OUT 2>/dev/null
python - <<'PY'
import json
for l in open("gpurun_out/r02za.jsonl"):
    j = json.loads(l); ra = j["roofline_attn"]; rg = j["roofline_gather"]
    print(f'gather_ctas {j.get("gather_ctas")} ttft {j["ttft_ms"]:.3f} ld/layer {j["gather_ms_per_layer"]*1e3:.1f} us ({rg["frac"]:.3f}) attn pipe {ra["achieved"]:.0f} iso {ra["isolated"]["achieved"] if ra.get("isolated") else 0:.0f} TF/s T* {j["ttft_over_t_star"]:.3f} clk {j["clocks"]["sm_mhz"]}')
PY
