#!/bin/bash
# SURVEY 8(d) preset completeness: M7 hit ratio in eighths (adds 1/8, 3/8, 5/8, 7/8), M7 r=0.5 and
# L70 r=0.5 per-rank slices at P = 2, 4 (and 8 for M7)
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
OUT=gpurun_out/r02zw.jsonl; : > $OUT
A="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
for r in 0.125 0.375 0.625 0.875; do timeout 400 python bench.py --workload M7 --ratio $r $A >> $OUT 2>/dev/null; done
for P in 2 4 8; do timeout 400 python bench.py --workload M7 --ratio 0.5 --rank-slice $P $A >> $OUT 2>/dev/null; done
for P in 2 4; do timeout 600 python bench.py --workload L70 --ratio 0.5 --rank-slice $P --steps 5 --warmup 2 --no-e2e --no-cpu-baseline >> $OUT 2>/dev/null; done
python - <<'PY'
import json
for l in open("gpurun_out/r02zw.jsonl"):
    j = json.loads(l); ra = j["roofline_attn"]; rg = j["roofline_gather"]
    iso = ra["isolated"]["achieved"] if ra and ra.get("isolated") else 0
    print(f'{j["config"]["workload"][:60]:60s} {j["config"]["parallelism"][:24]:24s} ttft {j["ttft_ms"]:8.3f} dev {j["ttft_device_ms"]:8.3f} ld {j["gather_ms_per_layer"]*1e3:6.1f} us ({rg["frac"]:.3f}) attn alone {iso:5.0f} TF/s T* {j["ttft_over_t_star"] or 0:.3f} {j["roofline"]["kernel"][:9]} clk {j["clocks"]["sm_mhz"]}')
PY
