#!/bin/bash
# SM partition between the gather and the attention: co-resident (default) vs exclusive SMs for
# the gather (dynamic smem reservation) with the attention's split sizing on the remaining SMs
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r02f.jsonl; : > $OUT
run() {  # tag env... -- bench args
  tag=$1; shift
  env "$@" > /dev/null 2>&1
}
for cfg in "base||16" "excl16|PCR_GATHER_SMEM=40960 PCR_ATTN_SMS=132|16" "excl8|PCR_GATHER_SMEM=40960 PCR_ATTN_SMS=140|8" "share8||8"; do
  IFS='|' read tag envs ctas <<< "$cfg"
  for wl in "--workload L8" "--workload M7 --ratio 0.5" "--rank-slice 8"; do
    line=$(env $envs timeout 300 python bench.py $wl --gather-ctas $ctas --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-target-point 2>/dev/null | tail -1)
    echo "{\"tag\": \"$tag\", \"wl\": \"$wl\", \"line\": $line}" >> $OUT
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/r02f.jsonl"):
    try: j = json.loads(l)
    except Exception: print("bad", l[:200]); continue
    b = j["line"]; ra = b["roofline_attn"]
    print(f'{j["tag"]:7s} {j["wl"]:26s} ttft {b["ttft_ms"]:.3f} ld {b["gather_ms_per_layer"]*1e3:6.1f} us  attn {b["attn_ms_per_layer"]*1e3:6.1f} us (iso {ra["isolated"]["avg_launch_ms"]*1e3 if ra.get("isolated") else float("nan"):6.1f})  T* ratio {b["ttft_over_t_star"]:.3f}')
PY
