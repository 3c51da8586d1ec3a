#!/bin/bash
# f4 (the paper's fig:api analogue on B200): the a2 movers at L8, M7 r=0.5 and the P=8 rank slice --
# SM gather (streamed, and one launch per layer), copy engines with one cudaMemcpyAsync per merged
# run and per page image, TMA bulk copies -- each as a fraction of the live H2D peak
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r02m_f4.jsonl; : > $OUT
for wl in "--workload L8" "--workload M7 --ratio 0.5" "--rank-slice 8"; do
  for lm in "sm|1" "sm|0" "ce_runs|1" "ce_blocks|1" "tma|1"; do
    IFS='|' read m sg <<< "$lm"
    line=$(PCR_STREAM_GATHER=$sg timeout 300 python bench.py $wl --load-mode $m --steps 15 --warmup 3 --no-e2e --no-cpu-baseline --no-target-point 2>/dev/null | tail -1)
    echo "{\"wl\": \"$wl\", \"mover\": \"$m\", \"streamed\": $sg, \"line\": $line}" >> $OUT
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/r02m_f4.jsonl"):
    try: j = json.loads(l)
    except Exception: print("bad", l[:200]); continue
    b = j["line"]; r = b["roofline_gather"]
    print(f'{j["wl"]:26s} {j["mover"]:9s} streamed={j["streamed"]} ttft {b["ttft_ms"]:7.3f} load/layer {b["gather_ms_per_layer"]*1e3:6.1f} us  {r["achieved"]:5.1f} GB/s = {r["frac"]:.3f} of {r["peak"]:.1f}  launches {b["gpu_launches"]}')
PY
