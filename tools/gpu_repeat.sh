#!/bin/bash
# Run-to-run spread of the headline numbers on one box: 5 x L8 default bench, 5 x M7 r=0.5.
mkdir -p gpurun_out
OUT=gpurun_out/repeat.jsonl; : > $OUT
for i in 1 2 3 4 5; do
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline >> $OUT 2>/dev/null
  timeout 300 python bench.py --workload M7 --ratio 0.5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> $OUT 2>/dev/null
done
python - <<'PY'
import json, statistics as st
rows = [json.loads(l) for l in open("gpurun_out/repeat.jsonl")]
for wl in ("L8", "M7"):
    r = [j for j in rows if j["config"]["workload"].startswith(wl)]
    tt = [j["ttft_ms"] for j in r]; v = [j["value"] for j in r]
    fr = [j["roofline"]["frac"] for j in r]; at = [j["roofline_attn"]["achieved"] for j in r]
    print(wl, "n=%d ttft %.3f +- %.3f ms, value %.0f +- %.0f tok/s, load frac %.3f +- %.3f, attn %.0f +- %.0f TF/s"
          % (len(r), st.mean(tt), st.pstdev(tt), st.mean(v), st.pstdev(v), st.mean(fr), st.pstdev(fr), st.mean(at), st.pstdev(at)))
PY
