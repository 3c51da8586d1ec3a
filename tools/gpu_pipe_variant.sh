#!/bin/bash
# Kernel variant under compile-time flags, measured inside the pipeline: gpu_pipe_variant.sh
# "-DA=1" ... ("" = default build): attention parity subset, then M7 bench lines (attention
# beside the next layer's load).  Restores the default build.
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
OUT=gpurun_out/pipe_variant.jsonl; : > $OUT
for rep in 1 2; do
for F in "$@"; do
  echo "== flags: $F"
  PCR_NVCC_EXTRA="$F" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; continue; }
  [ $rep = 1 ] && timeout 600 python -m pytest tests -m gpu -q -x -k "${PYTEST_K:-attention_and_pool or split_kv or m7_half}" 2>&1 | tail -2
  for r in ${RATIOS:-0.5 0.25}; do
    timeout 300 python bench.py --workload M7 --ratio $r --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
      | sed "s/^{/{\"flags\": \"$F\", /" >> $OUT 2>> gpurun_out/pipe_variant.err
  done
done
done
python - <<'PY'
import json
for l in open("gpurun_out/pipe_variant.jsonl"):
    try: j = json.loads(l)
    except Exception: continue
    print(repr(j["flags"]), j["config"]["workload"][40:75], "ttft %.3f" % j["ttft_ms"],
          "attn/layer %.1fus" % (j["attn_ms_per_layer"] * 1e3),
          "iso %.1fus" % (j["roofline_attn"]["isolated"]["avg_launch_ms"] * 1e3), "mhz", j["clocks"]["sm_mhz"])
PY
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
