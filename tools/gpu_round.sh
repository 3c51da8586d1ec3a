#!/bin/bash
# Round artifacts: parity, the default bench line, the reference arm, load-path and hit-ratio
# sweeps, the ncu launch list and full captures of the two dominant kernels.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; rc=$?; echo "pytest rc=$rc" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
if [ $rc -ne 0 ]; then grep -E "Error|assert|FAILED" gpurun_out/gpu_tests.log | head -20; exit 1; fi
timeout 240 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
OUT=gpurun_out/modes.jsonl; : > $OUT
for m in sm ce_runs ce_blocks tma; do
  timeout 200 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --load-mode $m >> $OUT 2>> gpurun_out/modes.err
  timeout 300 python bench.py --workload M7 --ratio 0.5 --steps 10 --warmup 2 --no-e2e --no-cpu-baseline --load-mode $m >> $OUT 2>> gpurun_out/modes.err
done
timeout 200 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --mode sync >> $OUT 2>> gpurun_out/modes.err
for r in 0.0 0.25 0.5 0.75 1.0; do
  timeout 300 python bench.py --workload M7 --ratio $r --steps 10 --warmup 2 --no-e2e --no-cpu-baseline >> $OUT 2>> gpurun_out/modes.err
  timeout 300 python bench.py --workload M7 --ratio $r --steps 10 --warmup 2 --no-e2e --no-cpu-baseline --mode sync >> $OUT 2>> gpurun_out/modes.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_L8.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile-steps 1 > /dev/null 2> gpurun_out/ncu_launch.err; echo "ncu launches rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_L8_sm.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile-steps 1 --load-mode sm > /dev/null 2>> gpurun_out/ncu_launch.err; echo "ncu launches sm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kv_gather -s 40 -c 1 -o gpurun_out/prof_gather -f \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile-steps 1 --load-mode sm > /dev/null 2> gpurun_out/ncu_gather.err; echo "ncu gather rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:suffix_attn -s 40 -c 1 -o gpurun_out/prof_attn_M7 -f \
    python bench.py --workload M7 --ratio 0.5 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile-steps 1 > /dev/null 2> gpurun_out/ncu_attn.err; echo "ncu attn rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:suffix_attn -s 6 -c 1 -o gpurun_out/prof_attn_micro -f \
    python tools/attn_bench.py --iters 1 > /dev/null 2> gpurun_out/ncu_attn_micro.err; echo "ncu attn micro rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/modes.jsonl"):
    j=json.loads(l)
    print(j["config"]["workload"][:40], j.get("pipeline"), "ttft %.2f"%j["ttft_ms"], "load/layer %.1fus"%(j["gather_ms_per_layer"]*1e3), "attn/layer %.1fus %.0f TF/s (%.1f%%)"%(j["attn_ms_per_layer"]*1e3, j["roofline_attn"]["achieved"], 100*j["roofline_attn"]["frac"]))
PY
cat gpurun_out/bench_default.json
timeout 300 python tools/attn_bench.py > gpurun_out/attn_micro.jsonl 2> gpurun_out/attn_micro.err; cat gpurun_out/attn_micro.jsonl
