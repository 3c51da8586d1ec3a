mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
timeout 240 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 400 python bench.py > gpurun_out/bench_auto.json 2> gpurun_out/bench_auto.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_auto.err
OUT=gpurun_out/m7.jsonl; : > $OUT
for m in sm ce_runs; do for r in 0.5 0.75 1.0; do
timeout 300 python bench.py --workload M7 --ratio $r --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --load-mode $m >> $OUT 2>> gpurun_out/m7.err
done; done
python - <<'PY'
import json
for f in ["gpurun_out/bench_auto.json","gpurun_out/m7.jsonl"]:
    for l in open(f):
        j=json.loads(l)
        print(j["config"]["workload"][:3], j.get("pipeline"), "val %.0f ttft %.3f"%(j["value"], j["ttft_ms"]), "load %.1fus"%(j["gather_ms_per_layer"]*1e3), "attn %.1fus"%(j["attn_ms_per_layer"]*1e3), j["roofline"]["kernel"][:60], "frac %.3f"%j["roofline"]["frac"], j.get("load_path"), (j.get("roofline_gather_sm") or {}).get("frac"), (j.get("e2e") or {}).get("value"))
PY
