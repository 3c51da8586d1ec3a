#!/bin/bash
# Workload coverage: Z trace (W sweep, DRAM only / + SSD tier), f3 layer body, L70, T.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
OUT=gpurun_out/workloads.jsonl; [ -n "$APPEND" ] || : > $OUT
# SECTIONS (default all but zq): z zq ssd f3 l70 t
rm -f /tmp/pcr_ssd_tier.bin   # a leftover tier file from an interrupted run
df -h /tmp | tail -1 > gpurun_out/disk.txt
S=" ${SECTIONS:-z ssd f3 l70 t} "
if [[ $S == *" z "* ]]; then
for W in 0 4; do
  timeout 900 python bench.py --workload Z --window $W >> $OUT 2>> gpurun_out/workloads.err; echo "Z W=$W rc=$?"
done
fi
if [[ $S == *" zq "* ]]; then
# Poisson arrivals with the f3 layer body, so a prefix hit saves real recompute:
# PCR with W=4, with W=0, and the no-reuse baseline, all at the SAME arrival rates (rho x the
# W=4 run's mean service time).
ZQ="--workload Z --layer-body --requests ${ZQ_REQ:-300} --store-frac ${ZQ_STORE:-0.10}"
timeout 900 python bench.py $ZQ --window 4 --rho 0.5,0.8,0.95 >> $OUT 2>> gpurun_out/workloads.err; echo "Zq W=4 rc=$?"
SVC=$(tail -1 $OUT | python -c "import json,sys; print(json.loads(sys.stdin.read())['ttft_wall_ms_mean'])")
timeout 900 python bench.py $ZQ --window 0 --rho 0.5,0.8,0.95 --rho-service-ms $SVC >> $OUT 2>> gpurun_out/workloads.err; echo "Zq W=0 rc=$?"
timeout 900 python bench.py $ZQ --window 0 --no-reuse --rho 0.5,0.8,0.95 --rho-service-ms $SVC >> $OUT 2>> gpurun_out/workloads.err; echo "Zq no-reuse rc=$?"
fi
if [[ $S == *" ssd "* ]]; then
timeout 900 python bench.py --workload Z --window 4 --requests 300 --store-frac 0.03 --ssd-frac 0.25 >> $OUT 2>> gpurun_out/workloads.err; echo "Z ssd rc=$?"
timeout 900 python bench.py --workload Z --window 0 --requests 300 --store-frac 0.03 --ssd-frac 0.25 >> $OUT 2>> gpurun_out/workloads.err; echo "Z ssd W0 rc=$?"
fi
if [[ $S == *" f3 "* ]]; then
timeout 300 python bench.py --steps 10 --warmup 2 --no-e2e --no-cpu-baseline --layer-body >> $OUT 2>> gpurun_out/workloads.err; echo "f3 L8 rc=$?"
timeout 300 python bench.py --workload M7 --ratio 0.5 --steps 10 --warmup 2 --no-e2e --no-cpu-baseline --layer-body >> $OUT 2>> gpurun_out/workloads.err; echo "f3 M7 rc=$?"
timeout 300 python bench.py --workload M7 --ratio 1.0 --steps 10 --warmup 2 --no-e2e --no-cpu-baseline --layer-body >> $OUT 2>> gpurun_out/workloads.err; echo "f3 M7 r1 rc=$?"
fi
if [[ $S == *" l70 "* ]]; then
for r in 0.5 1.0; do
  timeout 600 python bench.py --workload L70 --ratio $r --steps 5 --warmup 2 --no-e2e --no-cpu-baseline >> $OUT 2>> gpurun_out/workloads.err; echo "L70 $r rc=$?"
done
fi
if [[ $S == *" t "* ]]; then
timeout 300 python bench.py --workload T --steps 20 --warmup 3 --no-e2e --no-cpu-baseline >> $OUT 2>> gpurun_out/workloads.err; echo "T rc=$?"
fi
python - <<'PY'
import json
for l in open("gpurun_out/workloads.jsonl"):
    j=json.loads(l)
    keep={k:j.get(k) for k in ("value","ttft_ms","ttft_ms_mean","ttft_ms_p95","ttft_wall_ms_mean","chunk_hit_ratio","gather_ms_per_layer","attn_ms_per_layer","tier_stats")}
    print(j["config"]["workload"][:110], json.dumps(keep))
    for pz in j.get("poisson", []):
        print("   rho %.2f: TTFT mean %.2f p95 %.2f p99 %.2f ms (queue+service), service %.2f, pending %.2f, hit %.3f" % (
            pz["rho"], pz["ttft_ms_mean"], pz["ttft_ms_p95"], pz["ttft_ms_p99"], pz["service_ms_mean"],
            pz["mean_pending"], pz["chunk_hit_ratio"]))
PY
tail -5 gpurun_out/workloads.err
