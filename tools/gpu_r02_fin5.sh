#!/bin/bash
# FINAL round-2 measurements, fifth pass (fused-append placement per launch, split-KV below 48 CTAs; dominant kernel by own speed, e2e warm-up step, device TTFT; split-KV sizing on 136 SMs, whole-pool smoke; producer fix, TMA epilogue, Q0 in TMEM, priority gather stream):
# GPU parity + smoke, default line x3, reference arm, sweeps, attention microbench + yardstick, ncu
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 1500 python -m pytest tests -m gpu -q -x -rA > gpurun_out/r02z_fin5_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02z_fin5_gpu_tests.log
grep -E "passed|failed|L8 full|layer-body" gpurun_out/r02z_fin5_gpu_tests.log | tail -3
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02z_fin5_smoke.log 2>&1; tail -1 gpurun_out/r02z_fin5_smoke.log
: > gpurun_out/r02z_fin5_bench.jsonl
for i in 1 2 3; do timeout 600 python bench.py >> gpurun_out/r02z_fin5_bench.jsonl 2>> gpurun_out/r02z_fin5_bench.err; done
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02z_fin5_ref.jsonl 2> gpurun_out/r02z_fin5_ref.err
OUT=gpurun_out/r02z_fin5_sweeps.jsonl; : > $OUT
for P in 2 4 8; do timeout 300 python bench.py --rank-slice $P --steps 20 --warmup 3 --no-cpu-baseline --no-target-point >> $OUT 2>> gpurun_out/r02z_fin5_sweeps.err; done
for r in 0.0 0.25 0.5 0.75 1.0; do
  timeout 300 python bench.py --workload M7 --ratio $r --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> $OUT 2>> gpurun_out/r02z_fin5_sweeps.err
done
for r in 0.0 0.25 0.5 0.75 1.0; do
  timeout 300 python bench.py --workload M7 --ratio $r --rank-slice 8 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> $OUT 2>> gpurun_out/r02z_fin5_sweeps.err
done
for r in 0.5 0.75 0.875 1.0; do
  timeout 600 python bench.py --workload L70 --rank-slice 8 --ratio $r --steps 5 --warmup 2 --no-e2e --no-cpu-baseline >> $OUT 2>> gpurun_out/r02z_fin5_sweeps.err
done
timeout 300 python tools/attn_bench.py > gpurun_out/r02z_fin5_attn.jsonl 2>&1; timeout 300 python tools/attn_bench.py --small >> gpurun_out/r02z_fin5_attn.jsonl 2>&1
timeout 900 python tools/attn_yardstick.py 2>&1 | grep -v Warning > gpurun_out/r02z_fin5_yardstick.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02z_fin5_launches_L8.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile-steps 1 --no-target-point > /dev/null 2> gpurun_out/r02z_fin5_ncu_launch.err; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:suffix_attn -s 40 -c 1 -o gpurun_out/r02z_fin5_prof_attn_M7 -f \
    python bench.py --workload M7 --ratio 0.5 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile-steps 1 > /dev/null 2> gpurun_out/r02z_fin5_ncu_attn.err; echo "ncu attn rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kv_gather_stream -s 3 -c 1 -o gpurun_out/r02z_fin5_prof_gather -f \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile-steps 1 --no-target-point > /dev/null 2> gpurun_out/r02z_fin5_ncu_gather.err; echo "ncu gather rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"suffix_attn|combine" -s 60 -c 2 -o gpurun_out/r02z_fin5_prof_attn_L8 -f \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile-steps 1 --no-target-point > /dev/null 2> gpurun_out/r02z_fin5_ncu_attn_l8.err; echo "ncu attn L8 rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r02z_fin5_bench.jsonl"):
    j = json.loads(l); ns = j["north_star_point"]
    print(f'{j["roofline"]["kernel"][:9]} L8 ttft {j["ttft_ms"]:.3f} dev {j["ttft_device_ms"]:.3f} value {j["value"]/1e3:.1f}k gather {j["roofline"]["frac"]:.3f} e2e {j["e2e"]["value"]/1e3:.1f}k attn-own {j["roofline_attn"]["isolated"]["avg_launch_ms"]*1e3:.1f} us clk {j["clocks"]["sm_mhz"]} | M7 ttft {ns["ttft_ms"]:.2f} load {ns["load_frac_of_h2d_peak"]:.3f} attn {ns["attn_frac_of_bf16_peak"]:.3f} hidden {ns["hidden_load_pct"]:.1f} T* {ns["ttft_over_t_star"]:.3f} clk {ns["clocks"]["sm_mhz"]}')
for l in open("gpurun_out/r02z_fin5_sweeps.jsonl"):
    try: j = json.loads(l)
    except Exception: continue
    ra = j["roofline_attn"]; rg = j["roofline_gather"]; iso = ra["isolated"]["achieved"] if ra and ra.get("isolated") else 0
    print(f'{j["config"]["workload"][:58]:58s} {j["config"]["parallelism"][:22]:22s} ttft {j["ttft_ms"]:8.3f} ld {j["gather_ms_per_layer"]*1e3:6.1f} us ({rg["frac"]:.3f}) attn iso {iso:5.0f} TF/s T* {j["ttft_over_t_star"] or 0:.3f} e2e {(j.get("e2e") or {}).get("value", 0)/1e3:.0f}k clk {j["clocks"]["sm_mhz"]}')
PY
cut -c1-170 gpurun_out/r02z_fin5_attn.jsonl; cut -c1-200 gpurun_out/r02z_fin5_yardstick.jsonl | grep -v error
