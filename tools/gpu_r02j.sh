#!/bin/bash
# round 2 artifacts on the current build: GPU parity, smoke, default bench line x3 (repeatability),
# reference arm, ncu launch list of the default command, ncu --set full of the streamed gather
# (L8) and of suffix_attn (M7 r=0.5 and L8), the attention microbenchmark
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x -rA > gpurun_out/r02j_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02j_gpu_tests.log
grep -E "passed|failed|L8 full" gpurun_out/r02j_gpu_tests.log | tail -3
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02j_smoke.log 2>&1; tail -1 gpurun_out/r02j_smoke.log
: > gpurun_out/r02j_bench.jsonl
for i in 1 2 3; do timeout 600 python bench.py >> gpurun_out/r02j_bench.jsonl 2>> gpurun_out/r02j_bench.err; echo "bench $i rc=$?"; done
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02j_ref.jsonl 2> gpurun_out/r02j_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02j_launches_L8.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile-steps 1 --no-target-point > /dev/null 2> gpurun_out/r02j_ncu_launch.err; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kv_gather_stream -s 3 -c 1 -o gpurun_out/r02j_prof_gather -f \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile-steps 1 --no-target-point > /dev/null 2> gpurun_out/r02j_ncu_gather.err; echo "ncu gather rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:suffix_attn -s 40 -c 1 -o gpurun_out/r02j_prof_attn_M7 -f \
    python bench.py --workload M7 --ratio 0.5 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile-steps 1 > /dev/null 2> gpurun_out/r02j_ncu_attn.err; echo "ncu attn rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"suffix_attn|combine" -s 60 -c 2 -o gpurun_out/r02j_prof_attn_L8 -f \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile-steps 1 --no-target-point > /dev/null 2> gpurun_out/r02j_ncu_attn_l8.err; echo "ncu attn L8 rc=$?"
timeout 300 python tools/attn_bench.py > gpurun_out/r02j_attn_micro.jsonl 2>&1; timeout 300 python tools/attn_bench.py --small >> gpurun_out/r02j_attn_micro.jsonl 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/r02j_bench.jsonl"):
    j = json.loads(l); ns = j["north_star_point"]
    print(f'L8 ttft {j["ttft_ms"]:.3f} value {j["value"]/1e3:.1f}k gather {j["roofline"]["achieved"]:.1f} GB/s frac {j["roofline"]["frac"]:.3f} e2e {j["e2e"]["value"]/1e3:.1f}k T* {j["ttft_over_t_star"]:.3f} clk {j["clocks"]["sm_mhz"]} {j["clocks"]["reasons"]} | M7 ttft {ns["ttft_ms"]:.2f} load {ns["load_frac_of_h2d_peak"]:.3f} attn {ns["attn_frac_of_bf16_peak"]:.3f} hidden {ns["hidden_load_pct"]:.1f} T* {ns["ttft_over_t_star"]:.3f}')
PY
cat gpurun_out/r02j_attn_micro.jsonl | cut -c1-160
