#!/bin/bash
# round 2: default bench line (L8 + the M7 r=0.5 north_star sub-record), reference arm, ncu launch
# list of the default command, ncu --set full of kv_gather (L8) and suffix_attn (M7 r=0.5)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python bench.py > gpurun_out/r02b_bench.jsonl 2> gpurun_out/r02b_bench.err; echo "bench rc=$?"
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02b_ref.jsonl 2> gpurun_out/r02b_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches_L8.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile-steps 1 --no-target-point > /dev/null 2> gpurun_out/r02b_ncu_launch.err; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kv_gather -s 40 -c 1 -o gpurun_out/r02b_prof_gather -f \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile-steps 1 --no-target-point > /dev/null 2> gpurun_out/r02b_ncu_gather.err; echo "ncu gather rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:suffix_attn -s 40 -c 1 -o gpurun_out/r02b_prof_attn_M7 -f \
    python bench.py --workload M7 --ratio 0.5 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile-steps 1 > /dev/null 2> gpurun_out/r02b_ncu_attn.err; echo "ncu attn rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"suffix_attn|combine|kv_append" -s 60 -c 3 -o gpurun_out/r02b_prof_attn_L8 -f \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile-steps 1 --no-target-point > /dev/null 2> gpurun_out/r02b_ncu_attn_l8.err; echo "ncu attn L8 rc=$?"
tail -c 3000 gpurun_out/r02b_bench.jsonl; tail -3 gpurun_out/r02b_bench.err; cat gpurun_out/r02b_ref.jsonl
