#!/bin/bash
# Bench + profiles on one B200: bench lines, the ncu launch list and full captures of the two kernels.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_L8.json 2> gpurun_out/bench_L8.err; echo "bench rc=$?"
timeout 300 python bench.py --workload M7 --ratio 0.5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_M7_r05.json 2> gpurun_out/bench_M7.err; echo "bench M7 rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_L8.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_launch.err; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kv_gather -s 40 -c 1 -o gpurun_out/prof_gather -f \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_gather.err; echo "ncu gather rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:suffix_attn -s 40 -c 1 -o gpurun_out/prof_attn_L8 -f \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_attn.err; echo "ncu attn rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:suffix_attn -s 40 -c 1 -o gpurun_out/prof_attn_M7 -f \
    python bench.py --workload M7 --ratio 0.5 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_attn_m7.err; echo "ncu attn M7 rc=$?"
cat gpurun_out/bench_L8.json gpurun_out/bench_M7_r05.json gpurun_out/bench_ref.json
tail -3 gpurun_out/bench_L8.err
