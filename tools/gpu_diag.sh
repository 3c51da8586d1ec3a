#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
free -g | head -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:suffix_attn -s 8 -c 1 -o gpurun_out/prof_attn_v2e -f \
   python tools/attn_bench.py --iters 2 > gpurun_out/ncu_attn_v2e.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_attn_v2e.log
timeout 600 python bench.py --workload Z --window 4 --requests 300 --store-frac 0.03 --ssd-frac 0.10 > gpurun_out/z_ssd.json 2> gpurun_out/z_ssd.err; echo "zssd rc=$?"; tail -20 gpurun_out/z_ssd.err; cat gpurun_out/z_ssd.json | cut -c1-600
timeout 600 python bench.py --workload L70 --ratio 0.5 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/l70.json 2> gpurun_out/l70.err; echo "l70 rc=$?"; tail -20 gpurun_out/l70.err; cut -c1-400 gpurun_out/l70.json
timeout 300 python bench.py --steps 10 --warmup 2 --no-e2e --no-cpu-baseline --layer-body > gpurun_out/f3l8.json 2> gpurun_out/f3l8.err; echo "f3 rc=$?"; tail -20 gpurun_out/f3l8.err; cut -c1-400 gpurun_out/f3l8.json
