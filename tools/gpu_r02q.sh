#!/bin/bash
# after the split producer: full GPU parity, default bench line, attention microbench, a re-tune
# sweep of the exponential split and the exp ping-pong, and the per-phase clocks
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/r02q_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02q_gpu_tests.log; tail -2 gpurun_out/r02q_gpu_tests.log
timeout 600 python bench.py > gpurun_out/r02q_bench.jsonl 2> gpurun_out/r02q_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
j = json.loads(open("gpurun_out/r02q_bench.jsonl").read().strip().splitlines()[-1]); ns = j["north_star_point"]
print(f'L8 ttft {j["ttft_ms"]:.3f} gather frac {j["roofline"]["frac"]:.3f} e2e {j["e2e"]["value"]/1e3:.1f}k attn iso {j["roofline_attn"]["isolated"]["achieved"]:.0f} TF/s | M7 ttft {ns["ttft_ms"]:.2f} load {ns["load_frac_of_h2d_peak"]:.3f} attn {ns["attn_frac_of_bf16_peak"]:.3f} hidden {ns["hidden_load_pct"]:.1f} T* {ns["ttft_over_t_star"]:.3f} clk {ns["clocks"]["sm_mhz"]} {ns["clocks"]["reasons"]}')
PY
timeout 300 python tools/attn_bench.py > gpurun_out/r02q_attn.jsonl 2>&1; timeout 300 python tools/attn_bench.py --small >> gpurun_out/r02q_attn.jsonl 2>&1; cut -c1-150 gpurun_out/r02q_attn.jsonl
PYTEST_K=l8_full bash tools/gpu_variant.sh "-DPCR_POLY_PAIRS=0" "-DPCR_POLY_PAIRS=2" "-DPCR_POLY_PAIRS=4" "-DPCR_EXP_PINGPONG=0" "" 2>&1 | grep -E "flags|tflops|passed|failed" | cut -c1-150
PCR_NVCC_EXTRA="-DPCR_ATTN_TIMING=1" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1
timeout 300 python tools/attn_bench.py --shape 4096,4224,32,8 --iters 1 > gpurun_out/r02q_timing.txt 2>&1
grep -E "TIMING blk 300 " gpurun_out/r02q_timing.txt | head -10
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
