#!/bin/bash
# gather on the library's greatest-priority stream: regression test, full GPU suite, timeline script
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "default_priority" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
PCR_NVCC_EXTRA="-DPCR_ATTN_TIMELINE=1" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
for i in 1 2; do timeout 300 python tools/attn_timeline.py 2>&1 | cut -c1-700 | tail -4; done
PCR_BENCH_TIMELINE=1 timeout 300 python bench.py --workload M7 --ratio 0.5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep -E "tag|timeline_step|Error|error" | cut -c1-700
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
timeout 300 python bench.py --workload M7 --ratio 0.5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('M7 ttft', j['ttft_ms'], 'clk', j['clocks']['sm_mhz'])"
