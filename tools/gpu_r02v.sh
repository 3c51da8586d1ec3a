#!/bin/bash
# in-kernel split reduce through L2: parity suite, short-suffix attention A/B, L8 / P=8 lines
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/r02v_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02v_gpu_tests.log; tail -3 gpurun_out/r02v_gpu_tests.log
for sp in 1 0 1 0; do echo "== PCR_SPLIT_SPIN=$sp"; PCR_SPLIT_SPIN=$sp timeout 300 python tools/attn_bench.py --small --iters 40 2>&1 | cut -c1-150; done
for sp in 1 0; do for wl in "--workload L8" "--rank-slice 8"; do
  PCR_SPLIT_SPIN=$sp timeout 300 python bench.py $wl --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-target-point 2>/dev/null | tail -1 | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('spin=$sp $wl ttft %.3f iso attn %.1f us launches %d' % (j['ttft_ms'], j['roofline_attn']['isolated']['avg_launch_ms']*1e3, j['gpu_launches']))"
done; done
