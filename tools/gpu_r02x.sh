#!/bin/bash
# late PDL wait on the long shapes (tail wave of layer l overlapped by layer l+1) and the M7 line
export PYTHONUNBUFFERED=1
for v in 1 0 1 0; do echo "== PCR_LATE_DEP_WAIT=$v"; PCR_LATE_DEP_WAIT=$v timeout 300 python tools/attn_bench.py --iters 20 2>&1 | grep -v '"n2": 128' | cut -c1-150; done
for v in 1 0 1 0; do
  PCR_LATE_DEP_WAIT=$v timeout 300 python bench.py --workload M7 --ratio 0.5 --steps 15 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('late=$v M7 r=0.5 ttft %.3f attn/layer %.1f us (%.0f TF/s) clk %s' % (j['ttft_ms'], j['attn_ms_per_layer']*1e3, j['roofline_attn']['achieved'], j['clocks']['sm_mhz']))"
done
