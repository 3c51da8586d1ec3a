#!/bin/bash
# e2e host buffers: hugepage-registered vs torch pinned (alternating, 3 reps)
export PYTHONUNBUFFERED=1
for rep in 1 2 3; do for tp in 0 1; do
  PCR_BENCH_TORCH_PINNED=$tp timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-target-point 2>/dev/null | tail -1 | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('torch_pinned=$tp rep=$rep ttft %.3f e2e %.1fk' % (j['ttft_ms'], j['e2e']['value']/1e3))"
done; done
