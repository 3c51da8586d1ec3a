#!/bin/bash
# e2e (host_io) A/B: streamed gather vs per-layer gathers, 3 repetitions each, alternating
export PYTHONUNBUFFERED=1
for rep in 1 2 3; do for sg in 1 0; do
  PCR_STREAM_GATHER=$sg timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-target-point 2>/dev/null | tail -1 | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('sg=$sg rep=$rep ttft %.3f e2e %.1fk' % (j['ttft_ms'], j['e2e']['value']/1e3), j['clocks']['sm_mhz'])"
done; done
