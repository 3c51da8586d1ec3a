#!/bin/bash
# e2e across consecutive bench processes on one box, with the host buffers' huge-page coverage
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for i in 1 2 3 4; do
  timeout 600 python bench.py --no-cpu-baseline --no-target-point > gpurun_out/r02zt_$i.jsonl 2>/dev/null
  python -c "
import json; j=json.loads(open('gpurun_out/r02zt_$i.jsonl').read().strip().splitlines()[-1]); e=j['e2e']
print('run $i ttft', round(j['ttft_ms'],3), 'e2e', round(e['value']), 'huge', e.get('host_hugepage_frac'), 'steps', e.get('step_ms'))"
  grep -E "AnonHugePages|MemFree|MemAvailable" /proc/meminfo | tr '\n' ' '; echo
done
cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag
