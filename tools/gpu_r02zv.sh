#!/bin/bash
# dominant kernel by its own speed; b2b attention timing on every rank (shared-GPU N-rank check)
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02zv_$i.jsonl 2>/dev/null; python -c "
import json; j=json.loads(open('gpurun_out/r02zv_$i.jsonl').read().strip().splitlines()[-1]); r=j['roofline']
print('run $i', r['kernel'][:20], round(r['frac'],3), 'ttft', round(j['ttft_ms'],3), 'dev', round(j['ttft_device_ms'],3), 'e2e', round(j['e2e']['value']), 'attn own', round(j['roofline_attn']['isolated']['avg_launch_ms']*1e3,1))"; done
bash tools/gpu_r02o.sh
python -c "
import json
for P in (2, 8):
    j=json.loads(open(f'gpurun_out/r02o_share{P}.jsonl').read().strip().splitlines()[-1]); ra=j['roofline_attn']
    print(P, j['roofline']['kernel'][:20], 'isolated', ra.get('isolated'))"
