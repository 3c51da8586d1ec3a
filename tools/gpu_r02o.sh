#!/bin/bash
# functional check of the multi-rank bench path on ONE GPU (every rank on cuda:0, gloo control
# collectives; NCCL refuses two ranks per device so no output re-assembly): P = 2 and 8
export PYTHONUNBUFFERED=1
for P in 2 8; do
  PCR_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus $P --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02o_share$P.jsonl 2> gpurun_out/r02o_share$P.err; echo "share$P rc=$?"
  python -c "
import json; j=json.loads(open('gpurun_out/r02o_share$P.jsonl').read().strip().splitlines()[-1])
print('n_gpus', j['n_gpus'], 'ttft', round(j['ttft_ms'],3), 'e2e', j['e2e'] and round(j['e2e']['value']/1e3,1), 'h2d concurrent', j.get('h2d_peak_concurrent_gbs',{}).get('aggregate'), 'parallelism', j['config']['parallelism'], 'M7', j['north_star_point']['ttft_ms'])" 2>&1 | tail -2
  grep -iE "Error|Traceback" gpurun_out/r02o_share$P.err | head -5
done
