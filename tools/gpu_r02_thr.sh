#!/bin/bash
# split-KV CTA threshold 32 / 48 / 64 on the one-kv-head slices and the Z trace (P=8 per rank)
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
A="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
for T in 48 32 64 48; do
  echo "== PCR_SPLIT_MAX_CTAS=$T"
  PCR_NVCC_EXTRA="-DPCR_SPLIT_MAX_CTAS=$T" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; continue; }
  for r in 0.625 0.75 0.875; do timeout 400 python bench.py --workload M7 --ratio $r --rank-slice 8 $A 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('M7 r=$r P=8 ttft', round(j['ttft_ms'],3))"; done
  timeout 900 python bench.py --workload Z --rank-slice 8 --z-windows 4 --z-store-fracs 0.1 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    j=json.loads(l); print('Z P=8 W=4 ttft mean', round(j['ttft_ms_mean'],3), 'p95', round(j['ttft_ms_p95'],3))"
done
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
