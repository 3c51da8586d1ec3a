#!/bin/bash
# L8 P=8 slice attention: tail stores waited for reads (default) vs full completion; alternating
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for F in "" "-DPCR_TAIL_WAIT_FULL=1" "" "-DPCR_TAIL_WAIT_FULL=1"; do
  echo "== flags: $F"
  PCR_NVCC_EXTRA="$F" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; continue; }
  for SH in 4096,128,4,1 4096,128,32,8; do timeout 300 python tools/attn_bench.py --shape $SH --iters 20 2>&1 | tail -1 | cut -c1-150; done
  timeout 400 python bench.py --rank-slice 8 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('L8 P=8 ttft', round(j['ttft_ms'],3), 'own us', round(j['roofline_attn']['isolated']['avg_launch_ms']*1e3,1))"
done
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
