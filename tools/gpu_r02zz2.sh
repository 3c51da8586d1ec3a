#!/bin/bash
# fused append by the owning CTA vs the last M-block, tail stores waited for reads only:
# multi-wave (M7 P=1), single-wave (M7 r=0.5 P=8 slice: one kv head, 2 splits) and short suffix
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for F in "-DPCR_APPEND_OWNER=1" "" "-DPCR_APPEND_OWNER=1" ""; do
  echo "== flags: $F"
  PCR_NVCC_EXTRA="$F" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; continue; }
  timeout 600 python -m pytest tests -m gpu -q -x -k "fused_append or attention_and_pool and iid or split_kv or bench_north" 2>&1 | tail -1
  for SH in 4096,4224,32,8 4096,4224,4,1 0,8320,32,8 4096,128,32,8 8192,8320,8,1; do timeout 300 python tools/attn_bench.py --shape $SH --iters 10 2>&1 | tail -1 | cut -c1-160; done
done
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
