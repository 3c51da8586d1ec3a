#!/bin/bash
# which side bounds the attention at the M7 r=0.5 shape: PCR_ATTN_PROFILE bit masks
# (1 skip softmax arithmetic, 2 skip MMAs, 4 skip K/V TMA loads, 8 MMA warp does not wait for P)
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for F in "" "-DPCR_ATTN_PROFILE=4" "-DPCR_ATTN_PROFILE=1" "-DPCR_ATTN_PROFILE=5" "-DPCR_ATTN_PROFILE=2" "-DPCR_ATTN_PROFILE=8" "-DPCR_ATTN_PROFILE=12"; do
  PCR_NVCC_EXTRA="$F" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || { tail -3 gpurun_out/build.log; continue; }
  echo "== $F"; timeout 300 python tools/attn_bench.py --shape 4096,4224,32,8 --iters 20 2>&1 | tail -1 | cut -c1-160
done
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
