#!/bin/bash
# mbarrier polling experiments: one thread checks K/V for tile 0 (PCR_KV_WAIT_ONE), lane-0 waits
# in the producer / MMA / softmax warps (PCR_LANE0_WAIT)
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
PYTEST_K="attention_and_pool or split_kv or self_consistency or page_size or l8_full or m7_half or fused_append or sharding or bitwise" \
  bash tools/gpu_variant.sh "" "-DPCR_KV_WAIT_ONE=1" "-DPCR_LANE0_WAIT=1" "-DPCR_KV_WAIT_ONE=1 -DPCR_LANE0_WAIT=1" 2>&1 | tee gpurun_out/r02z5_variant.txt
for F in "-DPCR_ATTN_TIMING=1 -DPCR_KV_WAIT_ONE=1 -DPCR_LANE0_WAIT=1"; do
  echo "== timing flags: $F"
  PCR_NVCC_EXTRA="$F" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; continue; }
  timeout 120 python tools/attn_bench.py --shape 4096,4224,32,8 --iters 1 2>&1 | grep -E "TIMING" | tail -22
done 2>&1 | tee gpurun_out/r02z5_timing.txt
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
