#!/bin/bash
# per-phase clocks of the attention's softmax warps (PCR_ATTN_TIMING build) at the M7 r=0.5 shape,
# then the default build: the f3 layer-body reuse == full recompute test
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
PCR_NVCC_EXTRA="-DPCR_ATTN_TIMING=1" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 300 python tools/attn_bench.py --shape 4096,4224,32,8 --iters 1 > gpurun_out/r02k_timing.txt 2>&1
grep -E "TIMING|MMATIMING" gpurun_out/r02k_timing.txt | sort | uniq -c | sort -rn | head -5
grep -E "TIMING blk 0 |MMATIMING blk 0" gpurun_out/r02k_timing.txt | head -12
grep -E "TIMING blk 300 |MMATIMING blk 300" gpurun_out/r02k_timing.txt | head -12
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "layer_body" -s 2>&1 | tail -4
