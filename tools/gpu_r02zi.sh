#!/bin/bash
# TMA-store epilogue: wait for the staging reads only (default) vs full completion
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
ATTN_BENCH_ARGS="--small" PYTEST_K="attention_and_pool or split_kv or self_consistency or l8_full or m7_half or fused_append or context_split or bitwise" \
  bash tools/gpu_variant.sh "" "-DPCR_EPI_WAIT_READ=0" "" "-DPCR_EPI_WAIT_READ=0" 2>&1
timeout 300 python tools/attn_bench.py --shape 4096,4224,32,8 2>&1 | tail -1
