#!/bin/bash
# re-tune with the fixed producers: polynomial exp2 pairs and K/V ring depth (Q0 in TMEM frees 32 KB)
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
ATTN_BENCH_ARGS="--iters 20" PYTEST_K="attention_and_pool and iid or split_kv or m7_half or fused_append" \
  bash tools/gpu_variant.sh "" "-DPCR_POLY_PAIRS=0" "-DPCR_POLY_PAIRS=2" "-DPCR_POLY_PAIRS=3" "-DPCR_KV_STAGES=5" "" 2>&1
