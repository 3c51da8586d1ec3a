#!/bin/bash
# cluster split-KV reduce: active-cluster occupancy table and cluster-size caps (attention microbench)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for cap in 16 8 4 2; do
  echo "== cap $cap"; PCR_DEBUG=1 PCR_MAX_CLUSTER=$cap timeout 300 python tools/attn_bench.py --small --iters 40 2>&1 | cut -c1-200
done
echo "== workspace + combine"; PCR_SPLIT_CLUSTER=0 timeout 300 python tools/attn_bench.py --small --iters 40 2>&1 | cut -c1-200
