#!/bin/bash
# round 2: fused append + cluster split-KV reduce -- GPU parity suite, attention microbench A/B,
# default bench, rank-slice P=8 line, h2d probe variants
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/r02c_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02c_gpu_tests.log
tail -4 gpurun_out/r02c_gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02c_smoke.log 2>&1; tail -1 gpurun_out/r02c_smoke.log
for v in "1 1" "0 0" "0 1" "1 0"; do set -- $v
  PCR_FUSED_APPEND=$1 PCR_SPLIT_CLUSTER=$2 timeout 300 python tools/attn_bench.py > gpurun_out/r02c_attn_f$1_c$2.jsonl 2>&1; echo "attn f$1 c$2 rc=$?"
  PCR_FUSED_APPEND=$1 PCR_SPLIT_CLUSTER=$2 timeout 300 python tools/attn_bench.py --small >> gpurun_out/r02c_attn_f$1_c$2.jsonl 2>&1
done
timeout 600 python bench.py > gpurun_out/r02c_bench.jsonl 2> gpurun_out/r02c_bench.err; echo "bench rc=$?"
timeout 300 python bench.py --rank-slice 8 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-target-point > gpurun_out/r02c_rankslice8.jsonl 2>&1; echo "rs8 rc=$?"
PCR_FUSED_APPEND=0 PCR_SPLIT_CLUSTER=0 timeout 300 python bench.py --rank-slice 8 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-target-point > gpurun_out/r02c_rankslice8_old.jsonl 2>&1; echo "rs8 old rc=$?"
timeout 120 ./tools/h2d_probe2 > gpurun_out/r02c_h2d_probe2.txt 2>&1; echo "probe rc=$?"
cat gpurun_out/r02c_h2d_probe2.txt
for f in gpurun_out/r02c_attn_*.jsonl; do echo $f; cat $f | cut -c1-300; done
