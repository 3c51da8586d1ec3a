#!/bin/bash
# End-of-session check: full GPU parity, smoke, compute-sanitizer on the PDL launch chain
# (smoke: every kernel; split-KV parity cases: append -> attention -> combine under PDL).
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 240 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
S=gpurun_out/sanitizer_pdl.txt
echo "# compute-sanitizer with programmatic dependent launch on (default build)" > $S
for tool in memcheck racecheck initcheck synccheck; do
  echo "## $tool (python __graft_entry__.py smoke)" >> $S
  timeout 600 compute-sanitizer --tool $tool python __graft_entry__.py smoke 2>&1 | grep -E "smoke ok|SUMMARY" >> $S
done
for tool in memcheck synccheck; do
  echo "## $tool: pytest split_kv_edge_sweep + programmatic_dependent_launch" >> $S
  timeout 900 compute-sanitizer --tool $tool python -m pytest tests -m gpu -q -x -k "split_kv_edge or programmatic_dependent" 2>&1 | grep -E "passed|failed|SUMMARY" >> $S
done
cat $S
