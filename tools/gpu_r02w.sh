#!/bin/bash
# late PDL wait: parity suite, short-suffix A/B (PCR_LATE_DEP_WAIT), compute-sanitizer synccheck/racecheck
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/r02w_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02w_gpu_tests.log; tail -3 gpurun_out/r02w_gpu_tests.log
for v in 1 0 1 0; do echo "== PCR_LATE_DEP_WAIT=$v"; PCR_LATE_DEP_WAIT=$v timeout 300 python tools/attn_bench.py --small --iters 40 2>&1 | cut -c1-150; done
PCR_LATE_DEP_WAIT=1 timeout 300 python tools/attn_bench.py --iters 20 2>&1 | cut -c1-150
for v in 1 0; do for wl in "--workload L8" "--rank-slice 8"; do
  PCR_LATE_DEP_WAIT=$v timeout 300 python bench.py $wl --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-target-point 2>/dev/null | tail -1 | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('late=$v $wl ttft %.3f iso attn %.1f us' % (j['ttft_ms'], j['roofline_attn']['isolated']['avg_launch_ms']*1e3))"
done; done
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "overlap_sync or split_kv_edge" > gpurun_out/r02w_sync.log 2>&1; echo "synccheck rc=$?"; tail -1 gpurun_out/r02w_sync.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "overlap_sync" > gpurun_out/r02w_race.log 2>&1; echo "racecheck rc=$?"; tail -1 gpurun_out/r02w_race.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "overlap_sync or split_kv_edge or host_io" > gpurun_out/r02w_mem.log 2>&1; echo "memcheck rc=$?"; tail -1 gpurun_out/r02w_mem.log
