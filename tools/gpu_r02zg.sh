#!/bin/bash
# Q tile 0 in TMEM as the default: full GPU suite, attention microbench, compute-sanitizer
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python tools/attn_bench.py 2>&1 | tail -5
timeout 300 python tools/attn_bench.py --small 2>&1 | tail -5
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/r02zg_$tool.log 2>&1; echo "$tool smoke rc=$?"; tail -1 gpurun_out/r02zg_$tool.log
done
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "overlap_sync or host_io_matches_device_buffers or split_kv_edge or offload_third_stream or layer_body or context_split_partials" > gpurun_out/r02zg_memcheck_tests.log 2>&1; echo "memcheck tests rc=$?"; tail -2 gpurun_out/r02zg_memcheck_tests.log
timeout 1200 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "overlap_sync or split_kv_edge" > gpurun_out/r02zg_synccheck_tests.log 2>&1; echo "synccheck tests rc=$?"; tail -2 gpurun_out/r02zg_synccheck_tests.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "overlap_sync" > gpurun_out/r02zg_racecheck_tests.log 2>&1; echo "racecheck tests rc=$?"; tail -2 gpurun_out/r02zg_racecheck_tests.log
