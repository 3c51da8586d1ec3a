#!/bin/bash
# streamed gather (one launch per request, per-layer counters acquired by the attention):
# GPU parity suite, smoke, A/B bench lines (L8, M7 r=0.5, rank slice 8), compute-sanitizer
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/r02h_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02h_gpu_tests.log
tail -3 gpurun_out/r02h_gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02h_smoke.log 2>&1; tail -1 gpurun_out/r02h_smoke.log
OUT=gpurun_out/r02h_ab.jsonl; : > $OUT
for sg in 1 0; do
  for wl in "--workload L8" "--workload M7 --ratio 0.5" "--rank-slice 8" "--rank-slice 4" "--rank-slice 2"; do
    line=$(PCR_STREAM_GATHER=$sg timeout 300 python bench.py $wl --steps 20 --warmup 3 --no-cpu-baseline --no-target-point 2>/dev/null | tail -1)
    echo "{\"sg\": $sg, \"wl\": \"$wl\", \"line\": $line}" >> $OUT
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/r02h_ab.jsonl"):
    try: j = json.loads(l)
    except Exception: print("bad", l[:300]); continue
    b = j["line"]; ra = b["roofline_attn"]; e = b.get("e2e") or {}
    print(f'sg={j["sg"]} {j["wl"]:26s} ttft {b["ttft_ms"]:.3f} ld {b["gather_ms_per_layer"]*1e3:6.1f} us attn {b["attn_ms_per_layer"]*1e3:6.1f} us  launches {b["gpu_launches"]}  e2e {e.get("value", 0)/1e3:.1f}k tok/s  T* {b["ttft_over_t_star"]:.3f}')
PY
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "overlap_sync or host_io_matches_device_buffers or split_kv_edge" > gpurun_out/r02h_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/r02h_memcheck.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/r02h_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/r02h_synccheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/r02h_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/r02h_racecheck.log
