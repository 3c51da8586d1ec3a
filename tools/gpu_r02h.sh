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
# Z with the SSD tier under Poisson arrivals at ONE arrival rate for every W (rate = rho / 5.05 ms,
# the W>=2 saturated service time): what the look-ahead prefetch buys at equal load
mkdir -p gpurun_out/z_plans_fixed
timeout 1500 python bench.py --workload Z --rank-slice 8 --z-windows 0,2,4,6,8 --z-store-fracs 0.1 --ssd-frac 0.5 \
    --ssd-path /tmp/pcr_ssd_tier.bin --rho 0.5,0.8 --rho-service-ms 5.05 --z-log gpurun_out/z_plans_fixed \
    > gpurun_out/r02h_z_fixed.jsonl 2> gpurun_out/r02h_z_fixed.err; echo "z fixed-rate rc=$?"
rm -f /tmp/pcr_ssd_tier.bin
python - <<'PY'
import json
for l in open("gpurun_out/r02h_z_fixed.jsonl"):
    try: j = json.loads(l)
    except Exception: continue
    c = j["config"]
    print(f'W={c["window"]}: sat wall {j["ttft_wall_ms_mean"]:.2f} ms', " | ".join(f'rho {p["rho"]}: mean {p["ttft_ms_mean"]:.1f} p95 {p["ttft_ms_p95"]:.1f} svc {p["service_ms_mean"]:.2f} pend {p["mean_pending"]:.2f}' for p in j.get("poisson", [])))
PY
