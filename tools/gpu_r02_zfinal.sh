#!/bin/bash
# final build: the driver's exact round-end commands timed, then the preset Z sweep (W x store, SSD tier
# with Poisson passes at one rate, P = 1), plan logs for the oracle replay
mkdir -p gpurun_out/z3
export PYTHONUNBUFFERED=1
s=$(date +%s.%N); python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02zf_ref.jsonl 2> gpurun_out/r02zf_ref.err; echo "ref rc=$? $(echo "$(date +%s.%N) - $s" | bc) s"
s=$(date +%s.%N); python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02zf_bench.jsonl 2> gpurun_out/r02zf_bench.err; echo "bench rc=$? $(echo "$(date +%s.%N) - $s" | bc) s"
s=$(date +%s.%N); python3 -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02zf_smoke.log 2>&1; echo "smoke rc=$? $(echo "$(date +%s.%N) - $s" | bc) s"; tail -1 gpurun_out/r02zf_smoke.log
OUT=gpurun_out/r02zf_z.jsonl; : > $OUT
timeout 1200 python bench.py --workload Z --rank-slice 8 --z-windows 0,2,4,6,8 --z-store-fracs 0.1,0.25,0.5 --z-log gpurun_out/z3 >> $OUT 2> gpurun_out/r02zf_z1.err; echo "dram rc=$?"
timeout 1500 python bench.py --workload Z --rank-slice 8 --z-windows 0,2,4,6,8 --z-store-fracs 0.1 --ssd-frac 0.5 \
    --ssd-path /tmp/pcr_ssd_tier.bin --rho 0.5,0.8 --rho-service-ms 5.05 --z-log gpurun_out/z3 >> $OUT 2> gpurun_out/r02zf_z2.err; echo "ssd rc=$?"
rm -f /tmp/pcr_ssd_tier.bin
timeout 1200 python bench.py --workload Z --z-windows 0,2,4,6,8 --z-store-fracs 0.1 --z-log gpurun_out/z3 >> $OUT 2> gpurun_out/r02zf_z3.err; echo "P1 rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r02zf_z.jsonl"):
    try: j = json.loads(l)
    except Exception: continue
    c = j["config"]
    print(f'P={c["rank_slice"]} W={c["window"]} store={c["store_frac"]:.0%} ssd={c["ssd_chunks"]}: ttft {j["ttft_ms_mean"]:.3f}/{j["ttft_ms_p95"]:.3f} step {j["step_ms_mean"]:.3f} wall {j["ttft_wall_ms_mean"]:.3f} hit {j["chunk_hit_ratio"]:.4f}',
          " | ".join(f'rho {p["rho"]}: {p["ttft_ms_mean"]:.1f}/{p["ttft_ms_p95"]:.1f} svc {p["service_ms_mean"]:.2f} dev {p["device_ttft_ms_mean"]:.2f}' for p in j.get("poisson", [])))
PY
