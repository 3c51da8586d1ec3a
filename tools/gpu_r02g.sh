#!/bin/bash
# f2 / preset Z sweep: W in {0,2,4,6,8} x DRAM store {10,25,50}% at the P=8
# per-rank geometry (4 MiB chunks; 50% of the trace = 25 GB pinned), the same with an SSD tier
# (store 10% + SSD 50%) including Poisson passes, and W sweep at the P=1 geometry (store 10%).
# Every pass logs its pcr_match_prefix inputs + decisions for the CPU oracle replay.
mkdir -p gpurun_out/z_plans
export PYTHONUNBUFFERED=1
df -h /tmp | tail -1; free -g | head -2
OUT=gpurun_out/r02g_z.jsonl; : > $OUT
timeout 1200 python bench.py --workload Z --rank-slice 8 --z-windows 0,2,4,6,8 --z-store-fracs 0.1,0.25,0.5 \
    --z-log gpurun_out/z_plans >> $OUT 2> gpurun_out/r02g_z1.err; echo "dram sweep rc=$?"
timeout 1500 python bench.py --workload Z --rank-slice 8 --z-windows 0,2,4,6,8 --z-store-fracs 0.1 --ssd-frac 0.5 \
    --ssd-path /tmp/pcr_ssd_tier.bin --rho 0.5,0.8,0.95 --z-log gpurun_out/z_plans >> $OUT 2> gpurun_out/r02g_z2.err; echo "ssd sweep rc=$?"
rm -f /tmp/pcr_ssd_tier.bin
timeout 1200 python bench.py --workload Z --z-windows 0,2,4,6,8 --z-store-fracs 0.1 --z-log gpurun_out/z_plans >> $OUT 2> gpurun_out/r02g_z3.err; echo "P1 sweep rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r02g_z.jsonl"):
    try: j = json.loads(l)
    except Exception: continue
    c = j["config"]
    print(f'P={c["rank_slice"]} W={c["window"]} store={c["store_frac"]:.0%} ssd={c["ssd_chunks"]}: ttft mean {j["ttft_ms_mean"]:.3f} p95 {j["ttft_ms_p95"]:.3f} wall {j["ttft_wall_ms_mean"]:.3f} hit {j["chunk_hit_ratio"]:.3f} pin {j["store_pin_s"]:.1f}s',
          " | ".join(f'rho {p["rho"]}: {p["ttft_ms_mean"]:.2f}/{p["ttft_ms_p95"]:.2f} hit {p["chunk_hit_ratio"]:.3f}' for p in j.get("poisson", [])))
PY
ls gpurun_out/z_plans | wc -l
