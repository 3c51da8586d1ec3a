#!/bin/bash
# cluster reduce vs workspace+combine: per-launch durations (ncu, serialised) on the short-suffix shapes
mkdir -p gpurun_out
for c in 1 0; do
  PCR_SPLIT_CLUSTER=$c timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,smsp__cycles_active.avg --clock-control none --csv \
     --log-file gpurun_out/r02e_ncu_c$c.csv python tools/attn_bench.py --small --iters 2 > /dev/null 2>&1; echo "c$c rc=$?"
done
python - <<'PY'
import csv, collections
for c in (1, 0):
    rows = list(csv.reader(open(f"gpurun_out/r02e_ncu_c{c}.csv")))
    hdr = None
    d = collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r: hdr = r; continue
        if not hdr or len(r) != len(hdr): continue
        k = r[hdr.index("Kernel Name")][:40]; m = r[hdr.index("Metric Name")]; v = r[hdr.index("Metric Value")]
        if m == "gpu__time_duration.sum": d[k].append(float(v.replace(",", "")))
    print("cluster" if c else "ws+combine")
    for k, v in d.items(): print("  ", k, len(v), "launches; durations (ns, first 24):", [int(x) for x in v[:24]])
PY
