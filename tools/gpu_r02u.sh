#!/bin/bash
# the driver's exact commands, timed
export PYTHONUNBUFFERED=1
s=$(date +%s.%N); python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02u_ref.jsonl 2> gpurun_out/r02u_ref.err; echo "ref rc=$? $(echo "$(date +%s.%N) - $s" | bc) s"
s=$(date +%s.%N); python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02u_bench.jsonl 2> gpurun_out/r02u_bench.err; echo "bench rc=$? $(echo "$(date +%s.%N) - $s" | bc) s"
s=$(date +%s.%N); python3 -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02u_smoke.log 2>&1; echo "smoke rc=$? $(echo "$(date +%s.%N) - $s" | bc) s"; tail -1 gpurun_out/r02u_smoke.log
python3 -c "
import json; j=json.loads(open('gpurun_out/r02u_bench.jsonl').read().strip().splitlines()[-1])
print({k: j[k] for k in ['metric','value','unit','n_gpus','steps','warmup','ms_per_step','dtype','gpu_launches']})
print('roofline', {k: j['roofline'][k] for k in ['bound','kernel','achieved','peak','frac','traffic','unit']})
print('cpu_baseline', j['cpu_baseline']); print('e2e', j['e2e']); print('clocks', j['clocks'])
r=json.loads(open('gpurun_out/r02u_ref.jsonl').read().strip().splitlines()[-1]); print('ref', r['value'], r['ms_per_step'], r['cpu_baseline'])"
