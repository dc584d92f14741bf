#!/bin/bash
# C4 world-count sweep at 2000 contacts/world: wave quantisation of the step kernel
# (4 resident worlds per SM x 148 SMs = 592 slots).  tools/sweep_worlds.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}_worlds_sweep.jsonl
: > $OUT
for W in 148 296 444 592 740 888 1024 1184 1480 1776 2048 4096; do
  timeout 300 python bench.py --worlds $W --steps 50 --cpu-seconds 0.1 --e2e-steps 1 2>/dev/null | tail -1 >> $OUT
done
python - "$OUT" <<'PY'
import json, sys
print(f"{'W':>6} {'us/step':>9} {'ns/world':>9} {'frac':>6}")
for l in open(sys.argv[1]):
    d = json.loads(l)
    W = d['config']['worlds_per_gpu']
    print(f"{W:>6} {d['ms_per_step']*1e3:9.1f} {d['ms_per_step']*1e6/W:9.1f} {d['roofline']['frac']:6.3f}")
PY
