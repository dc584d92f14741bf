#!/bin/bash
# C4 contact-count sweep: one bench line per contacts/world.
#   tools/sweep_contacts.sh TAG   -> gpurun_out/TAG_c4_sweep.jsonl
TAG=${1:-r01}
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}_c4_sweep.jsonl
: > $OUT
for C in 125 250 500 1000 2000 4000 8000; do
  timeout 600 python bench.py --contacts $C --steps 50 --cpu-seconds 0.2 --e2e-steps 1 2>/dev/null | tail -1 >> $OUT
done
python - "$OUT" <<'PY'
import json, sys
print(f"{'C_w':>6} {'us/step':>9} {'Mworld-steps/s':>15} {'Gcontacts/s':>12} {'GB/s':>8} {'frac':>6}")
for l in open(sys.argv[1]):
    d = json.loads(l)
    print(f"{d['config']['contacts_per_world']:>6} {d['ms_per_step']*1e3:9.1f} {d['value']/1e6:15.2f} "
          f"{d['contacts_per_s']/1e9:12.2f} {d['roofline']['achieved']:8.0f} {d['roofline']['frac']:6.3f}")
PY
