"""Print 'us_per_step roofline_frac' from a bench.py JSON line on stdin."""
import json
import sys

d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print(f"{d['ms_per_step'] * 1e3:.2f} {d['roofline']['frac']:.3f}")
