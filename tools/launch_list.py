"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) for profiles/.

    python tools/launch_list.py gpurun_out/TAG_launches_pile.csv > profiles/r01_launches_pile.txt
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
print("ncu --metrics gpu__time_duration.sum --clock-control none: python bench.py --steps 4 --warmup 3 (pile)")
print("(cold-cache, serialised; every launch of the process in order; k_step = the fused S0-S7 step;")
print(" the FillFunctor / reduce launches are bench.py's L2 flush (256 MB write, then read back) between")
print(" timed steps, outside the timed region)")
ks = []
for r in rows[i + 1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    us = float(d["Metric Value"].replace(",", "")) * scale[d["Metric Unit"]]
    name = d["Kernel Name"][:60]
    print(f"{int(d['ID']):4d} {name:60s} grid {d['Grid Size']:>14s} block {d['Block Size']:>12s} {us:9.2f} us")
    if "k_step" in name:
        ks.append(us)
print(f"k_step launches: {len(ks)}, mean {sum(ks) / len(ks):.2f} us; the timed step is this one kernel (100% of it)")
