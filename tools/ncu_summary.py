#!/usr/bin/env python
"""Summarise an ncu report of the fused step kernel for profiles/.

    python tools/ncu_summary.py REPORT.ncu-rep --workload pile --worlds 1024 --contacts 2000 \
        [--json profiles/step_kernel_traffic.json] > profiles/<round>_k_step_ncu.txt
"""
import argparse
import csv
import io
import json
import subprocess


def page(rep, name):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--workload", default="pile")
    ap.add_argument("--worlds", type=int, default=1024)
    ap.add_argument("--contacts", type=int, default=2000)
    ap.add_argument("--json")
    a = ap.parse_args()
    raw = page(a.report, "raw")
    h, units, vals = raw[0], raw[1], raw[2]
    d = dict(zip(h, vals))
    u = dict(zip(h, units))

    def num(k):
        v = float(d[k].replace(",", ""))
        unit = u.get(k, "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        return v * scale
    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__throughput.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__occupancy_limit_shared_mem", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
    for k in keys:
        if k in d:
            print(f"{k:60s} {d[k]} {u.get(k, '')}")
    stalls = sorted(((k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                      float(d[k])) for k in h if k.startswith("smsp__average_warps_issue_stalled_")
                     and k.endswith("per_issue_active.ratio") and d[k] not in ("", "n/a")),
                    key=lambda t: -t[1])
    print("stalls per issued instruction: " + ", ".join(f"{k}={v:.2f}" for k, v in stalls[:10]))
    print(f"dram bytes per launch (read + write) = {rd + wr:.0f}")
    if a.json:
        json.dump({"workload": a.workload, "worlds": a.worlds, "contacts_per_world": a.contacts,
                   "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
                   "source": a.report.split("/")[-1],
                   "note": "ncu --set full --clock-control none, one launch; writes still in L2 at "
                           "kernel end are not counted by dram__bytes_write"},
                  open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
