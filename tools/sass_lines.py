"""Per-source-line totals of an ncu SASS page (instructions executed, stall
samples): `ncu -i rep --page source --csv --print-source sass` joined with the
line info of `nvdisasm -g -c` of the same cubin (built with -lineinfo).
  python tools/sass_lines.py sass.csv disasm.sass KERNEL_SUBSTRING [top]"""
import csv
import re
import sys
from collections import defaultdict


def line_map(path, kernel):
    m, cur, on = {}, None, False
    for ln in open(path):
        if ln.startswith(".text.") or ln.lstrip().startswith(".section"):
            on = kernel in ln and ln.startswith(".text.")
            continue
        if not on:
            continue
        g = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if g:
            cur = (g.group(1).rsplit("/", 1)[-1], int(g.group(2)))
            continue
        g = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if g:
            m[int(g.group(1), 16)] = cur
    return m


def main():
    csvp, sassp, kernel = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    lm = line_map(sassp, kernel)
    rows = list(csv.reader(open(csvp)))
    hdr = rows[1]
    ia, ii, isamp = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    base = int(rows[2][ia], 16)
    inst, samp = defaultdict(float), defaultdict(float)
    for r in rows[2:]:
        if len(r) <= max(ia, ii, isamp):
            continue
        off = int(r[ia], 16) - base
        key = lm.get(off, ("?", 0))
        inst[key] += float(r[ii] or 0)
        samp[key] += float(r[isamp] or 0)
    ti, ts = sum(inst.values()), sum(samp.values())
    print(f"total warp instructions {ti:.0f}, stall samples {ts:.0f}")
    for k in sorted(samp, key=lambda k: -samp[k])[:top]:
        print(f"{k[0]}:{k[1]:<5d} samples {samp[k] / ts * 100:5.1f}%  inst {inst[k] / ti * 100:5.1f}%")


if __name__ == "__main__":
    main()
