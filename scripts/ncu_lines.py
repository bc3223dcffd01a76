"""Per-source-line instruction and stall-sample totals from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys
from collections import defaultdict

path, kernel_filter = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
rows = list(csv.reader(open(path)))
file_path = func = None
hdr = None
agg = defaultdict(lambda: [0, 0, ""])   # (func, file, line) -> [inst, samples, text]
tot = defaultdict(lambda: [0, 0])
i = 0
while i < len(rows):
    r = rows[i]
    if r and r[0] == "File Path":
        file_path = r[1]
    elif r and r[0] == "Function Name":
        func = r[1]
    elif r and r[0] == "Line No":
        hdr = r
        i_inst, i_samp = hdr.index("Instructions Executed"), hdr.index("# Samples")
    elif hdr and len(r) > 5 and func and kernel_filter in func:
        try:
            line = int(r[0]) if r[0] else cur_line
        except ValueError:
            i += 1
            continue
        cur_line = line
        key = (func.split("(")[0][-30:], file_path.split("/")[-1], line)
        if r[1]:
            agg[key][2] = r[1].strip()[:90]
        try:
            agg[key][0] += int(r[i_inst]); agg[key][1] += int(r[i_samp])
            tot[key[0]][0] += int(r[i_inst]); tot[key[0]][1] += int(r[i_samp])
        except ValueError:
            pass
    i += 1
for f, (ti, ts) in tot.items():
    print(f"== {f}: {ti} warp-instructions, {ts} samples")
    items = sorted(((k, v) for k, v in agg.items() if k[0] == f), key=lambda kv: -kv[1][0])[:top]
    for (fn, fl, ln), (inst, samp, text) in items:
        print(f"  {100*inst/max(ti,1):5.1f}% inst {100*samp/max(ts,1):5.1f}% samp  {fl}:{ln:<4d} {text}")
