#!/usr/bin/env python
"""profiles/traffic.json from an `ncu --page raw --csv` export of a `--set full` capture of one frame:
dram__bytes_read.sum + dram__bytes_write.sum per launch, keyed the way bench.py names kernels
(k_raster_bwd<camera> ...). The first view of a frame is the lidar (template argument 0), the second the camera (1)."""
import csv
import json
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}


def to_bytes(v, u):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]


out, seen = {}, {}
for d in data:
    name = d[ix["Kernel Name"]]
    m = re.match(r"(?:void )?(?:sb::)?(k_\w+)(?:<(?:\(bool\))?(\d)(?:,\s*\(?\w*\)?\s*(\d))?>)?", name)
    if not m:
        continue
    base, targ = m.group(1), m.group(2)
    n = seen.get(base, 0)
    seen[base] = n + 1
    sensor = ("camera" if targ == "1" else "lidar") if targ is not None else ("lidar" if n == 0 else "camera")
    key = f"{base}<{sensor}>"
    rd = to_bytes(d[ix["dram__bytes_read.sum"]], units[ix["dram__bytes_read.sum"]])
    wr = to_bytes(d[ix["dram__bytes_write.sum"]], units[ix["dram__bytes_write.sum"]])
    out.setdefault(key, rd + wr)
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
