#!/usr/bin/env python
"""profiles/counters.json (and the legacy traffic.json) from an `ncu --page raw --csv` export of a `--set full` capture of
ONE serialised frame (bench.py --serial: the lidar's kernels first, then the camera's). Per kernel and sensor, summed over
the kernel's launches in the frame: DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum), duration, launches, and the
duration-weighted means of the utilisation counters bench.py quotes (issue slots, SM throughput, resident warps, DRAM
throughput). Keys are bench.py's kernel names: k_raster_bwd<camera>, k_radix_pass<lidar>, k_expand<camera>, ...

  python scripts/make_counters_json.py raw.csv profiles/counters.json [profiles/traffic.json]
"""
import csv
import json
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
         "second": 1e3, "nsecond": 1e-6, "%": 1.0, "": 1.0}
PCT = {"issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
       "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "lanes_per_inst": "smsp__thread_inst_executed_per_inst_executed.ratio", "warp_instructions": "smsp__inst_executed.sum",
       "l2_hit_pct": "lts__t_sector_hit_rate.pct", "red_sectors": "lts__t_sectors_srcunit_tex_op_red.sum"}
SUMS = ("warp_instructions", "red_sectors")   # summed over a kernel's launches; everything else is a duration-weighted mean


def val(d, name):
    if name not in ix:
        return None
    try:
        return float(d[ix[name]].replace(",", "")) * SCALE.get(units[ix[name]], 1.0)
    except ValueError:
        return None


out, sensor = {}, "lidar"
for d in data:
    name = d[ix["Kernel Name"]]
    m = re.match(r"(?:void )?(?:sb::)?(k_\w+)", name)
    if not m:
        continue
    base = m.group(1)
    if base == "k_project" and re.search(r"k_project<(?:\(bool\))?(?:1|true)>", name):
        sensor = "camera"        # the camera's projection opens the second half of the serialised frame
    if base in ("k_conv3x3_tc", "k_conv3x3_wgrad_tc", "k_dec_fold", "k_dec_head_bwd", "k_decoder_input", "k_dec_transpose_w"):
        key = base
    else:
        key = f"{base}<{sensor}>"
    e = out.setdefault(key, {"launches": 0, "time_ms": 0.0, "dram_bytes": 0.0, **{k: 0.0 for k in PCT}})
    t = val(d, "gpu__time_duration.sum") or 0.0
    e["launches"] += 1
    e["time_ms"] += t
    e["dram_bytes"] += (val(d, "dram__bytes_read.sum") or 0.0) + (val(d, "dram__bytes_write.sum") or 0.0)
    for k, metric in PCT.items():
        v = val(d, metric)
        if v is not None:
            e[k] += v if k in SUMS else v * t
for e in out.values():
    for k in PCT:
        if k in SUMS:
            continue
        e[k] = e[k] / e["time_ms"] if e["time_ms"] > 0 else None
json.dump(out, open(sys.argv[2], "w"), indent=1)
if len(sys.argv) > 3:
    json.dump({k: e["dram_bytes"] for k, e in out.items()}, open(sys.argv[3], "w"), indent=1)
print(json.dumps(out, indent=1))
