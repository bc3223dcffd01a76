#!/usr/bin/env bash
# Run in the build container after scripts/gpu_profile_run.sh <tag>: summaries of gpurun_out/ -> profiles/ (committed).
set -euo pipefail
TAG="${1:-r1}"
G=gpurun_out
P=profiles
cp "$G/bench_${TAG}.json" "$G/bench_${TAG}_reference_arm.json" "$P/"
[ -f "$G/bench_${TAG}_cfg4.json" ] && cp "$G/bench_${TAG}_cfg4.json" "$P/"
cp "$G/launches_${TAG}.csv" "$P/"
python - "$G/launches_${TAG}.csv" > "$P/launches_${TAG}_summary.txt" <<'PY'
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]; ki, vi = h.index("Kernel Name"), h.index("Metric Value")
tot = defaultdict(lambda: [0.0, 0])
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    tot[r[ki][:70]][0] += v / 1000.0; tot[r[ki][:70]][1] += 1
s = sum(v[0] for v in tot.values())
print("ncu --metrics gpu__time_duration.sum --clock-control none -c 600 : python bench.py --steps 2 --warmup 1 --no-cpu --serial  (one stream: deterministic kernel order; ncu serialises launches anyway)")
print("per-kernel totals over the captured launches (cold-cache, serialised: compare SHARES with bench.py's roofline.stage_ms)")
for k, (us, n) in sorted(tot.items(), key=lambda x: -x[1][0]):
    print(f"{us:10.1f} us {n:4d}x {100 * us / s:5.1f}%  {k}")
PY
ncu -i "$G/prof_${TAG}.ncu-rep" --page raw --csv > /tmp/prof_${TAG}_raw.csv
python scripts/ncu_summary.py /tmp/prof_${TAG}_raw.csv > "$P/ncu_full_${TAG}.txt"
python scripts/make_counters_json.py /tmp/prof_${TAG}_raw.csv "$P/counters.json" "$P/traffic.json" > /dev/null
ncu -i "$G/prof_${TAG}.ncu-rep" --page source --csv --print-source cuda,sass > /tmp/prof_${TAG}_src.csv
: > "$P/ncu_source_lines_${TAG}.txt"
for k in "k_raster_fwd_lidar" "k_raster_fwd<(bool)1" "k_raster_bwd_lidar" "k_raster_bwd<(bool)1" "k_expand" "k_radix_pass<(int)2"; do
  echo "#### $k" >> "$P/ncu_source_lines_${TAG}.txt"
  python scripts/ncu_lines.py /tmp/prof_${TAG}_src.csv "$k" 25 >> "$P/ncu_source_lines_${TAG}.txt"
done
if [ -f "$G/launches_decoder_${TAG}.csv" ]; then
  cp "$G/launches_decoder_${TAG}.csv" "$G/decoder_${TAG}.txt" "$P/"
  ncu -i "$G/prof_decoder_${TAG}.ncu-rep" --page raw --csv > /tmp/prof_decoder_${TAG}_raw.csv
  python scripts/ncu_summary.py /tmp/prof_decoder_${TAG}_raw.csv > "$P/ncu_full_decoder_${TAG}.txt"
fi
for t in memcheck racecheck; do
  grep -E "COMPUTE-SANITIZER|passed|failed|ERROR SUMMARY|RACECHECK SUMMARY|hazard" "$G/sanitizer_${t}_${TAG}.log" | tail -6 > "$P/sanitizer_${t}_${TAG}.log" || true
done
ls -la "$P"
