#!/usr/bin/env bash
# A/B of prebuilt library variants on ONE box: scripts/ab.sh <rounds>  (variants: paper_2411_16816_b200/variants/*.so)
R="${1:-2}"
LIB=paper_2411_16816_b200/libsplat_b200.so
cp "$LIB" /tmp/lib_orig.so
for r in $(seq 1 "$R"); do
  for v in paper_2411_16816_b200/variants/*.so; do
    cp "$v" "$LIB"
    timeout 300 python bench.py --no-cpu --steps 20 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['roofline']['stage_ms']
print('%-28s step %.3f ms | lidar fwd %.3f bwd %.3f | camera fwd %.3f bwd %.3f | bin l %.3f c %.3f | pbwd l %.3f c %.3f' % ('$(basename $v)', d['ms_per_step'], s['lidar']['raster_fwd'], s['lidar']['raster_bwd'], s['camera']['raster_fwd'], s['camera']['raster_bwd'], sum(s['lidar'][k] for k in ('depth_sort_scan','tile_counts','tile_sort')), sum(s['camera'][k] for k in ('depth_sort_scan','tile_counts','tile_sort')), s['lidar']['project_bwd'], s['camera']['project_bwd']))"
  done
done
cp /tmp/lib_orig.so "$LIB"
