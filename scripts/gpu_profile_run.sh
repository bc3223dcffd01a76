#!/usr/bin/env bash
# Runs ON THE GPU BOX (under gpurun): everything profiles/ is refreshed from.
# Usage: scripts/gpu_profile_run.sh <tag> [main|decoder|sanitize]  (separate calls: gpurun brings back at most 64 MiB per call)
# Outputs land in gpurun_out/; scripts/profiles_postprocess.sh <tag> (run in the build container) turns them into
# the committed summaries under profiles/.
set -uo pipefail
TAG="${1:-r1}"
PART="${2:-main}"
OUT=gpurun_out
mkdir -p "$OUT"
if [ "$PART" = "main" ]; then
# 1. the bench lines (not under a profiler)
timeout 600 python bench.py > "$OUT/bench_${TAG}.json" 2> "$OUT/bench_${TAG}.err"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > "$OUT/bench_${TAG}_reference_arm.json" 2>> "$OUT/bench_${TAG}.err"
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 1 > "$OUT/bench_${TAG}_cfg4.json" 2>> "$OUT/bench_${TAG}.err"
# 2. launch list of the same command (shares only; cold-cache, serialised)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file "$OUT/launches_${TAG}.csv" \
    python bench.py --steps 2 --warmup 1 --no-cpu --serial > /dev/null 2>&1
# 3. full-set capture of every hand-written kernel of one frame (second frame: warm)
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"^(k_|void k_|sb::k_|void sb::k_)" -s 30 -c 30 \
    -o "$OUT/prof_${TAG}" python bench.py --steps 1 --warmup 1 --no-cpu --serial > "$OUT/ncu_${TAG}.log" 2>&1
fi
if [ "$PART" = "decoder" ]; then
# 3b. the camera ConvDecoder: timing, launch list, full-set capture of its tensor-core kernels
PYTHONPATH=. timeout 300 python scripts/time_decoder.py 10 > "$OUT/decoder_${TAG}.txt" 2>&1
PYTHONPATH=. timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"conv|dec" -c 60 --csv \
    --log-file "$OUT/launches_decoder_${TAG}.csv" python scripts/time_decoder.py 1 > /dev/null 2>&1
PYTHONPATH=. timeout 900 ncu --set full --clock-control none -k regex:"k_conv3x3|k_dec" -s 27 -c 27 \
    -o "$OUT/prof_decoder_${TAG}" python scripts/time_decoder.py 2 > "$OUT/ncu_decoder_${TAG}.log" 2>&1
fi
if [ "$PART" = "sanitize" ]; then
# 4. sanitizers on the small parity configs (racecheck without the tensor-core kernels: their bounded barrier waits
#    expire under its instrumentation)
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests -m gpu -q -x -k "config1 or lidar_forward_backward or camera_forward_backward or edge_cases or more_than_256 or one_level or radix_sort or assign_points or line_of_sight or set_rays or overlapped or view_streams or conv3x3 or decode_image_matches or decode_image_backward_matches or kernel_pairs or async_scene" \
    > "$OUT/sanitizer_memcheck_${TAG}.log" 2>&1
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests -m gpu -q -x -k "config1 or camera_forward_backward or more_than_256 or line_of_sight or assign_points_matches" \
    > "$OUT/sanitizer_racecheck_${TAG}.log" 2>&1
fi
ls -la "$OUT"
