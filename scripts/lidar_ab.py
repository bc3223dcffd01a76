"""GPU-box A/B of the lidar warp-patch grouping (SPLATB200_PATCH_D, read when a view's rays are uploaded): per-stage
CUDA-event times of the north-star lidar sweep (1M Gaussians) and the evaluated / staged counters.
  PYTHONPATH=. python scripts/lidar_ab.py 0 0.004 0.0087 0.015"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
os.environ["SPLATB200_STATS"] = "1"
from paper_2411_16816_b200 import api, synth  # noqa: E402
from paper_2411_16816_b200.model import RasterSettings  # noqa: E402

st = RasterSettings()
ctx = api.Context(0)
sc = synth.make_scene(1_000_000, seed=3)
ctx.upload_scene(sc)
lid = synth.lidar128()
rays = synth.grid_rays(lid)
ref_nc = None
for d in sys.argv[1:]:
    os.environ["SPLATB200_PATCH_D"] = d
    v = ctx.lidar_view(lid, rays, st)
    gb, ga = synth.upstream(v.P, seed=11)
    gb[:, 14:] = 0
    for _ in range(3):
        v.forward(0.0)
        v.backward(gb, ga)
    s0 = v.array("raster_stats").copy()
    ctx.set_profiling(True)
    for _ in range(10):
        v.forward(0.0)
        v.backward(gb, ga)
    ms = v.stage_ms()
    ctx.set_profiling(False)
    s1 = v.array("raster_stats")
    nc = v.array("n_contrib")
    if ref_nc is None:
        ref_nc = nc
    ds = (s1 - s0) / 10.0
    print(f"patch_d={d}: raster_fwd {ms['raster_fwd']:.4f} ms, raster_bwd {ms['raster_bwd']:.4f} ms; staged {ds[0]:.0f}, evaluated per warp-entry {ds[1]:.0f} "
          f"({ds[1] / max(ds[0], 1) / 8:.3f} of staged per warp), group-list entries {ds[2]:.0f}, loop iterations {ds[3]:.0f}; n_contrib identical: {np.array_equal(nc, ref_nc)}; blends {nc.sum()}", flush=True)
    v.close()
ctx.close()
