"""GPU box: how tight is the per-warp cull? (warp, entry) pairs that survive it vs pairs in which some lane blends
(the hit bits), for both north-star sensors.   PYTHONPATH=. SPLATB200_STATS=1 python scripts/cull_yield.py"""
import os, sys
import numpy as np
sys.path.insert(0, ".")
os.environ["SPLATB200_STATS"] = "1"
from paper_2411_16816_b200 import api, synth
from paper_2411_16816_b200.model import RasterSettings
st = RasterSettings(); ctx = api.Context(0)
sc = synth.make_scene(1_000_000, seed=3); ctx.upload_scene(sc)
lid = synth.lidar128(); rays = synth.grid_rays(lid)
for name, v in (("lidar", ctx.lidar_view(lid, rays, st)), ("camera", ctx.camera_view(synth.make_camera(), st))):
    v.forward(0.0)
    rs = v.array("raster_stats"); hb = v.array("hit_bits").astype(np.uint8)
    useful = int(np.unpackbits(hb).sum()); nc = v.array("n_contrib")
    tb, te = v.array("tile_begin"), v.array("tile_end")
    print(f"{name}: I {len(hb)}, staged {rs[0]}, warp survivors {rs[1]}, (warp, entry) pairs with a blending lane {useful} "
          f"({useful / max(rs[1], 1):.2%} of survivors), entries hit by any warp {(hb != 0).sum()} ({(hb != 0).sum() / max(rs[0], 1):.2%} of staged), "
          f"blends {nc.sum()} = {nc.sum() / max(useful, 1):.1f} lanes per useful pair, non-finite records {rs[4]}"
          + (f"; lidar kernel pair: {rs[2]} (entry, ray) candidates after the exact-qf prefilter ({nc.sum() / max(rs[2], 1):.1%} of them blend), "
             f"{rs[3]} phase-2 trips (longest lane per round: one trip per {nc.sum() / max(rs[3], 1):.1f} blends)"
             if name == "lidar" and not os.environ.get("SPLATB200_LIDAR_V1") else ""))
