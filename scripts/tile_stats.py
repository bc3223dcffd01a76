"""Debug: distribution of tile list lengths (load balance of the compositing grids)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2411_16816_b200 import api, synth
from paper_2411_16816_b200.model import RasterSettings
ST = RasterSettings()
ctx = api.Context(0)
sc = synth.make_scene(1_000_000, seed=3)
ctx.upload_scene(sc)
lid = synth.lidar128()
for name, v in (("lidar128", ctx.render_lidar(lid, synth.grid_rays(lid), ST)), ("camera1080p", ctx.render_camera(synth.make_camera(), ST))):
    tb, te = v.array("tile_begin"), v.array("tile_end")
    L = (te - tb).astype(np.int64)
    li = v.array("last_idx")
    st = v.stats()
    print(name, "tiles", len(L), "mean", L.mean(), "median", np.median(L), "p90", np.quantile(L, .9), "p99", np.quantile(L, .99), "max", L.max(),
          "| sum of top 5%:", np.sort(L)[-len(L)//20:].sum() / L.sum())
    if name.startswith("lidar"):
        print("   per tile row mean length:", L.reshape(st["tiles_y"], st["tiles_x"]).mean(1).astype(int))
    print("   last_idx (entries walked per query): mean", li.mean(), "max", li.max())
