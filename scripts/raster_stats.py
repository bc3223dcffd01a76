"""Debug: how many list entries the compositing forward stages / evaluates per query (SPLATB200_STATS=1)."""
import os, sys
os.environ["SPLATB200_STATS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2411_16816_b200 import api, synth
from paper_2411_16816_b200.model import RasterSettings

ST = RasterSettings()
ctx = api.Context(0)
sc = synth.make_scene(int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000, seed=3)
ctx.upload_scene(sc)
lid = synth.lidar128()
for name, v in (("lidar128", ctx.render_lidar(lid, synth.grid_rays(lid), ST)), ("camera1080p", ctx.render_camera(synth.make_camera(), ST))):
    st, rs = v.stats(), v.array("raster_stats")
    nc = v.array("n_contrib")
    hit = None
    tiles = st["tiles_x"] * st["tiles_y"]
    print(f"{name}: I={st['n_intersections']} tiles={tiles} queries={st['n_queries']} staged={rs[0]} ({rs[0] / tiles:.0f}/tile) "
          f"warp-survivors={rs[1]} ({rs[1] / (8 * tiles):.0f}/warp/tile = {rs[1] / max(rs[0], 1) / 8:.3f} of staged) "
          f"blends={int(nc.sum())} ({nc.mean():.1f}/query; per warp-survivor {nc.sum() / max(rs[1], 1):.2f} lanes)")
