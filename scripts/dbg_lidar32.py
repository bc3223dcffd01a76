import numpy as np, sys
sys.path.insert(0,'.')
from oracle import oracle_py as op
from paper_2411_16816_b200 import api, synth
from paper_2411_16816_b200.model import RasterSettings
ST=RasterSettings()
ctx=api.Context(0)
sc=synth.make_scene(10000, seed=0x5eed0001 & 0xffff)
ctx.upload_scene(sc)
lid=synth.lidar32(); rays=synth.grid_rays(lid)
gv=ctx.render_lidar(lid, rays, ST)
ov=op.OracleScene(sc, np.float32).render_lidar(lid, rays, ST, workers=8)
a,b=gv.array("n_contrib"), ov.array("n_contrib")
bad=np.flatnonzero(a!=b)
print("mismatch", len(bad), bad[:20], a[bad[:20]], b[bad[:20]])
print("beam", rays.beam[bad[:20]], "az", rays.azbin[bad[:20]])
