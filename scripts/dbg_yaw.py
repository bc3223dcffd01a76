import numpy as np, sys
sys.path.insert(0,'.')
from oracle import oracle_py as op
from paper_2411_16816_b200 import api, synth
from paper_2411_16816_b200.model import RasterSettings
ST=RasterSettings()
sc = synth.make_scene(6000, seed=23, r_max=40.0, scale_mean=0.1)
cam2 = synth.make_camera(width=320, height=192, yaw=0.7)
gb, ga = synth.upstream(320*192, seed=5)
res={}
for mode in ("fresh","reuse"):
    ctx=api.Context(0); ctx.upload_scene(sc)
    view = ctx.camera_view(synth.make_camera(width=320, height=192), ST)
    if mode=="reuse":
        view.forward(0.0); ctx.zero_grads(); view.backward(gb,ga)
    view.set_camera(cam2); view.forward(0.0); ctx.zero_grads(); view.backward(gb, ga)
    res[mode]=ctx.grads()["d_mean"].reshape(-1,3).astype(np.float64)
    ctx.close()
o64 = op.OracleScene(sc, np.float64); o64.zero_grads(); o64.render_camera(cam2, ST, workers=8).backward(gb, ga, workers=8)
o32 = op.OracleScene(sc, np.float32); o32.zero_grads(); o32.render_camera(cam2, ST, workers=8).backward(gb, ga, workers=8)
g64=o64.grads()["d_mean"].reshape(-1,3); g32=o32.grads()["d_mean"].reshape(-1,3).astype(np.float64)
def err(a): 
    sc_=np.maximum(np.abs(g64).max(1), 1e-3*np.abs(g64).max()); return np.abs(a-g64).max(1)/sc_
for k,v in res.items():
    e=err(v); print(k, "bad rows", (e>1e-3).sum(), "worst", e.max(), "argmax", e.argmax())
e=err(g32); print("ref32 bad", (e>1e-3).sum(), e.max(), e.argmax())
i=err(res["fresh"]).argmax(); print("row", i, res["fresh"][i], res["reuse"][i], g32[i], g64[i])
print("fresh vs reuse max rel", np.abs(res["fresh"]-res["reuse"]).max()/np.abs(g64).max())
