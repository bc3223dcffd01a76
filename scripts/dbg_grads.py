import sys, numpy as np
sys.path.insert(0, '.')
from oracle import oracle_py as op
from paper_2411_16816_b200 import api, synth
from paper_2411_16816_b200.model import RasterSettings
st = RasterSettings()
ctx = api.Context(0)
sc = synth.make_scene(4000, seed=5, r_max=40.0)
ctx.upload_scene(sc)
cam = synth.make_camera(width=320, height=192)
gv = ctx.render_camera(cam, st)
gb, ga = synth.upstream(gv.P)
ctx.zero_grads(); gv.backward(gb, ga); g = ctx.grads()
for dt in (np.float32, np.float64):
    osc = op.OracleScene(sc, dt)
    ov = osc.render_camera(cam, st, workers=4)
    ov.backward(gb, ga, workers=4)
    og = osc.grads()
    print(dt.__name__)
    for k in ("d_mean", "d_scale_log", "d_quat", "d_opacity_logit", "d_color", "d_feature"):
        a, b = g[k].astype(np.float64), og[k].reshape(g[k].shape).astype(np.float64)
        scale = np.abs(b).max()
        d = np.abs(a-b)
        i = np.unravel_index(np.argmax(d), d.shape)
        print(f"  {k}: max|b|={scale:.4g} maxdiff={d.max():.4g} rel={d.max()/scale:.3g} at {i} a={a[i]:.6g} b={b[i]:.6g}; nnz a={np.count_nonzero(a)} b={np.count_nonzero(b)}")
    if dt == np.float64:
        for name in ("rg_conic","rg_mean2d","rg_vel","rg_rho"):
            pass
    print('  sensor', gv.sensor_grads(), ov.array('sensor_grads'))
