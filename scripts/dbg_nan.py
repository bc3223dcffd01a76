import numpy as np, sys
sys.path.insert(0,'.')
from paper_2411_16816_b200 import api, synth
from paper_2411_16816_b200.model import RasterSettings
ST=RasterSettings()
n=3_000_000
sc = synth.make_scene(n, seed=4, n_actors=32, dynamic_fraction=0.02)
ctx=api.Context(0); ctx.upload_scene(sc)
lid = synth.lidar128()
for name, v in (("camera", ctx.camera_view(synth.make_camera(yaw=np.pi / 3.0), ST)), ("lidar", ctx.lidar_view(lid, synth.grid_rays(lid), ST))):
    v.forward(0.05)
    gb, ga = synth.upstream(v.P, seed=9)
    if name=="lidar": gb[:,14:]=0
    ctx.zero_grads(); v.backward(gb, ga)
    g=ctx.grads()
    print(name, v.stats())
    for k in ("d_mean","d_scale_log","d_quat","d_opacity_logit","d_color","d_feature"):
        x=g[k].reshape(n,-1); bad=np.flatnonzero(~np.isfinite(x).all(1))
        print("  ",k,"nonfinite rows",len(bad), bad[:8])
    bad=np.flatnonzero(~np.isfinite(g["d_mean"].reshape(n,-1)).all(1))
    if len(bad):
        src=v.array("source_index"); pos={int(s):i for i,s in enumerate(src)} if len(bad)<50 else None
        i=int(bad[0]); k=int(np.searchsorted(src,i))
        print("  row",i,"actor",sc.actor_id[i],"visible",src[k]==i)
        for f in ("mean2d","depth_key","cov2d","velocity","conic","det_ratio","mu_sensor","rel_vel_sensor"):
            a=v.array(f); w=a.size//len(src); print("    ",f,a.reshape(len(src),w)[k])
        print("    raw mean",sc.mean[i],"scale_log",sc.scale_log[i],"quat",sc.quat[i],"opl",sc.opacity_logit[i])
        print("    grads", {kk:g[kk].reshape(n,-1)[i] for kk in ("d_mean","d_scale_log","d_quat","d_opacity_logit")})
