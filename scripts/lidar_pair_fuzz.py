"""GPU box: the lidar kernel pair against the shared kernels over a sweep of scenes (footprint sizes from sub-ray to
tile-filling, anisotropic, fast sensors, the azimuth seam, ragged ray sets). Each variant runs in its own process
(SPLATB200_LIDAR_V1 is read once per process); forward outputs must be bit-identical, gradients equal up to atomic order.
  PYTHONPATH=. python scripts/lidar_pair_fuzz.py"""
import os
import subprocess
import sys
import tempfile

import numpy as np

CHILD = r"""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2411_16816_b200 import api, synth
from paper_2411_16816_b200.model import RasterSettings, RaySet
out = {}
ctx = api.Context(0)
cases = [(4000, 0.02, 0.0, 32), (6000, 0.3, 30.0, 32), (3000, 1.5, 5.0, 32), (20000, 0.08, 10.0, 128), (50000, 0.05, 0.0, 128),
         (8000, 0.6, 60.0, 128), (2000, 3.0, 0.0, 32)]
for ci, (n, scale, speed, beams) in enumerate(cases):
    sc = synth.make_scene(n, seed=100 + ci, r_max=40.0, scale_mean=scale)
    sc.scale_log[:, 0] += 0.8 * (ci % 3)
    lid = synth.lidar128() if beams == 128 else synth.lidar32()
    lid.vel_lin = np.array([speed, 0.3 * speed, 0.0])
    lid.vel_ang = np.array([0.0, 0.0, 0.02 * speed])
    rs = synth.grid_rays(lid)
    if ci % 2 == 1:      # ragged: drop a pseudo-random third of the rays (tiles with partial warps, some nearly empty)
        rng = np.random.default_rng(ci)
        keep = rng.random(len(rs.rays)) > 0.33
        parts, begin, end, cur = [], [], [], 0
        for t in range(len(rs.begin)):
            seg = rs.rays[rs.begin[t]:rs.end[t]][keep[rs.begin[t]:rs.end[t]]]
            parts.append(seg); begin.append(cur); cur += len(seg); end.append(cur)
        rs = RaySet(rays=np.concatenate(parts).astype(np.float32), begin=np.array(begin, np.int64), end=np.array(end, np.int64))
    ctx.upload_scene(sc)
    v = ctx.render_lidar(lid, rs, RasterSettings())
    gb, ga = synth.upstream(v.P, seed=ci)
    gb[:, 14:] = 0
    ctx.zero_grads()
    v.backward(gb, ga)
    g = ctx.grads()
    for k in ("blend", "alpha", "n_contrib", "last_idx", "hit_bits"):
        out[f"{ci}_{k}"] = v.array(k)
    for k in ("d_mean", "d_scale_log", "d_quat", "d_opacity_logit", "d_feature"):
        out[f"{ci}_{k}"] = g[k]
    v.close()
np.savez(sys.argv[1], **out)
"""

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
res = []
with tempfile.TemporaryDirectory() as td:
    for tag, env in (("pair", {}), ("shared", {"SPLATB200_LIDAR_V1": "1"})):
        e = {k: v for k, v in os.environ.items() if k != "SPLATB200_LIDAR_V1"}
        e.update(env)
        path = os.path.join(td, tag + ".npz")
        subprocess.run([sys.executable, "-c", CHILD, path], cwd=root, env=e, check=True, timeout=1200)
        res.append(dict(np.load(path)))
a, b = res
bad = 0
for k in sorted(a):
    if k.split("_", 1)[1] in ("blend", "alpha", "n_contrib", "last_idx", "hit_bits"):
        ok = np.array_equal(a[k], b[k])
    else:
        ok = np.abs(a[k].astype(np.float64) - b[k]).max() <= 1e-4 * max(np.abs(b[k]).max(), 1e-30)
    bad += not ok
    if not ok or k.endswith("n_contrib"):
        print(f"{k:22s} {'ok' if ok else 'DIFFERS'}" + (f"  blends {int(a[k].sum())}" if k.endswith("n_contrib") else ""))
print("all identical" if bad == 0 else f"{bad} arrays differ")
sys.exit(1 if bad else 0)
