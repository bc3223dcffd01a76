#!/usr/bin/env python
"""Generate tests/golden/ref_*.npz from the UNMODIFIED reference headers compiled against the Eigen shim
(oracle/_ref/libsplat_ref.so, built by oracle/ref_build.sh from /root/reference). Run in the build
container (the GPU box has no /root/reference); the fixtures are committed so every box can check the
oracle and the CUDA path against the reference's own outputs.

Each fixture holds the inputs (GaussianSet arrays, actor tracks, packed sensor, settings, query time), the
reference's compose + projection outputs, a set of ProjectedGrads (source-indexed; produced by the oracle's
rasterizer backward, any values would do) and the reference's project_*_backward + compose_backward outputs.
All values are fp64 results of the reference's double instantiation on fp32-representable inputs.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle_py as op, ref_py as rp                      # noqa: E402
from paper_2411_16816_b200 import synth                               # noqa: E402
from paper_2411_16816_b200.model import RasterSettings               # noqa: E402

PROJ = ("mean2d", "depth_key", "cov2d", "velocity", "aabb", "conic", "det_ratio", "mu_sensor", "rel_vel_sensor")
COMPOSED = ("mean_w", "cov_w", "vel_dyn_w", "opacity")
PG = ("pg_mean2d", "pg_range", "pg_cov2d", "pg_velocity", "pg_opacity")
BWD = ("cg_mean_w", "cg_vel_dyn_w", "cg_cov_w", "d_mean", "d_scale_log", "d_quat", "d_opacity_logit", "sensor_grads")


def cases():
    st = RasterSettings()
    static = synth.make_scene(400, seed=21, r_max=30.0, scale_mean=0.1)
    dyn = synth.make_scene(400, seed=22, n_actors=2, dynamic_fraction=0.4, r_max=30.0, scale_mean=0.1)
    for k, tr in enumerate(dyn.tracks):
        tr.t[:] = np.array([8.0 + 3 * k, -2.0 + 3 * k, 1.0]) + np.outer(tr.stamps, [6.0, 1.0, 0.0])
    cam = synth.make_camera(width=96, height=64, time_offset=0.002)
    lid = synth.lidar32()
    lid.vel_lin, lid.vel_ang = np.array([12.0, 1.0, 0.0]), np.array([0.0, 0.02, 0.3])
    yield "static_camera", static, ("camera", cam), st, 0.0
    yield "static_lidar", static, ("lidar", lid), st, 0.0
    yield "dynamic_camera", dyn, ("camera", cam), st, 0.03
    yield "dynamic_lidar", dyn, ("lidar", synth.lidar128()), st, 0.03
    yield "dynamic_camera_extrapolated", dyn, ("camera", cam), st, 0.17      # beyond the last stamp (scene.hpp:247-256)


def main():
    out_dir = os.path.join(ROOT, "tests", "golden")
    os.makedirs(out_dir, exist_ok=True)
    for name, sc, (kind, sensor), st, t_scene in cases():
        o, r = op.OracleScene(sc, np.float64), rp.RefScene(sc, np.float64)
        if kind == "camera":
            ov = o.render_camera(sensor, st, t_scene=t_scene)
            V = r.project_camera(sensor, st, t_scene)
        else:
            rays = synth.grid_rays(sensor)
            ov = o.render_lidar(sensor, rays, st, t_scene=t_scene)
            V = r.project_lidar(sensor, st, t_scene)
        gb, ga = synth.upstream(ov.P, seed=5)
        if kind == "lidar":
            gb[:, 14:] = 0
        ov.backward(gb, ga)
        pg = {k: ov.array(k) for k in PG}
        r.backward(*[pg[k] for k in PG])
        d = dict(kind=kind, t_scene=t_scene, settings=st.packed(np.float64), sensor=sensor.packed(np.float64),
                 mean=sc.mean, scale_log=sc.scale_log, quat=sc.quat, opacity_logit=sc.opacity_logit, color=sc.color,
                 feature=sc.feature, actor_id=sc.actor_id, n_tracks=len(sc.tracks), source_index=r.array("source_index"))
        if kind == "lidar":
            d["elev"] = sensor.elev(np.float64)
        for a, tr in enumerate(sc.tracks):
            for f in ("stamps", "R", "t", "pose_offset", "vel_offset"):
                d[f"track{a}_{f}"] = np.asarray(getattr(tr, f), np.float64)
            d[f"ref_actor_vel{a}"] = r.array(f"actor_vel:{a}")
            d[f"ref_actor_d_pose_offset{a}"] = r.array(f"actor_d_pose_offset:{a}")
            d[f"ref_actor_d_vel_offset{a}"] = r.array(f"actor_d_vel_offset:{a}")
        for k in PROJ + COMPOSED + BWD:
            d["ref_" + k] = r.array(k)
        d.update(pg)
        path = os.path.join(out_dir, f"ref_{name}.npz")
        np.savez_compressed(path, **d)
        print(f"{path}: N={sc.n} V={V} ({os.path.getsize(path) / 1024:.0f} KiB)")


if __name__ == "__main__":
    main()
