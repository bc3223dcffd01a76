"""Load tests/golden/ref_*.npz (made by scripts/make_golden.py from the compiled, unmodified reference headers)."""
import glob
import os

import numpy as np

from paper_2411_16816_b200.model import ActorTrack, CameraModel, LidarModel, RasterSettings, Scene

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
PROJ = ("mean2d", "depth_key", "cov2d", "velocity", "aabb", "conic", "det_ratio", "mu_sensor", "rel_vel_sensor")
WIDTH = dict(mean2d=2, depth_key=1, cov2d=4, velocity=3, aabb=4, conic=4, det_ratio=1, mu_sensor=3, rel_vel_sensor=3)
COMPOSED = ("mean_w", "cov_w", "vel_dyn_w", "opacity")
PG = ("pg_mean2d", "pg_range", "pg_cov2d", "pg_velocity", "pg_opacity")


def names():
    return sorted(os.path.basename(p)[4:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "ref_*.npz")))


def load(name):
    z = np.load(os.path.join(GOLDEN_DIR, f"ref_{name}.npz"))
    tracks = []
    for a in range(int(z["n_tracks"])):
        # velocities were initialised from the poses when the fixture was made (scene.hpp:70-83)
        tracks.append(ActorTrack(stamps=z[f"track{a}_stamps"], R=z[f"track{a}_R"], t=z[f"track{a}_t"],
                                 pose_offset=z[f"track{a}_pose_offset"], vel_offset=z[f"track{a}_vel_offset"],
                                 init_velocity_from_poses=True))
    sc = Scene(z["mean"], z["scale_log"], z["quat"], z["opacity_logit"], z["color"], z["feature"], z["actor_id"], tracks)
    s = z["settings"]
    st = RasterSettings(*[float(x) for x in s])
    p = z["sensor"]
    if str(z["kind"]) == "camera":
        sensor = CameraModel(fx=p[0], fy=p[1], cx=p[2], cy=p[3], width=int(p[4]), height=int(p[5]), R=p[6:15].reshape(3, 3),
                             t=p[15:18], vel_lin=p[18:21], vel_ang=p[21:24], shutter_duration=p[24], time_offset=p[25],
                             timestamp=p[26])
    else:
        sensor = LidarModel(elevation_channels=z["elev"], azimuth_resolution=p[0], scan_duration=p[1], beam_divergence_h=p[2],
                            beam_divergence_v=p[3], R=p[4:13].reshape(3, 3), t=p[13:16], vel_lin=p[16:19], vel_ang=p[19:22],
                            timestamp=p[22], max_range=p[23])
    return z, sc, sensor, st, float(z["t_scene"])


def rel_err(a, b, floor=1e-9):
    a, b = np.asarray(a, np.float64).ravel(), np.asarray(b, np.float64).ravel()
    scale = np.maximum(np.abs(b), floor * max(1e-300, np.abs(b).max(initial=0.0)))
    return float(np.max(np.abs(a - b) / np.maximum(scale, 1e-300), initial=0.0))
