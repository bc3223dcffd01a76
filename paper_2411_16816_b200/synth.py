"""Synthetic scenes and sensors (`synth-v1`). Host-side numpy only.

All values are generated in float64 with numpy's PCG64 and rounded once to float32, so the
oracle (fp32 / fp64) and the CUDA path see bit-identical inputs.
"""
from __future__ import annotations

import numpy as np

from .model import (ActorTrack, CameraModel, LidarModel, N_OMEGA, N_PHI, RaySet, Scene)


def _f32(a):
    return np.ascontiguousarray(np.asarray(a, np.float64).astype(np.float32))


def make_scene(n: int, seed: int = 0, d_f: int = 13, n_actors: int = 0, dynamic_fraction: float = 0.02,
               r_min: float = 3.0, r_max: float = 80.0, scale_mean: float = 0.05) -> Scene:
    """Annulus of Gaussians around the origin: r~U[3,80] m, azimuth~U[0,2pi), z~U[-2,6] m,
    scale_log~N(ln .05,.5), quat~N(0,I), opacity_logit~N(0,1.5), color~U[0,1], feature~N(0,1)."""
    rng = np.random.Generator(np.random.PCG64(0x5EED0000 + seed))
    r = rng.uniform(r_min, r_max, n)
    th = rng.uniform(0.0, 2.0 * np.pi, n)
    z = rng.uniform(-2.0, 6.0, n)
    mean = np.stack([r * np.cos(th), r * np.sin(th), z], 1)
    scale_log = rng.normal(np.log(scale_mean), 0.5, (n, 3))
    quat = rng.normal(0.0, 1.0, (n, 4))
    opacity_logit = rng.normal(0.0, 1.5, n)
    color = rng.uniform(0.0, 1.0, (n, 3))
    feature = rng.normal(0.0, 1.0, (n, d_f))
    actor_id = np.zeros(n, np.int32)
    tracks = []
    if n_actors > 0:
        per = max(1, int(n * dynamic_fraction / n_actors))
        idx = rng.permutation(n)
        for a in range(n_actors):
            sel = idx[a * per:(a + 1) * per]
            actor_id[sel] = a + 1
            mean[sel] = rng.uniform(-0.5, 0.5, (len(sel), 3)) * np.array([4.5, 2.0, 1.6])
            # 3-pose track at t in {-0.1, 0, 0.1} s, 5-20 m/s, yaw rate <= 0.3 rad/s
            ar, ath = rng.uniform(8.0, 60.0), rng.uniform(0.0, 2.0 * np.pi)
            pos0 = np.array([ar * np.cos(ath), ar * np.sin(ath), 0.8])
            yaw0, yaw_rate, speed = rng.uniform(0, 2 * np.pi), rng.uniform(-0.3, 0.3), rng.uniform(5.0, 20.0)
            stamps = np.array([-0.1, 0.0, 0.1])
            Rs, ts = [], []
            for s in stamps:
                yaw = yaw0 + yaw_rate * s
                c, sn = np.cos(yaw), np.sin(yaw)
                Rs.append(np.array([[c, -sn, 0.0], [sn, c, 0.0], [0.0, 0.0, 1.0]]))
                ts.append(pos0 + speed * s * np.array([np.cos(yaw0), np.sin(yaw0), 0.0]))
            tracks.append(ActorTrack(stamps=stamps, R=np.array(Rs), t=np.array(ts), init_velocity_from_poses=True,
                                     pose_offset=rng.normal(0, 0.01, (3, 6)), vel_offset=rng.normal(0, 0.05, 6)))
    return Scene(_f32(mean), _f32(scale_log), _f32(quat), _f32(opacity_logit), _f32(color), _f32(feature),
                 actor_id, tracks)


def _yaw(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


# camera frame: x right, y down, z forward; world: x forward, y left, z up
_CAM_FROM_WORLD = np.array([[0.0, -1.0, 0.0], [0.0, 0.0, -1.0], [1.0, 0.0, 0.0]])


def make_camera(width=1920, height=1080, yaw=0.0, position=(0.0, 0.0, 1.5), f=1000.0, moving=True,
                shutter=0.03, time_offset=0.0) -> CameraModel:
    R = _CAM_FROM_WORLD @ _yaw(yaw).T
    t = -R @ np.asarray(position, np.float64)
    return CameraModel(fx=f * width / 1920.0, fy=f * width / 1920.0, cx=width / 2.0, cy=height / 2.0, width=width,
                       height=height, R=R, t=t,
                       vel_lin=np.array([0.0, 0.0, 15.0]) if moving else np.zeros(3),
                       vel_ang=np.array([0.0, 0.1, 0.0]) if moving else np.zeros(3),
                       shutter_duration=shutter, time_offset=time_offset)


def lidar32(position=(0.0, 0.0, 1.8), yaw=0.0) -> LidarModel:
    """32 uniform channels -30.67..+10.67 deg, 1024 azimuth bins, static sensor (BASELINE config 1)."""
    elev = np.deg2rad(np.linspace(-30.67, 10.67, 32))
    R = _yaw(yaw).T
    return LidarModel(elevation_channels=elev, azimuth_resolution=2.0 * np.pi / 1024.0, scan_duration=0.1,
                      beam_divergence_h=3e-3, beam_divergence_v=1.5e-3, R=R, t=-R @ np.asarray(position, np.float64))


def lidar128(position=(0.0, 0.0, 1.8), yaw=0.0, moving=True) -> LidarModel:
    """128 non-uniform channels w_k = -5deg + 20deg*sinh(2.5u)/sinh(2.5), 1800 bins (0.2deg => phi_max=364.8deg)."""
    u = (2.0 * np.arange(128) + 1.0) / 128.0 - 1.0
    elev = np.deg2rad(-5.0 + 20.0 * np.sinh(2.5 * u) / np.sinh(2.5))
    R = _yaw(yaw).T
    return LidarModel(elevation_channels=elev, azimuth_resolution=np.deg2rad(0.2), scan_duration=0.1,
                      beam_divergence_h=3e-3, beam_divergence_v=1.5e-3, R=R, t=-R @ np.asarray(position, np.float64),
                      vel_lin=np.array([15.0, 0.0, 0.0]) if moving else np.zeros(3),
                      vel_ang=np.array([0.0, 0.0, 0.1]) if moving else np.zeros(3))


def grid_rays(lidar: LidarModel, n_azimuth: int = None) -> RaySet:
    """One ray per (beam, azimuth bin): phi=(a+.5)res, omega=channel[b], t_l=(phi/2pi-.5)*scan_duration,
    stored tile-major (tile = (b//8)*M_phi + a//32) => exactly <=256 rays per tile."""
    res = float(np.float32(lidar.azimuth_resolution))
    if n_azimuth is None:
        n_azimuth = int(round(2.0 * np.pi / res))
    m_phi, m_omega = lidar.grid()
    nb = lidar.n_beams
    b, a = np.meshgrid(np.arange(nb), np.arange(n_azimuth), indexing="ij")
    b, a = b.ravel(), a.ravel()
    tile = (b // N_OMEGA) * m_phi + (a // N_PHI)
    order = np.lexsort((a % N_PHI, b % N_OMEGA, tile))
    b, a, tile = b[order], a[order], tile[order]
    phi = (a + 0.5) * res
    omega = np.asarray(lidar.elevation_channels, np.float64)[b]
    t_l = (phi / (2.0 * np.pi) - 0.5) * lidar.scan_duration
    rays = _f32(np.stack([phi, omega, t_l], 1))
    T = m_phi * m_omega
    counts = np.bincount(tile, minlength=T).astype(np.int64)
    end = np.cumsum(counts)
    begin = end - counts
    assert counts.max() <= 256
    return RaySet(rays=rays, begin=begin.astype(np.int64), end=end.astype(np.int64), beam=b.astype(np.int32),
                  azbin=a.astype(np.int32))


def upstream(P: int, seed: int = 1):
    """N(0,1) upstream gradients for the 16 blend slots and the accumulated opacity."""
    rng = np.random.Generator(np.random.PCG64(0x5EED1000 + seed))
    return _f32(rng.normal(0, 1, (P, 16))), _f32(rng.normal(0, 1, P))
