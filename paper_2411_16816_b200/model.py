"""Host-side mirror of the reference's scene/sensor structs (numpy, no torch).

Field names follow /root/reference/proj/include/splat/scene.hpp and projection.hpp:
  GaussianSet  scene.hpp:11-45      ActorTrack  scene.hpp:50-96
  CameraModel  scene.hpp:98-137     LidarModel  scene.hpp:139-168
  RasterSettings projection.hpp:7-15
Arrays use the reference's physical layout: Eigen column-major 3xN == N x 3 C-contiguous
(xyz interleaved), quaternion (w, x, y, z), feature D_f contiguous floats per Gaussian.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

import numpy as np

TILE = 16
N_PHI = 32     # SPEC.md:181 / PAPER.md:450
N_OMEGA = 8


@dataclass
class RasterSettings:
    dilation: float = 0.3
    alpha_clamp: float = 0.999
    alpha_min: float = 1.0 / 255.0
    qform_max: float = 9.0
    transmittance_min: float = 1e-4
    near_plane: float = 0.05
    lidar_min_range: float = 0.25

    def packed(self, dtype=np.float32) -> np.ndarray:
        v = np.array([self.dilation, self.alpha_clamp, self.alpha_min, self.qform_max,
                      self.transmittance_min, self.near_plane, self.lidar_min_range], dtype=dtype)
        return v.astype(np.float64)


@dataclass
class ActorTrack:
    stamps: np.ndarray                 # (n,) strictly increasing
    R: np.ndarray                      # (n,3,3) actor -> world
    t: np.ndarray                      # (n,3)
    pose_offset: np.ndarray = None     # (n,6): translation (world), rotvec (actor frame)
    vel_lin: np.ndarray = None         # body frame
    vel_ang: np.ndarray = None
    vel_offset: np.ndarray = None      # (6,)
    init_velocity_from_poses: bool = False
    box_size: np.ndarray = None        # (3,) actor box (scene.hpp:51); not used by the rasterizer, carried through SPZ1

    def __post_init__(self):
        n = len(self.stamps)
        self.stamps = np.asarray(self.stamps, np.float64)
        self.R = np.asarray(self.R, np.float64).reshape(n, 3, 3)
        self.t = np.asarray(self.t, np.float64).reshape(n, 3)
        self.pose_offset = np.zeros((n, 6)) if self.pose_offset is None else np.asarray(self.pose_offset, np.float64).reshape(n, 6)
        self.vel_lin = np.zeros(3) if self.vel_lin is None else np.asarray(self.vel_lin, np.float64)
        self.vel_ang = np.zeros(3) if self.vel_ang is None else np.asarray(self.vel_ang, np.float64)
        self.vel_offset = np.zeros(6) if self.vel_offset is None else np.asarray(self.vel_offset, np.float64)
        self.box_size = np.zeros(3) if self.box_size is None else np.asarray(self.box_size, np.float64).reshape(3)


@dataclass
class Scene:
    """GaussianSet + actor tracks (SceneGraph, scene.hpp:171-187)."""
    mean: np.ndarray
    scale_log: np.ndarray
    quat: np.ndarray
    opacity_logit: np.ndarray
    color: np.ndarray
    feature: np.ndarray
    actor_id: np.ndarray
    tracks: List[ActorTrack] = field(default_factory=list)

    @property
    def n(self) -> int:
        return int(self.opacity_logit.shape[0])

    @property
    def d_f(self) -> int:
        return int(self.feature.shape[1]) if self.feature.ndim == 2 else 0

    def astype(self, dtype) -> "Scene":
        c = lambda a: np.ascontiguousarray(a, dtype=dtype)
        return Scene(c(self.mean), c(self.scale_log), c(self.quat), c(self.opacity_logit), c(self.color),
                     c(self.feature), np.ascontiguousarray(self.actor_id, np.int32), list(self.tracks))


@dataclass
class CameraModel:
    fx: float = 100.0
    fy: float = 100.0
    cx: float = 50.0
    cy: float = 50.0
    width: int = 100
    height: int = 100
    R: np.ndarray = field(default_factory=lambda: np.eye(3))     # world -> sensor
    t: np.ndarray = field(default_factory=lambda: np.zeros(3))
    vel_lin: np.ndarray = field(default_factory=lambda: np.zeros(3))
    vel_ang: np.ndarray = field(default_factory=lambda: np.zeros(3))
    shutter_duration: float = 0.0
    time_offset: float = 0.0
    timestamp: float = 0.0

    def packed(self, dtype=np.float32) -> np.ndarray:
        v = np.concatenate([[self.fx, self.fy, self.cx, self.cy], np.zeros(2), np.asarray(self.R).reshape(9),
                            np.asarray(self.t).reshape(3), np.asarray(self.vel_lin).reshape(3),
                            np.asarray(self.vel_ang).reshape(3),
                            [self.shutter_duration, self.time_offset, self.timestamp]]).astype(dtype).astype(np.float64)
        v[4], v[5] = self.width, self.height
        return v

    @property
    def tiles(self):
        return (self.width + TILE - 1) // TILE, (self.height + TILE - 1) // TILE


@dataclass
class LidarModel:
    elevation_channels: np.ndarray = None    # strictly increasing, radians
    azimuth_resolution: float = 0.0
    scan_duration: float = 0.0
    beam_divergence_h: float = 0.0
    beam_divergence_v: float = 0.0
    R: np.ndarray = field(default_factory=lambda: np.eye(3))
    t: np.ndarray = field(default_factory=lambda: np.zeros(3))
    vel_lin: np.ndarray = field(default_factory=lambda: np.zeros(3))
    vel_ang: np.ndarray = field(default_factory=lambda: np.zeros(3))
    timestamp: float = 0.0
    max_range: float = 120.0

    def packed(self, dtype=np.float32) -> np.ndarray:
        return np.concatenate([[self.azimuth_resolution, self.scan_duration, self.beam_divergence_h,
                                self.beam_divergence_v], np.asarray(self.R).reshape(9), np.asarray(self.t).reshape(3),
                               np.asarray(self.vel_lin).reshape(3), np.asarray(self.vel_ang).reshape(3),
                               [self.timestamp, self.max_range]]).astype(dtype).astype(np.float64)

    def elev(self, dtype=np.float32) -> np.ndarray:
        return np.asarray(self.elevation_channels, dtype).astype(np.float64)

    @property
    def n_beams(self) -> int:
        return len(self.elevation_channels)

    def grid(self):
        """(M_phi, M_omega) — PAPER.md:451-452 with the 1e-4-tile guard described in DESIGN.md."""
        res = float(np.float32(self.azimuth_resolution))
        m_phi = int(np.ceil(2.0 * np.pi / (N_PHI * res) - 1e-4))
        m_omega = (self.n_beams + N_OMEGA - 1) // N_OMEGA
        return m_phi, m_omega


@dataclass
class RaySet:
    """Lidar rasterization points grouped per tile: tile t owns rays[begin[t]:end[t]]."""
    rays: np.ndarray        # (P,3): azimuth in [0,2pi), elevation, capture-time offset t_l
    begin: np.ndarray       # (T,) int64
    end: np.ndarray         # (T,) int64
    beam: np.ndarray = None     # (P,) beam index of each ray (grid sweeps)
    azbin: np.ndarray = None    # (P,) azimuth bin of each ray
