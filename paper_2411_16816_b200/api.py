"""Host-side mirror of the reference's operator interface for the hot path, over the C ABI of
libsplat_b200.so (include/splat_b200.h). ctypes only: no torch, no numpy math on the data path.

Reference names (under /root/reference/proj/include/splat/):
  compose_at_time      scene.hpp:273-308      project_camera / project_lidar  projection.hpp:88-118 / 140-174
  compose_backward     scene.hpp:386-458      project_*_backward              projection.hpp:250-288 / 322-357
  rasterize_camera / rasterize_lidar / backward
There is NO CPU fallback: importing works anywhere (so that the symbol table can be checked on a CPU
box), but creating a Context without a CUDA device raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .model import CameraModel, LidarModel, RasterSettings, RaySet, Scene

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsplat_b200.so")
_LIB = None

INT_ARRAYS = {"raster_stats", "hit_bits", "source_index", "rect", "isect_tile", "isect_depth_bits", "isect_src", "tile_begin", "tile_end",
              "grid", "n_contrib", "last_idx"}

# every symbol include/splat_b200.h declares
SYMBOLS = [
    "splatb200_ctx_create", "splatb200_ctx_destroy", "splatb200_last_error", "splatb200_ctx_sync",
    "splatb200_ctx_launch_count", "splatb200_ctx_library_launch_count",
    "splatb200_debug_depth_sort", "splatb200_assign_points", "splatb200_ctx_set_profiling", "splatb200_ctx_set_view_streams", "splatb200_ctx_join", "splatb200_view_stage_ms", "splatb200_scene_upload", "splatb200_scene_upload_async", "splatb200_scene_bind_device",
    "splatb200_scene_set_tracks", "splatb200_scene_actor_velocity", "splatb200_grads_zero", "splatb200_grads_size",
    "splatb200_grads_device_ptr", "splatb200_grads_bind_device", "splatb200_grads_download",
    "splatb200_grads_download_actor", "splatb200_view_create_camera", "splatb200_view_create_lidar",
    "splatb200_view_destroy", "splatb200_view_set_camera", "splatb200_view_set_lidar_pose", "splatb200_view_set_rays", "splatb200_optimizer_step", "splatb200_optimizer_step_range", "splatb200_grads_nonfinite_range", "splatb200_scene_download", "splatb200_conv_decoder_params", "splatb200_view_decode_image", "splatb200_debug_conv3x3", "splatb200_view_decode_image_backward", "splatb200_debug_conv3x3_backward", "splatb200_lidar_head_params", "splatb200_view_set_lidar_head", "splatb200_lidar_head_forward", "splatb200_lidar_head_backward", "splatb200_view_set_los", "splatb200_view_set_los_grad", "splatb200_lidar_grid",
    "splatb200_view_forward", "splatb200_view_stats_get", "splatb200_view_blend", "splatb200_view_alpha",
    "splatb200_view_n_contrib", "splatb200_view_backward", "splatb200_view_sensor_grads", "splatb200_view_download",
    "splatb200_view_backward_host", "splatb200_view_download_async", "splatb200_view_forward_to_host", "splatb200_view_backward_from_host", "splatb200_view_backward_host_overlapped", "splatb200_view_array", "splatb200_view_composed", "splatb200_view_projected",
    "splatb200_view_project_backward", "splatb200_view_compose_backward", "splatb200_view_backward_projected",
    "splatb200_optimizer_reset", "splatb200_nccl_unique_id", "splatb200_ctx_comm_init", "splatb200_ctx_comm_bind",
    "splatb200_ctx_comm_destroy", "splatb200_ctx_comm_info", "splatb200_allreduce_grads", "splatb200_sharded_optimizer_step",
    "splatb200_ctx_set_decoder_precise",
]


class SplatError(RuntimeError):
    pass


class SettingsPOD(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("dilation", "alpha_clamp", "alpha_min", "qform_max", "transmittance_min",
                                         "near_plane", "lidar_min_range")]


class CameraPOD(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float), ("width", C.c_int32),
                ("height", C.c_int32), ("R", C.c_float * 9), ("t", C.c_float * 3), ("vel_lin", C.c_float * 3),
                ("vel_ang", C.c_float * 3), ("shutter_duration", C.c_float), ("time_offset", C.c_float),
                ("timestamp", C.c_float)]


class AdamConfigPOD(C.Structure):
    _fields_ = [("lr_init", C.c_float * 6), ("lr_final", C.c_float * 6), ("warmup_steps", C.c_int64 * 6), ("total_steps", C.c_int64)]


class LidarPOD(C.Structure):
    _fields_ = [("elevation_channels", C.POINTER(C.c_float)), ("n_beams", C.c_int32), ("azimuth_resolution", C.c_float),
                ("scan_duration", C.c_float), ("beam_divergence_h", C.c_float), ("beam_divergence_v", C.c_float),
                ("R", C.c_float * 9), ("t", C.c_float * 3), ("vel_lin", C.c_float * 3), ("vel_ang", C.c_float * 3),
                ("timestamp", C.c_float), ("max_range", C.c_float)]


class TrackPOD(C.Structure):
    _fields_ = [("n_poses", C.c_int32), ("stamps", C.POINTER(C.c_double)), ("R", C.POINTER(C.c_double)),
                ("t", C.POINTER(C.c_double)), ("pose_offset", C.POINTER(C.c_double)), ("vel_lin", C.c_double * 3),
                ("vel_ang", C.c_double * 3), ("vel_offset", C.c_double * 6), ("init_velocity_from_poses", C.c_int32)]


class SensorGradsPOD(C.Structure):
    _fields_ = [("d_vel_lin", C.c_float * 3), ("d_vel_ang", C.c_float * 3), ("d_time_offset", C.c_float)]


class StatsPOD(C.Structure):
    _fields_ = [("n_gaussians", C.c_int64), ("n_visible", C.c_int64), ("n_intersections", C.c_int64),
                ("n_queries", C.c_int64), ("tiles_x", C.c_int32), ("tiles_y", C.c_int32)]


def lib():
    """Load libsplat_b200.so. Raises if it has not been built: the product path never falls back."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise SplatError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                             "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.splatb200_last_error.restype = C.c_char_p
        L.splatb200_last_error.argtypes = [C.c_void_p]
        for n in ("splatb200_ctx_launch_count", "splatb200_ctx_library_launch_count", "splatb200_grads_size",
                  "splatb200_view_array"):
            getattr(L, n).restype = C.c_int64
        for n in ("splatb200_grads_device_ptr", "splatb200_view_blend", "splatb200_view_alpha", "splatb200_view_n_contrib"):
            getattr(L, n).restype = C.c_void_p
        L.splatb200_ctx_destroy.restype = None
        L.splatb200_view_destroy.restype = None
        L.splatb200_ctx_launch_count.argtypes = [C.c_void_p]
        L.splatb200_ctx_library_launch_count.argtypes = [C.c_void_p]
        L.splatb200_ctx_set_profiling.argtypes = [C.c_void_p, C.c_int32]
        L.splatb200_ctx_set_view_streams.argtypes = [C.c_void_p, C.c_int32]
        L.splatb200_ctx_join.argtypes = [C.c_void_p]
        L.splatb200_optimizer_step.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        L.splatb200_optimizer_step_range.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
        L.splatb200_grads_nonfinite_range.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p]
        L.splatb200_scene_download.argtypes = [C.c_void_p] * 7
        L.splatb200_lidar_head_params.argtypes = [C.c_int32]
        L.splatb200_conv_decoder_params.argtypes = []
        L.splatb200_conv_decoder_params.restype = C.c_int32
        L.splatb200_view_decode_image.argtypes = [C.c_void_p] * 5
        L.splatb200_view_decode_image_backward.argtypes = [C.c_void_p] * 6
        L.splatb200_debug_conv3x3_backward.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
        L.splatb200_debug_conv3x3.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
        L.splatb200_view_set_lidar_head.argtypes = [C.c_void_p, C.c_void_p]
        L.splatb200_lidar_head_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.splatb200_lidar_head_backward.argtypes = [C.c_void_p] * 5
        L.splatb200_view_set_los.argtypes = [C.c_void_p, C.c_void_p]
        L.splatb200_view_set_los_grad.argtypes = [C.c_void_p, C.c_void_p]
        L.splatb200_view_set_rays.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64]
        L.splatb200_assign_points.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int32, C.c_uint32] + [C.c_void_p] * 6
        L.splatb200_debug_depth_sort.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.splatb200_view_stage_ms.argtypes = [C.c_void_p, C.c_void_p]
        L.splatb200_grads_size.argtypes = [C.c_void_p]
        L.splatb200_grads_device_ptr.argtypes = [C.c_void_p]
        L.splatb200_ctx_destroy.argtypes = [C.c_void_p]
        L.splatb200_view_destroy.argtypes = [C.c_void_p]
        L.splatb200_ctx_sync.argtypes = [C.c_void_p]
        L.splatb200_grads_zero.argtypes = [C.c_void_p]
        for n in ("splatb200_view_blend", "splatb200_view_alpha", "splatb200_view_n_contrib"):
            getattr(L, n).argtypes = [C.c_void_p]
        L.splatb200_view_array.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]
        L.splatb200_view_projected.restype = C.c_int64
        L.splatb200_view_projected.argtypes = [C.c_void_p] * 3
        L.splatb200_view_composed.argtypes = [C.c_void_p] * 5
        L.splatb200_view_project_backward.argtypes = [C.c_void_p] * 5 + [C.c_int64, C.c_int64] + [C.c_void_p] * 3
        L.splatb200_view_compose_backward.argtypes = [C.c_void_p] * 5 + [C.c_int64, C.c_int64]
        L.splatb200_view_backward_projected.argtypes = [C.c_void_p] * 6
        L.splatb200_view_forward.argtypes = [C.c_void_p, C.c_float, C.c_int32]
        L.splatb200_view_backward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.splatb200_view_backward_host.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.splatb200_view_download.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.splatb200_view_download_async.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.splatb200_view_backward_host_overlapped.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.splatb200_view_forward_to_host.argtypes = [C.c_void_p, C.c_float, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32]
        L.splatb200_view_backward_from_host.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.splatb200_view_stats_get.argtypes = [C.c_void_p, C.c_void_p]
        L.splatb200_view_sensor_grads.argtypes = [C.c_void_p, C.c_void_p]
        L.splatb200_view_set_camera.argtypes = [C.c_void_p, C.c_void_p]
        L.splatb200_view_set_lidar_pose.argtypes = [C.c_void_p] + [C.c_void_p] * 4
        L.splatb200_grads_bind_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.splatb200_grads_download.argtypes = [C.c_void_p] * 7
        L.splatb200_grads_download_actor.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
        L.splatb200_scene_actor_velocity.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
        L.splatb200_scene_upload.argtypes = [C.c_void_p, C.c_int64, C.c_int32] + [C.c_void_p] * 7
        L.splatb200_scene_upload_async.argtypes = [C.c_void_p, C.c_int64, C.c_int32] + [C.c_void_p] * 7
        L.splatb200_scene_bind_device.argtypes = [C.c_void_p, C.c_int64, C.c_int32] + [C.c_void_p] * 7 + [C.c_int32]
        L.splatb200_scene_set_tracks.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
        L.splatb200_view_create_camera.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.splatb200_view_create_lidar.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                                  C.c_void_p, C.c_int64, C.c_void_p]
        L.splatb200_ctx_create.argtypes = [C.c_int, C.c_void_p, C.c_void_p]
        L.splatb200_lidar_grid.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.splatb200_optimizer_reset.argtypes = [C.c_void_p]
        L.splatb200_ctx_set_decoder_precise.argtypes = [C.c_void_p, C.c_int32]
        L.splatb200_nccl_unique_id.argtypes = [C.c_void_p]
        L.splatb200_ctx_comm_init.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32]
        L.splatb200_ctx_comm_bind.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32]
        L.splatb200_ctx_comm_destroy.argtypes = [C.c_void_p]
        L.splatb200_ctx_comm_info.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.splatb200_allreduce_grads.argtypes = [C.c_void_p]
        L.splatb200_sharded_optimizer_step.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        _LIB = L
    return _LIB


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the library's run-time NCCL binding: 128 bytes rank 0 hands to every rank."""
    buf = C.create_string_buffer(128)
    if lib().splatb200_nccl_unique_id(buf) != 0:
        raise SplatError("NCCL is not available (libnccl.so.2 could not be bound)")
    return buf.raw


def _f32(a):
    return np.ascontiguousarray(a, np.float32)


def _settings_pod(st: RasterSettings) -> SettingsPOD:
    return SettingsPOD(*[np.float32(getattr(st, n)) for n, _ in SettingsPOD._fields_])


def _fill3(dst, src, n):
    for k, x in enumerate(np.asarray(src, np.float64).reshape(n).astype(np.float32)):
        dst[k] = x


def _camera_pod(cam: CameraModel) -> CameraPOD:
    p = CameraPOD(fx=np.float32(cam.fx), fy=np.float32(cam.fy), cx=np.float32(cam.cx), cy=np.float32(cam.cy),
                  width=cam.width, height=cam.height, shutter_duration=np.float32(cam.shutter_duration),
                  time_offset=np.float32(cam.time_offset), timestamp=np.float32(cam.timestamp))
    _fill3(p.R, cam.R, 9); _fill3(p.t, cam.t, 3); _fill3(p.vel_lin, cam.vel_lin, 3); _fill3(p.vel_ang, cam.vel_ang, 3)
    return p


def _lidar_pod(lid: LidarModel):
    elev = _f32(lid.elevation_channels)
    p = LidarPOD(elevation_channels=elev.ctypes.data_as(C.POINTER(C.c_float)), n_beams=len(elev),
                 azimuth_resolution=np.float32(lid.azimuth_resolution), scan_duration=np.float32(lid.scan_duration),
                 beam_divergence_h=np.float32(lid.beam_divergence_h), beam_divergence_v=np.float32(lid.beam_divergence_v),
                 timestamp=np.float32(lid.timestamp), max_range=np.float32(lid.max_range))
    _fill3(p.R, lid.R, 9); _fill3(p.t, lid.t, 3); _fill3(p.vel_lin, lid.vel_lin, 3); _fill3(p.vel_ang, lid.vel_ang, 3)
    return p, elev


class Context:
    """One (GPU, stream): owns the device copy of a SceneGraph and its SceneParamGrads."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self.L = lib()
        h = C.c_void_p()
        rc = self.L.splatb200_ctx_create(C.c_int(device), C.c_void_p(stream), C.byref(h))
        if rc != 0:
            raise SplatError(f"splatb200_ctx_create failed ({rc}): {self.L.splatb200_last_error(None).decode()}")
        self.h = h
        self.n = 0
        self.d_f = 0
        self.n_tracks = 0
        self._keep = []

    def close(self):
        if getattr(self, "h", None):
            self.L.splatb200_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc < 0:
            msg = self.L.splatb200_last_error(self.h).decode()
            if rc == -3:
                raise IndexError(msg)          # std::out_of_range in the reference
            raise SplatError(f"[{rc}] {msg}")
        return rc

    def sync(self):
        self._check(self.L.splatb200_ctx_sync(self.h))

    @property
    def launch_count(self) -> int:
        return int(self.L.splatb200_ctx_launch_count(self.h))

    @property
    def library_launch_count(self) -> int:
        return int(self.L.splatb200_ctx_library_launch_count(self.h))

    def assign_points_to_tiles(self, lidar: LidarModel, xyz_world: np.ndarray, stamps: np.ndarray, train: bool = False, seed: int = 0):
        """lidar returns -> per-tile rasterization points (same dict as the oracle's
        assign_points_to_tiles, plus `rayset`: the RaySet view_create_lidar takes)."""
        xyz = np.ascontiguousarray(xyz_world, np.float32).reshape(-1, 3)
        ts = np.ascontiguousarray(stamps, np.float32)
        n = len(ts)
        pod, keep = _lidar_pod(lidar)
        m_phi, m_omega = lidar.grid()
        T = m_phi * m_omega
        tile, sph = np.zeros(n, np.int64), np.zeros((n, 4), np.float32)
        order, begin, end, cnt = np.zeros(n, np.int64), np.zeros(T, np.int64), np.zeros(T, np.int64), np.zeros(3, np.int64)
        self._check(self.L.splatb200_assign_points(self.h, C.byref(pod), n, _p(xyz), _p(ts), int(train), int(seed) & 0xffffffff,
                                                   _p(tile), _p(sph), _p(order), _p(begin), _p(end), _p(cnt)))
        order = order[:cnt[0]].copy()
        rays = np.ascontiguousarray(sph[order][:, :3])
        return {"tile": tile, "phi": sph[:, 0].copy(), "omega": sph[:, 1].copy(), "t_l": sph[:, 2].copy(), "range": sph[:, 3].copy(),
                "order": order, "begin": begin, "end": end, "rejected": int(cnt[1]), "dropped": int(cnt[2]),
                "rayset": RaySet(rays=rays, begin=begin.copy(), end=end.copy())}

    def optimizer_step(self, cfg: dict, step: int):
        """optimizer_step on the resident scene from the resident gradients; cfg: lr_init[6], lr_final[6],
        warmup_steps[6], total_steps. Returns the skipped groups."""
        pod = AdamConfigPOD()
        for k in range(6):
            pod.lr_init[k], pod.lr_final[k], pod.warmup_steps[k] = cfg["lr_init"][k], cfg["lr_final"][k], int(cfg["warmup_steps"][k])
        pod.total_steps = int(cfg["total_steps"])
        skipped = (C.c_int32 * 6)()
        self._check(self.L.splatb200_optimizer_step(self.h, C.byref(pod), int(step), skipped))
        return [k for k in range(6) if skipped[k]]

    @staticmethod
    def _adam_pod(cfg: dict):
        pod = AdamConfigPOD()
        for k in range(6):
            pod.lr_init[k], pod.lr_final[k], pod.warmup_steps[k] = cfg["lr_init"][k], cfg["lr_final"][k], int(cfg["warmup_steps"][k])
        pod.total_steps = int(cfg["total_steps"])
        return pod

    def grads_nonfinite_range(self, lo: int, hi: int):
        flags = (C.c_int32 * 6)()
        self._check(self.L.splatb200_grads_nonfinite_range(self.h, int(lo), int(hi), flags))
        return [int(flags[k]) for k in range(6)]

    def optimizer_step_range(self, cfg: dict, step: int, lo: int, hi: int, skip_groups=None):
        """optimizer_step on the slice [lo, hi) of the flat gradient layout (a rank's shard); skip_groups: 6 flags."""
        pod = self._adam_pod(cfg)
        skipped = (C.c_int32 * 6)()
        skip = None if skip_groups is None else (C.c_int32 * 6)(*[int(x) for x in skip_groups])
        self._check(self.L.splatb200_optimizer_step_range(self.h, C.byref(pod), int(step), int(lo), int(hi), skip, skipped))
        return [k for k in range(6) if skipped[k]]

    def optimizer_reset(self):
        """Forget the Adam moments (an upload_scene of the same shape keeps them)."""
        self._check(self.L.splatb200_optimizer_reset(self.h))

    # ---- multi-GPU (scene.hpp:351-362): the gradient all-reduce through the C ABI --------------------
    def comm_init(self, unique_id: bytes, rank: int, world: int):
        """ncclCommInitRank with the id from nccl_unique_id() (created on rank 0, distributed out of band)."""
        assert len(unique_id) == 128
        self._check(self.L.splatb200_ctx_comm_init(self.h, C.c_char_p(unique_id), int(rank), int(world)))

    def comm_bind(self, nccl_comm_ptr: int, rank: int, world: int):
        self._check(self.L.splatb200_ctx_comm_bind(self.h, C.c_void_p(nccl_comm_ptr), int(rank), int(world)))

    def comm_destroy(self):
        self._check(self.L.splatb200_ctx_comm_destroy(self.h))

    @property
    def comm_world(self) -> int:
        w = C.c_int32(0)
        self.L.splatb200_ctx_comm_info(self.h, None, C.byref(w))
        return int(w.value)

    def allreduce_grads(self):
        """In-place SUM of SceneParamGrads (and the ActorGrad slots) over the ranks of the ctx's communicator; ordered
        after every view stream, enqueued on the ctx stream."""
        self._check(self.L.splatb200_allreduce_grads(self.h))

    def sharded_optimizer_step(self, cfg: dict, step: int):
        """optimizer_step fused with the collective: reduce each shard to its owner, Adam on the shard, broadcast."""
        pod = self._adam_pod(cfg)
        skipped = (C.c_int32 * 6)()
        self._check(self.L.splatb200_sharded_optimizer_step(self.h, C.byref(pod), int(step), skipped))
        return [k for k in range(6) if skipped[k]]

    def download_scene(self):
        """Current parameters: (mean, scale_log, quat, opacity_logit, color, feature) as float32 arrays."""
        n, d_f = self.n, self.d_f
        out = [np.zeros((n, 3), np.float32), np.zeros((n, 3), np.float32), np.zeros((n, 4), np.float32), np.zeros(n, np.float32),
               np.zeros((n, 3), np.float32), np.zeros((n, d_f), np.float32)]
        self._check(self.L.splatb200_scene_download(self.h, *[_p(a) for a in out]))
        return out

    def debug_depth_sort(self, keys: np.ndarray, counts: np.ndarray):
        """Test hook: the binning stage's radix sort + count scan on caller data -> (order, offsets)."""
        keys = np.ascontiguousarray(keys, np.uint32)
        counts = np.ascontiguousarray(counts, np.uint32)
        n = len(keys)
        order, offsets = np.zeros(n, np.uint32), np.zeros(n + 1, np.uint32)
        self._check(self.L.splatb200_debug_depth_sort(self.h, n, _p(keys), _p(counts), _p(order), _p(offsets)))
        return order, offsets

    def debug_conv3x3(self, x, w, relu_in=False, res=None):
        """Test hook: one 3x3, 32 -> 32 reflect-padded convolution of the ConvDecoder (tensor cores) on host arrays."""
        x = np.ascontiguousarray(x, np.float32)
        w = np.ascontiguousarray(w, np.float32)
        H, W, ch = x.shape
        assert ch == 32 and w.size == 9248
        r = None if res is None else np.ascontiguousarray(res, np.float32)
        y = np.zeros_like(x)
        self._check(self.L.splatb200_debug_conv3x3(self.h, _p(x), H, W, _p(w), int(relu_in), _p(r), _p(y)))
        return y

    def debug_conv3x3_backward(self, x, w, g_y, relu_in=False):
        """Test hook: (g_x, g_w) of one decoder convolution (tensor cores) on host arrays."""
        x = np.ascontiguousarray(x, np.float32); w = np.ascontiguousarray(w, np.float32); g_y = np.ascontiguousarray(g_y, np.float32)
        H, W, _ = x.shape
        gx, gw = np.zeros_like(x), np.zeros(9248, np.float32)
        self._check(self.L.splatb200_debug_conv3x3_backward(self.h, _p(x), H, W, _p(w), int(relu_in), _p(g_y), _p(gx), _p(gw)))
        return gx, gw

    def set_decoder_precise(self, on: bool):
        """ConvDecoder convolutions in split-tf32 (three passes, fp32 accuracy) instead of plain tf32 (default)."""
        self._check(self.L.splatb200_ctx_set_decoder_precise(self.h, int(on)))

    def set_view_streams(self, on: bool):
        """Views run forward / backward on their own streams (sensors overlap); see splat_b200.h."""
        self._check(self.L.splatb200_ctx_set_view_streams(self.h, int(on)))

    def join(self):
        """Order the ctx stream after every view's own stream (before external work on the ctx stream reads results)."""
        self._check(self.L.splatb200_ctx_join(self.h))

    def set_profiling(self, on: bool):
        self._check(self.L.splatb200_ctx_set_profiling(self.h, int(on)))

    # ---- SceneGraph ---------------------------------------------------------------------------
    def upload_scene(self, scene: Scene):
        s = scene.astype(np.float32)
        self.n, self.d_f = s.n, s.d_f
        self._check(self.L.splatb200_scene_upload(self.h, s.n, s.d_f, _p(s.mean), _p(s.scale_log), _p(s.quat),
                                                  _p(s.opacity_logit), _p(s.color), _p(s.feature), _p(s.actor_id)))
        self.set_tracks(scene.tracks)

    def upload_scene_async(self, scene: Scene):
        """Geometry-first upload without the wait (splatb200_scene_upload_async): `scene` must already hold float32 /
        int32 arrays (pinned for a truly asynchronous copy) that stay alive and unchanged until the next sync(); tracks
        are not touched."""
        for a in (scene.mean, scene.scale_log, scene.quat, scene.opacity_logit, scene.color, scene.feature):
            if a.dtype != np.float32 or not a.flags["C_CONTIGUOUS"]:
                raise ValueError("upload_scene_async needs contiguous float32 arrays")
        if scene.actor_id.dtype != np.int32:
            raise ValueError("upload_scene_async needs an int32 actor_id array")
        self._keep_scene = scene
        self._check(self.L.splatb200_scene_upload_async(self.h, scene.n, scene.d_f, _p(scene.mean), _p(scene.scale_log), _p(scene.quat),
                                                        _p(scene.opacity_logit), _p(scene.color), _p(scene.feature), _p(scene.actor_id)))

    def bind_scene_device(self, n, d_f, mean, scale_log, quat, opacity_logit, color, feature, actor_id, max_actor_id=0):
        """Zero-copy: arguments are raw device addresses (e.g. torch.Tensor.data_ptr())."""
        self.n, self.d_f = int(n), int(d_f)
        self._check(self.L.splatb200_scene_bind_device(self.h, n, d_f, mean, scale_log, quat, opacity_logit, color,
                                                       feature, actor_id, max_actor_id))

    def set_tracks(self, tracks):
        arr = (TrackPOD * max(1, len(tracks)))()
        keep = []
        for k, tr in enumerate(tracks):
            f = lambda a: np.ascontiguousarray(a, np.float64)
            st, R, t, po = f(tr.stamps), f(tr.R), f(tr.t), f(tr.pose_offset)
            keep += [st, R, t, po]
            dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
            arr[k].n_poses = len(st)
            arr[k].stamps, arr[k].R, arr[k].t, arr[k].pose_offset = dp(st), dp(R), dp(t), dp(po)
            for j in range(3):
                arr[k].vel_lin[j] = float(tr.vel_lin[j]); arr[k].vel_ang[j] = float(tr.vel_ang[j])
            for j in range(6):
                arr[k].vel_offset[j] = float(tr.vel_offset[j])
            arr[k].init_velocity_from_poses = int(tr.init_velocity_from_poses)
        self._check(self.L.splatb200_scene_set_tracks(self.h, len(tracks), C.byref(arr)))
        self.n_tracks = len(tracks)
        self.track_poses = [len(tr.stamps) for tr in tracks]

    def actor_velocity(self, a):
        out = np.zeros(6)
        self._check(self.L.splatb200_scene_actor_velocity(self.h, a, _p(out)))
        return out[:3], out[3:]

    # ---- SceneParamGrads ----------------------------------------------------------------------
    def zero_grads(self):
        self._check(self.L.splatb200_grads_zero(self.h))

    @property
    def grads_size(self) -> int:
        return int(self.L.splatb200_grads_size(self.h))

    @property
    def grads_device_ptr(self) -> int:
        return int(self.L.splatb200_grads_device_ptr(self.h) or 0)

    def bind_grads_device(self, ptr: int, n_floats: int):
        self._check(self.L.splatb200_grads_bind_device(self.h, C.c_void_p(ptr), n_floats))

    def grads_into(self, d_mean, d_scale_log, d_quat, d_opacity_logit, d_color, d_feature):
        """Download SceneParamGrads into caller-owned (e.g. pinned) float32 arrays; None skips a group."""
        self._check(self.L.splatb200_grads_download(self.h, _p(d_mean), _p(d_scale_log), _p(d_quat), _p(d_opacity_logit),
                                                    _p(d_color), _p(d_feature)))

    def grads(self):
        n, d_f = self.n, self.d_f
        g = dict(d_mean=np.zeros((n, 3), np.float32), d_scale_log=np.zeros((n, 3), np.float32),
                 d_quat=np.zeros((n, 4), np.float32), d_opacity_logit=np.zeros(n, np.float32),
                 d_color=np.zeros((n, 3), np.float32), d_feature=np.zeros((n, d_f), np.float32))
        self._check(self.L.splatb200_grads_download(self.h, _p(g["d_mean"]), _p(g["d_scale_log"]), _p(g["d_quat"]),
                                                    _p(g["d_opacity_logit"]), _p(g["d_color"]), _p(g["d_feature"])))
        g["actors"] = []
        for a in range(self.n_tracks):
            dp, dv = np.zeros((self.track_poses[a], 6)), np.zeros(6)
            self._check(self.L.splatb200_grads_download_actor(self.h, a, _p(dp), _p(dv)))
            g["actors"].append(dict(d_pose_offset=dp, d_vel_offset=dv))
        return g

    # ---- views --------------------------------------------------------------------------------
    def camera_view(self, cam: CameraModel, settings: RasterSettings) -> "View":
        h = C.c_void_p()
        pod, st = _camera_pod(cam), _settings_pod(settings)
        self._check(self.L.splatb200_view_create_camera(self.h, C.byref(pod), C.byref(st), C.byref(h)))
        return View(self, h, True, cam.width * cam.height)

    def lidar_view(self, lidar: LidarModel, rayset: RaySet, settings: RasterSettings) -> "View":
        h = C.c_void_p()
        (pod, elev), st = _lidar_pod(lidar), _settings_pod(settings)
        rays = _f32(rayset.rays)
        rb, re = np.ascontiguousarray(rayset.begin, np.int64), np.ascontiguousarray(rayset.end, np.int64)
        self._check(self.L.splatb200_view_create_lidar(self.h, C.byref(pod), C.byref(st), _p(rays), len(rays), _p(rb),
                                                       _p(re), len(rb), C.byref(h)))
        return View(self, h, False, len(rays))

    # reference-shaped one-shot calls: compose + project + bin + composite for one sensor
    def render_camera(self, cam, settings, t_scene=0.0, stop_after=0) -> "View":
        v = self.camera_view(cam, settings)
        v.forward(t_scene, stop_after)
        return v

    def render_lidar(self, lidar, rayset, settings, t_scene=0.0, stop_after=0) -> "View":
        v = self.lidar_view(lidar, rayset, settings)
        v.forward(t_scene, stop_after)
        return v


class View:
    def __init__(self, ctx: Context, h, camera: bool, P: int):
        self.ctx, self.h, self.camera, self.P, self.L = ctx, h, camera, P, ctx.L

    def close(self):
        if getattr(self, "h", None) and getattr(self.ctx, "h", None):
            self.L.splatb200_view_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def decode_image(self, params, embedding, download=True, timed=False):
        """decode_image: the ConvDecoder over this camera view's blended features -> H*W x 3 image
        (None with download=False: read array("decoded")). timed=True also returns the device time in ms."""
        w = np.ascontiguousarray(params, np.float32)
        e = np.ascontiguousarray(embedding, np.float32)
        assert w.size == self.L.splatb200_conv_decoder_params() and e.size == 8
        img = np.zeros((self.P, 3), np.float32) if download else None
        ms = C.c_float(0)
        self.ctx._check(self.L.splatb200_view_decode_image(self.h, _p(w), _p(e), _p(img) if download else None,
                                                           C.byref(ms) if timed else None))
        return (img, ms.value) if timed else img

    def decode_image_backward(self, g_image, g_blend_device_ptr: int, timed=False):
        """Backward of decode_image: dL/dimage (P x 3) -> (dL/dparams, dL/dembedding[8]); dL/dF_rgb and dL/dfeature are
        added to the DEVICE buffer (P x 16: rgb, then d_f features) at g_blend_device_ptr — the upstream gradient of view.backward_device."""
        g = np.ascontiguousarray(g_image, np.float32)
        assert g.size == 3 * self.P
        gp = np.zeros(self.L.splatb200_conv_decoder_params(), np.float32)
        ge = np.zeros(8, np.float32)
        ms = C.c_float(0)
        self.ctx._check(self.L.splatb200_view_decode_image_backward(self.h, _p(g), _p(gp), _p(ge), C.c_void_p(g_blend_device_ptr),
                                                                    C.byref(ms) if timed else None))
        return (gp, ge, ms.value) if timed else (gp, ge)

    def set_lidar_head(self, weights):
        """Fused lidar head: every forward also decodes the blended features (array("lidar_head"): P x 2); None: off."""
        w = None if weights is None else np.ascontiguousarray(weights, np.float32)
        self.ctx._check(self.L.splatb200_view_set_lidar_head(self.h, _p(w)))

    def lidar_head_forward(self, weights) -> np.ndarray:
        """decode_lidar over this view's blended features: P x 2 (intensity, ray-drop probability)."""
        w = np.ascontiguousarray(weights, np.float32)
        assert w.size == self.L.splatb200_lidar_head_params(self.ctx.d_f)
        y = np.zeros((self.P, 2), np.float32)
        self.ctx._check(self.L.splatb200_lidar_head_forward(self.h, _p(w), _p(y)))
        return y

    def lidar_head_backward(self, weights, g_y, g_blend16_device_ptr: int) -> np.ndarray:
        """-> dL/dweights; dL/dfeature is added to the DEVICE buffer (P x 16) at g_blend16_device_ptr."""
        w = np.ascontiguousarray(weights, np.float32)
        gy = np.ascontiguousarray(g_y, np.float32)
        gw = np.zeros(w.size, np.float32)
        self.ctx._check(self.L.splatb200_lidar_head_backward(self.h, _p(w), _p(gy), _p(gw), C.c_void_p(g_blend16_device_ptr)))
        return gw

    def set_los(self, los_cut):
        """Line-of-sight channel: per-ray cut r_p - eps (None: off); the next forward fills array("los")."""
        cut = None if los_cut is None else np.ascontiguousarray(los_cut, np.float32)
        self.ctx._check(self.L.splatb200_view_set_los(self.h, _p(cut)))

    def set_los_grad(self, g_los):
        self.ctx._check(self.L.splatb200_view_set_los_grad(self.h, _p(np.ascontiguousarray(g_los, np.float32))))

    def set_rays(self, rayset: RaySet):
        """A new sweep for this lidar view (e.g. ctx.assign_points_to_tiles(...)["rayset"])."""
        rays = np.ascontiguousarray(rayset.rays, np.float32)
        rb, re = np.ascontiguousarray(rayset.begin, np.int64), np.ascontiguousarray(rayset.end, np.int64)
        self.ctx._check(self.L.splatb200_view_set_rays(self.h, _p(rays), len(rays), _p(rb), _p(re), len(rb)))
        self.P = len(rays)

    def set_camera(self, cam: CameraModel):
        pod = _camera_pod(cam)
        self.ctx._check(self.L.splatb200_view_set_camera(self.h, C.byref(pod)))

    def set_lidar_pose(self, lidar: LidarModel):
        R, t, vl, va = (_f32(np.asarray(x, np.float64).ravel()) for x in (lidar.R, lidar.t, lidar.vel_lin, lidar.vel_ang))
        self.ctx._check(self.L.splatb200_view_set_lidar_pose(self.h, _p(R), _p(t), _p(vl), _p(va)))

    def forward(self, t_scene=0.0, stop_after=0):
        self.ctx._check(self.L.splatb200_view_forward(self.h, C.c_float(t_scene), stop_after))

    STAGES = ("project", "depth_sort_scan", "tile_counts", "tile_sort", "_unused", "raster_fwd", "raster_bwd", "project_bwd")

    def stage_ms(self) -> dict:
        out = np.zeros(8, np.float32)
        self.ctx._check(self.L.splatb200_view_stage_ms(self.h, _p(out)))
        return {k: v for k, v in zip(self.STAGES, out.astype(float).tolist()) if not k.startswith("_")}

    def stats(self) -> dict:
        s = StatsPOD()
        self.ctx._check(self.L.splatb200_view_stats_get(self.h, C.byref(s)))
        return {n: int(getattr(s, n)) for n, _ in StatsPOD._fields_}

    def array(self, name):
        n = self.ctx._check(self.L.splatb200_view_array(self.h, name.encode(), None))
        out = np.empty(n, np.int64 if name in INT_ARRAYS else np.float32)
        self.ctx._check(self.L.splatb200_view_array(self.h, name.encode(), _p(out)))
        return out

    # device pointers of the rendered outputs
    @property
    def blend_ptr(self):
        return int(self.L.splatb200_view_blend(self.h))

    @property
    def alpha_ptr(self):
        return int(self.L.splatb200_view_alpha(self.h))

    def backward_device(self, g_blend16_ptr: int, g_alpha_ptr: int):
        self.ctx._check(self.L.splatb200_view_backward(self.h, C.c_void_p(g_blend16_ptr), C.c_void_p(g_alpha_ptr)))

    def backward(self, g_blend16, g_alpha):
        """Host-buffer backward (the end-to-end path)."""
        gb, ga = _f32(g_blend16), _f32(g_alpha)
        assert gb.size == 16 * self.P and ga.size == self.P
        self.ctx._check(self.L.splatb200_view_backward_host(self.h, _p(gb), _p(ga)))
        self.ctx.sync()   # gb / ga are pageable temporaries

    def backward_host_async(self, gb: np.ndarray, ga: np.ndarray):
        self.ctx._check(self.L.splatb200_view_backward_host(self.h, _p(gb), _p(ga)))

    def download_async(self, blend16=None, alpha=None, n_contrib=None):
        """Overlapped download into PINNED host arrays on the ctx's device-to-host copy stream; complete after ctx.sync()."""
        self.ctx._check(self.L.splatb200_view_download_async(self.h, _p(blend16), _p(alpha), _p(n_contrib)))

    def backward_host_overlapped(self, gb: np.ndarray, ga: np.ndarray):
        """Upstream gradients from PINNED host arrays, uploaded on the host-to-device copy stream (after this view's
        pending download_async), then the backward kernels."""
        self.ctx._check(self.L.splatb200_view_backward_host_overlapped(self.h, _p(gb), _p(ga)))

    def forward_to_host(self, t_scene: float, blend16=None, alpha=None, n_contrib=None, bands: int = 0):
        """forward + banded, overlapped download into PINNED host arrays (complete after ctx.sync())."""
        self.ctx._check(self.L.splatb200_view_forward_to_host(self.h, float(t_scene), _p(blend16), _p(alpha), _p(n_contrib), int(bands)))

    def backward_from_host(self, gb: np.ndarray, ga: np.ndarray):
        """banded, overlapped upload of the upstream gradients from PINNED host arrays + backward."""
        self.ctx._check(self.L.splatb200_view_backward_from_host(self.h, _p(gb), _p(ga)))

    def download(self, blend16=None, alpha=None, n_contrib=None):
        self.ctx._check(self.L.splatb200_view_download(self.h, _p(blend16), _p(alpha), _p(n_contrib)))

    # ---- reference-granularity calls (host buffers) ----------------------------------------------
    PROJECTED_FIELDS = (("mean2d", 0, 2), ("depth_key", 2, 1), ("cov2d", 3, 4), ("velocity", 7, 3), ("aabb", 10, 4),
                        ("conic", 14, 4), ("det_ratio", 18, 1), ("mu_sensor", 19, 3), ("rel_vel_sensor", 22, 3))

    def projected(self) -> dict:
        """project_camera / project_lidar result: dict of arrays, V rows in ascending source_index."""
        V = self.ctx._check(self.L.splatb200_view_projected(self.h, None, None))
        src, f = np.zeros(V, np.int64), np.zeros((V, 25), np.float32)
        self.ctx._check(self.L.splatb200_view_projected(self.h, _p(src), _p(f)))
        out = {"source_index": src}
        for name, off, w in self.PROJECTED_FIELDS:
            out[name] = f[:, off:off + w].copy()
        return out

    def composed(self) -> dict:
        n = self.ctx.n
        out = dict(mean_w=np.zeros((n, 3), np.float32), cov_w=np.zeros((n, 9), np.float32),
                   vel_dyn_w=np.zeros((n, 3), np.float32), opacity=np.zeros(n, np.float32))
        self.ctx._check(self.L.splatb200_view_composed(self.h, _p(out["mean_w"]), _p(out["cov_w"]), _p(out["vel_dyn_w"]),
                                                       _p(out["opacity"])))
        return out

    def project_backward(self, g_mean2d, g_range, g_cov2d, g_velocity, begin, end, compose_grads: dict):
        """project_*_backward over projected positions [begin, end); accumulates into compose_grads (N-row arrays)."""
        a = [None if x is None else _f32(x) for x in (g_mean2d, g_range, g_cov2d, g_velocity)]
        cg = compose_grads
        self.ctx._check(self.L.splatb200_view_project_backward(self.h, *[_p(x) for x in a], begin, end, _p(cg["g_mean_w"]),
                                                               _p(cg["g_cov_w"]), _p(cg["g_vel_dyn_w"])))

    def compose_backward(self, compose_grads: dict, g_opacity, begin, end):
        cg = compose_grads
        go = None if g_opacity is None else _f32(g_opacity)
        self.ctx._check(self.L.splatb200_view_compose_backward(self.h, _p(cg["g_mean_w"]), _p(cg["g_cov_w"]),
                                                               _p(cg["g_vel_dyn_w"]), _p(go), begin, end))

    def backward_projected(self, g_mean2d, g_range, g_cov2d, g_velocity, g_opacity):
        a = [None if x is None else _f32(x) for x in (g_mean2d, g_range, g_cov2d, g_velocity, g_opacity)]
        self.ctx._check(self.L.splatb200_view_backward_projected(self.h, *[_p(x) for x in a]))

    def sensor_grads(self):
        s = SensorGradsPOD()
        self.ctx._check(self.L.splatb200_view_sensor_grads(self.h, C.byref(s)))
        return np.array(list(s.d_vel_lin) + list(s.d_vel_ang) + [s.d_time_offset], np.float32)
