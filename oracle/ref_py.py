"""ctypes wrapper over oracle/_ref/libsplat_ref.so — the UNMODIFIED reference headers compiled against
oracle/eigen_shim (oracle/ref_build.sh). TEST INFRASTRUCTURE ONLY (tests/, scripts/make_golden.py).

Covers the part of the hot path the reference ships as code: compose_at_time, project_camera,
project_lidar, project_*_backward, compose_backward (scene.hpp / projection.hpp).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libsplat_ref.so")
REFERENCE = os.environ.get("SPLAT_REFERENCE", "/root/reference")
_LIB = None

INT_ARRAYS = {"source_index"}


def available() -> bool:
    """True if the compiled reference exists or can be built here (needs /root/reference)."""
    return os.path.exists(LIB_PATH) or os.path.isdir(os.path.join(REFERENCE, "proj", "include", "splat"))


def build():
    subprocess.check_call(["bash", os.path.join(_HERE, "ref_build.sh")])


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        for suf, ct in (("f32", C.c_float), ("f64", C.c_double)):
            getattr(L, f"ref_scene_new_{suf}").restype = C.c_void_p
            getattr(L, f"ref_scene_error_{suf}").restype = C.c_char_p
            getattr(L, f"ref_scene_error_{suf}").argtypes = [C.c_void_p]
            getattr(L, f"ref_scene_free_{suf}").argtypes = [C.c_void_p]
            for name in ("ref_view_camera", "ref_view_lidar", "ref_array"):
                getattr(L, f"{name}_{suf}").restype = C.c_int64
            getattr(L, f"ref_view_camera_{suf}").argtypes = [C.c_void_p, C.c_double, C.c_void_p, C.c_void_p]
            getattr(L, f"ref_view_lidar_{suf}").argtypes = [C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
            getattr(L, f"ref_array_{suf}").argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]
            getattr(L, f"ref_backward_{suf}").argtypes = [C.c_void_p] * 6
            for name in ("ref_wrap_pi", "ref_wrap_two_pi", "ref_sigmoid"):
                getattr(L, f"{name}_{suf}").restype = ct
                getattr(L, f"{name}_{suf}").argtypes = [ct]
        _LIB = L
    return _LIB


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class RefScene:
    """SceneGraph<S> built through the reference's own types; one sensor view at a time."""

    def __init__(self, scene, dtype=np.float64):
        self.dtype = np.dtype(dtype)
        self.suf = "f32" if self.dtype == np.float32 else "f64"
        self.L = lib()
        s = scene.astype(self.dtype)
        self.n, self.d_f = s.n, s.d_f
        self.h = C.c_void_p(getattr(self.L, f"ref_scene_new_{self.suf}")(
            C.c_int64(s.n), C.c_int(s.d_f), _p(s.mean), _p(s.scale_log), _p(s.quat), _p(s.opacity_logit), _p(s.color),
            _p(s.feature), _p(s.actor_id)))
        self.n_tracks = len(scene.tracks)
        for tr in scene.tracks:
            f = lambda a: np.ascontiguousarray(a, np.float64)
            st, R, t, po, vl, va, vo = f(tr.stamps), f(tr.R), f(tr.t), f(tr.pose_offset), f(tr.vel_lin), f(tr.vel_ang), f(tr.vel_offset)
            getattr(self.L, f"ref_scene_add_track_{self.suf}")(self.h, C.c_int(len(st)), _p(st), _p(R), _p(t), _p(po),
                                                            _p(vl), _p(va), _p(vo), C.c_int(int(tr.init_velocity_from_poses)))

    def __del__(self):
        try:
            getattr(self.L, f"ref_scene_free_{self.suf}")(self.h)
        except Exception:
            pass

    def _err(self):
        return getattr(self.L, f"ref_scene_error_{self.suf}")(self.h).decode()

    def project_camera(self, cam, settings, t_scene=0.0) -> int:
        """compose_at_time + project_camera; returns V. Raises like the reference."""
        v = getattr(self.L, f"ref_view_camera_{self.suf}")(self.h, C.c_double(t_scene), _p(cam.packed(self.dtype)),
                                                           _p(settings.packed(self.dtype)))
        if v < 0:
            raise RuntimeError(self._err())
        return int(v)

    def project_lidar(self, lidar, settings, t_scene=0.0) -> int:
        elev = lidar.elev(self.dtype)
        v = getattr(self.L, f"ref_view_lidar_{self.suf}")(self.h, C.c_double(t_scene), _p(lidar.packed(self.dtype)), _p(elev),
                                                          C.c_int(len(elev)), _p(settings.packed(self.dtype)))
        if v < 0:
            raise RuntimeError(self._err())
        return int(v)

    def backward(self, pg_mean2d, pg_range, pg_cov2d, pg_velocity, pg_opacity):
        """project_*_backward over the whole projected list + compose_backward over all Gaussians.
        Inputs are indexed by SOURCE index (N rows)."""
        a = [np.ascontiguousarray(x, self.dtype) for x in (pg_mean2d, pg_range, pg_cov2d, pg_velocity, pg_opacity)]
        assert a[0].size == 2 * self.n and a[2].size == 4 * self.n and a[4].size == self.n
        rc = getattr(self.L, f"ref_backward_{self.suf}")(self.h, *[_p(x) for x in a])
        if rc != 0:
            raise RuntimeError(self._err())

    def array(self, name):
        fn = getattr(self.L, f"ref_array_{self.suf}")
        n = fn(self.h, name.encode(), None)
        if n < 0:
            raise KeyError(name)
        out = np.empty(n, np.int64 if name in INT_ARRAYS else self.dtype)
        fn(self.h, name.encode(), _p(out))
        return out
