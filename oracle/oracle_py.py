"""ctypes wrapper over oracle/liboracle.so — TEST INFRASTRUCTURE ONLY.

Allowed importers: tests/, __graft_entry__.smoke(), bench.py (cpu_baseline / --impl reference).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

INT_ARRAYS = {"source_index", "rect", "isect_tile", "isect_depth_bits", "isect_src", "tile_begin", "tile_end",
              "grid", "n_contrib", "last_idx"}


def build():
    subprocess.check_call(["make", "-s", "-C", _HERE])


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        _LIB = C.CDLL(path)
        for suf in ("f32", "f64"):
            for name in ("orc_scene_new", "orc_view_camera", "orc_view_lidar"):
                getattr(_LIB, f"{name}_{suf}").restype = C.c_void_p
            getattr(_LIB, f"orc_scene_error_{suf}").restype = C.c_char_p
            for name in ("orc_scene_array", "orc_view_array"):
                getattr(_LIB, f"{name}_{suf}").restype = C.c_int64
            ct = C.c_float if suf == "f32" else C.c_double
            for name in ("orc_pixel_capture_offset", "orc_wrap_pi", "orc_wrap_two_pi", "orc_sigmoid"):
                getattr(_LIB, f"{name}_{suf}").restype = ct
            getattr(_LIB, f"orc_pixel_capture_offset_{suf}").argtypes = [C.c_int, C.c_int, ct, ct]
            getattr(_LIB, f"orc_wrap_pi_{suf}").argtypes = [ct]
            getattr(_LIB, f"orc_wrap_two_pi_{suf}").argtypes = [ct]
            getattr(_LIB, f"orc_sigmoid_{suf}").argtypes = [ct]
    return _LIB


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _suf(dtype):
    return "f32" if np.dtype(dtype) == np.float32 else "f64"


class OracleScene:
    def __init__(self, scene, dtype=np.float32):
        self.dtype = np.dtype(dtype)
        self.suf = _suf(dtype)
        self.L = lib()
        s = scene.astype(self.dtype)
        self.n, self.d_f = s.n, s.d_f
        self.h = C.c_void_p(getattr(self.L, f"orc_scene_new_{self.suf}")(
            C.c_int64(s.n), C.c_int(s.d_f), _p(s.mean), _p(s.scale_log), _p(s.quat), _p(s.opacity_logit), _p(s.color),
            _p(s.feature), _p(s.actor_id)))
        self.tracks = list(scene.tracks)
        for tr in scene.tracks:
            f = lambda a: np.ascontiguousarray(a, np.float64)
            st, R, t, po, vl, va, vo = f(tr.stamps), f(tr.R), f(tr.t), f(tr.pose_offset), f(tr.vel_lin), f(tr.vel_ang), f(tr.vel_offset)
            getattr(self.L, f"orc_scene_add_track_{self.suf}")(self.h, C.c_int(len(st)), _p(st), _p(R), _p(t), _p(po),
                                                            _p(vl), _p(va), _p(vo), C.c_int(int(tr.init_velocity_from_poses)))

    def __del__(self):
        try:
            getattr(self.L, f"orc_scene_free_{self.suf}")(self.h)
        except Exception:
            pass

    def zero_grads(self):
        getattr(self.L, f"orc_scene_zero_grads_{self.suf}")(self.h)

    def array(self, name):
        fn = getattr(self.L, f"orc_scene_array_{self.suf}")
        n = fn(self.h, name.encode(), None)
        if n < 0:
            raise KeyError(name)
        dt = np.float64 if name.startswith("actor_") else self.dtype
        out = np.empty(n, dt)
        fn(self.h, name.encode(), _p(out))
        return out

    def grads(self):
        g = {k: self.array(k) for k in ("d_mean", "d_scale_log", "d_quat", "d_opacity_logit", "d_color", "d_feature")}
        g["d_mean"] = g["d_mean"].reshape(-1, 3)
        g["d_scale_log"] = g["d_scale_log"].reshape(-1, 3)
        g["d_quat"] = g["d_quat"].reshape(-1, 4)
        g["d_color"] = g["d_color"].reshape(-1, 3)
        g["d_feature"] = g["d_feature"].reshape(self.n, -1)
        g["actors"] = [dict(d_pose_offset=self.array(f"actor_d_pose_offset:{a}").reshape(-1, 6),
                            d_vel_offset=self.array(f"actor_d_vel_offset:{a}")) for a in range(len(self.tracks))]
        return g

    def actor_velocity(self, a):
        v = self.array(f"actor_vel:{a}")
        return v[:3], v[3:]

    def render_camera(self, cam, settings, t_scene=0.0, workers=1, stop_after=0):
        h = getattr(self.L, f"orc_view_camera_{self.suf}")(
            self.h, C.c_double(t_scene), _p(cam.packed(self.dtype)), _p(settings.packed(self.dtype)), C.c_int(workers),
            C.c_int(stop_after))
        if not h:
            raise RuntimeError(getattr(self.L, f"orc_scene_error_{self.suf}")(self.h).decode())
        return OracleView(self, C.c_void_p(h), True, cam.width * cam.height)

    def render_lidar(self, lidar, rayset, settings, t_scene=0.0, workers=1, stop_after=0):
        rays = np.ascontiguousarray(rayset.rays, self.dtype)
        rb = np.ascontiguousarray(rayset.begin, np.int64)
        re = np.ascontiguousarray(rayset.end, np.int64)
        elev = lidar.elev(self.dtype)
        h = getattr(self.L, f"orc_view_lidar_{self.suf}")(
            self.h, C.c_double(t_scene), _p(lidar.packed(self.dtype)), _p(elev), C.c_int(len(elev)),
            _p(settings.packed(self.dtype)), _p(rays), C.c_int64(len(rays)), _p(rb), _p(re), C.c_int64(len(rb)),
            C.c_int(workers), C.c_int(stop_after))
        if not h:
            raise RuntimeError(getattr(self.L, f"orc_scene_error_{self.suf}")(self.h).decode())
        return OracleView(self, C.c_void_p(h), False, len(rays))


class OracleView:
    def __init__(self, scene, h, camera, P):
        self.scene, self.h, self.camera, self.P = scene, h, camera, P
        self.L, self.suf, self.dtype = scene.L, scene.suf, scene.dtype

    def __del__(self):
        try:
            getattr(self.L, f"orc_view_free_{self.suf}")(self.h)
        except Exception:
            pass

    def array(self, name):
        fn = getattr(self.L, f"orc_view_array_{self.suf}")
        n = fn(self.h, name.encode(), None)
        if n < 0:
            raise KeyError(name)
        out = np.empty(n, np.int64 if name in INT_ARRAYS else self.dtype)
        fn(self.h, name.encode(), _p(out))
        return out

    def backward(self, g_blend16, g_alpha, workers=1):
        gb = np.ascontiguousarray(g_blend16, self.dtype)
        ga = np.ascontiguousarray(g_alpha, self.dtype)
        assert gb.size == 16 * self.P and ga.size == self.P
        getattr(self.L, f"orc_view_backward_{self.suf}")(self.h, _p(gb), _p(ga), C.c_int(workers))

    def set_los(self, los_cut, workers=1):
        """Line-of-sight channel: per-ray cut r_p - eps; array("los") holds the accumulator afterwards."""
        cut = np.ascontiguousarray(los_cut, self.dtype)
        assert cut.size == self.P and not self.camera
        getattr(self.L, f"orc_view_set_los_{self.suf}")(self.h, _p(cut), C.c_int(workers))

    def set_los_grad(self, g_los):
        g = np.ascontiguousarray(g_los, self.dtype)
        assert g.size == self.P
        getattr(self.L, f"orc_view_set_los_grad_{self.suf}")(self.h, _p(g))

    def brute_force(self, early_exit=True):
        blend = np.empty((self.P, 16), self.dtype)
        alpha = np.empty(self.P, self.dtype)
        nc = np.empty(self.P, np.int64)
        getattr(self.L, f"orc_view_brute_{self.suf}")(self.h, C.c_int(int(early_exit)), _p(blend), _p(alpha), _p(nc))
        return blend, alpha, nc

    def contrib(self, gauss_flag=None, query_flag=None, want_hash=False, workers=1):
        """Contributor introspection (gradient parity gate): per-query signature of the blended (source index, clamped)
        sequence; a query blending a Gaussian with gauss_flag set is added to query_flag; every Gaussian blended by a
        flagged query is marked. Returns (hash or None, query_flag, gauss_mask)."""
        n = self.scene.n
        gf = None if gauss_flag is None else np.ascontiguousarray(gauss_flag, np.uint8)
        qf = np.zeros(self.P, np.uint8) if query_flag is None else np.ascontiguousarray(query_flag, np.uint8).copy()
        gm = np.zeros(n, np.uint8)
        h = np.zeros(self.P, np.uint64) if want_hash else None
        getattr(self.L, f"orc_view_contrib_{self.suf}")(self.h, _p(gf) if gf is not None else None, _p(qf), _p(gm),
                                                        _p(h) if h is not None else None, C.c_int(workers))
        return h, qf, gm

    def ms(self):
        return self.array("ms").astype(np.float64)


def assign_points_to_tiles(lidar, xyz_world, stamps, train=False, seed=0, dtype=np.float32):
    """lidar returns -> per-tile rasterization points. Returns a dict: tile (n, -1 = rejected),
    phi / omega / t_l / range (n), order (kept points, tile-major), begin / end (per tile), rejected, dropped."""
    L = lib()
    suf = _suf(dtype)
    xyz = np.ascontiguousarray(xyz_world, dtype).reshape(-1, 3)
    ts = np.ascontiguousarray(stamps, dtype)
    n = len(ts)
    m_phi, m_omega = lidar.grid()
    T = m_phi * m_omega
    tile = np.zeros(n, np.int64)
    sph = np.zeros((n, 4), dtype)
    order, begin, end, cnt = np.zeros(n, np.int64), np.zeros(T, np.int64), np.zeros(T, np.int64), np.zeros(3, np.int64)
    elev = lidar.elev(dtype)
    f = getattr(L, f"orc_assign_points_{suf}")
    f.restype = C.c_int64
    f(_p(lidar.packed(dtype)), _p(elev), C.c_int(len(elev)), _p(xyz), _p(ts), C.c_int64(n), C.c_int(int(train)), C.c_uint32(seed),
      _p(tile), _p(sph), _p(order), _p(begin), _p(end), _p(cnt))
    return {"tile": tile, "phi": sph[:, 0].copy(), "omega": sph[:, 1].copy(), "t_l": sph[:, 2].copy(), "range": sph[:, 3].copy(),
            "order": order[:cnt[0]].copy(), "begin": begin, "end": end, "rejected": int(cnt[1]), "dropped": int(cnt[2])}


def adam_lr(cfg, group, step):
    """linear warm-up from 0, then exponential interpolation lr_init -> lr_final."""
    w = float(cfg["warmup_steps"][group])
    ramp = min(1.0, step / w) if w > 0 else 1.0
    denom = float(cfg["total_steps"]) - w
    t = min(1.0, max(0.0, (step - w) / denom)) if denom > 0 else 1.0
    return ramp * cfg["lr_init"][group] * (cfg["lr_final"][group] / cfg["lr_init"][group]) ** t


def adam_step(params, grads, m, v, cfg, step, dtype=np.float64):
    """optimizer_step: Adam, beta = (0.9, 0.999), eps = 1e-15, per-group scheduled learning rate; a
    group with a non-finite gradient is skipped. params / grads / m / v: lists of 6 arrays (mean, scale_log, quat,
    opacity_logit, color, feature); updated in place. Returns the list of skipped groups."""
    b1, b2, eps = dtype(0.9), dtype(0.999), dtype(1e-15)
    t1 = step + 1.0
    bc1, bc2 = dtype(1.0 / (1.0 - 0.9 ** t1)), dtype(1.0 / (1.0 - 0.999 ** t1))
    skipped = []
    for k in range(6):
        g = grads[k].astype(dtype)
        if not np.isfinite(g).all():
            skipped.append(k)
            continue
        lr = dtype(adam_lr(cfg, k, step))
        m[k][...] = b1 * m[k] + (dtype(1) - b1) * g
        v[k][...] = b2 * v[k] + (dtype(1) - b2) * g * g
        params[k][...] = params[k] - lr * (m[k] * bc1) / (np.sqrt(v[k] * bc2) + eps)
    return skipped


HEAD_HIDDEN = 32


def lidar_head_params(d_f):
    return HEAD_HIDDEN * (d_f + 3) + HEAD_HIDDEN + 2 * HEAD_HIDDEN + 2


def lidar_head_forward(w, feat, sph, dtype=np.float32):
    """decode_lidar: feat n x d_f blended features, sph n x 2 (azimuth, elevation) -> n x 2
    (intensity, ray-drop probability)."""
    L, suf = lib(), _suf(dtype)
    feat = np.ascontiguousarray(feat, dtype); sph = np.ascontiguousarray(sph, dtype); w = np.ascontiguousarray(w, dtype)
    n, d_f = feat.shape
    assert w.size == lidar_head_params(d_f)
    y = np.zeros((n, 2), dtype)
    getattr(L, f"orc_lidar_head_forward_{suf}")(_p(w), C.c_int(d_f), C.c_int64(n), _p(feat), _p(sph), _p(y))
    return y


def lidar_head_backward(w, feat, sph, g_y, dtype=np.float32):
    """-> (dL/dw [params], dL/dfeat [n x d_f])"""
    L, suf = lib(), _suf(dtype)
    feat = np.ascontiguousarray(feat, dtype); sph = np.ascontiguousarray(sph, dtype); w = np.ascontiguousarray(w, dtype)
    g_y = np.ascontiguousarray(g_y, dtype)
    n, d_f = feat.shape
    gw, gf = np.zeros(w.size, dtype), np.zeros((n, d_f), dtype)
    getattr(L, f"orc_lidar_head_backward_{suf}")(_p(w), C.c_int(d_f), C.c_int64(n), _p(feat), _p(sph), _p(g_y), _p(gw), _p(gf))
    return gw, gf


DEC_WIDTH, DEC_CONVS = 32, 5
DEC_CONV_PARAMS = DEC_WIDTH * 9 * DEC_WIDTH + DEC_WIDTH
DEC_HEAD_OFFSET = DEC_CONVS * DEC_CONV_PARAMS
DEC_PARAMS = DEC_HEAD_OFFSET + 6 * DEC_WIDTH + 6


def decoder_forward(params, rgb, feat, intr, emb, dtype=np.float32, want_h2=False, workers=1):
    """decode_image (decoder_oracle.hpp): rgb H x W x 3, feat H x W x d_f, intr (fx, fy, cx, cy),
    emb[8] -> image H x W x 3 (and the trunk output H x W x 32 when want_h2)."""
    L, suf = lib(), _suf(dtype)
    rgb = np.ascontiguousarray(rgb, dtype); feat = np.ascontiguousarray(feat, dtype)
    params = np.ascontiguousarray(params, dtype); intr = np.ascontiguousarray(intr, dtype); emb = np.ascontiguousarray(emb, dtype)
    H, W, d_f = feat.shape
    assert params.size == DEC_PARAMS and rgb.shape == (H, W, 3) and emb.size == 8 and d_f + 11 <= DEC_WIDTH
    image = np.zeros((H, W, 3), dtype)
    h2 = np.zeros((H, W, DEC_WIDTH), dtype) if want_h2 else None
    getattr(L, f"orc_decoder_forward_{suf}")(_p(params), C.c_int(H), C.c_int(W), C.c_int(d_f), _p(rgb), _p(feat), _p(intr),
                                             _p(emb), _p(image), _p(h2) if want_h2 else None, C.c_int(workers))
    return (image, h2) if want_h2 else image


def decoder_backward(params, rgb, feat, intr, emb, g_image, dtype=np.float64):
    """-> (dL/dparams, dL/drgb, dL/dfeat, dL/demb)"""
    L, suf = lib(), _suf(dtype)
    rgb = np.ascontiguousarray(rgb, dtype); feat = np.ascontiguousarray(feat, dtype); g_image = np.ascontiguousarray(g_image, dtype)
    params = np.ascontiguousarray(params, dtype); intr = np.ascontiguousarray(intr, dtype); emb = np.ascontiguousarray(emb, dtype)
    H, W, d_f = feat.shape
    gp, grgb, gf, ge = np.zeros(DEC_PARAMS, dtype), np.zeros((H, W, 3), dtype), np.zeros((H, W, d_f), dtype), np.zeros(8, dtype)
    getattr(L, f"orc_decoder_backward_{suf}")(_p(params), C.c_int(H), C.c_int(W), C.c_int(d_f), _p(rgb), _p(feat), _p(intr),
                                              _p(emb), _p(g_image), _p(gp), _p(grgb), _p(gf), _p(ge))
    return gp, grgb, gf, ge


def decoder_backward_from_state(params, rgb, acts, d_f, g_image):
    """Backward of decode_image from saved activations (6 x H x W x 32: x0, h0, t1, h1, t2, h2), fp64: the ReLU masks
    are those of the forward that produced `acts`. -> (dL/dparams, dL/drgb, dL/dfeat, dL/demb)"""
    L, dtype = lib(), np.float64
    rgb = np.ascontiguousarray(rgb, dtype); acts = np.ascontiguousarray(acts, dtype); g_image = np.ascontiguousarray(g_image, dtype)
    params = np.ascontiguousarray(params, dtype)
    H, W, _ = rgb.shape
    assert acts.shape == (6, H, W, DEC_WIDTH)
    gp, grgb, gf, ge = np.zeros(DEC_PARAMS, dtype), np.zeros((H, W, 3), dtype), np.zeros((H, W, d_f), dtype), np.zeros(8, dtype)
    L.orc_decoder_backward_state_f64(_p(params), C.c_int(H), C.c_int(W), C.c_int(d_f), _p(rgb), _p(acts), _p(g_image), _p(gp),
                                     _p(grgb), _p(gf), _p(ge))
    return gp, grgb, gf, ge


def detmath_eval(fn, x, y=None):
    x = np.ascontiguousarray(x, np.float32)
    y = np.zeros_like(x) if y is None else np.ascontiguousarray(y, np.float32)
    out = np.empty_like(x)
    lib().orc_detmath_eval(C.c_int(fn), _p(x), _p(y), _p(out), C.c_int64(x.size))
    return out


def hardware_threads():
    return int(lib().orc_hardware_threads())
