"""Parity of the sm_100a path (through the C ABI) with the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star): cull mask, tile rectangles, intersection list, sorted keys and
per-pixel / per-ray contributor counts BIT-EXACT (vs the fp32 oracle, which runs the identical IEEE
operation sequence); rendered outputs within 1e-4 relative; gradients within 1e-3 relative (vs the
fp64 oracle).
"""
import numpy as np
import pytest

from paper_2411_16816_b200 import synth
from paper_2411_16816_b200.model import ActorTrack, CameraModel, LidarModel, RasterSettings, Scene

pytestmark = pytest.mark.gpu

ST = RasterSettings()
RENDER_RTOL = 1e-4
GRAD_RTOL = 1e-3

PROJ_FIELDS = ("mean2d", "depth_key", "cov2d", "velocity", "aabb", "conic", "det_ratio", "mu_sensor", "rel_vel_sensor")
INT_FIELDS = ("source_index", "rect", "isect_tile", "isect_depth_bits", "isect_src", "tile_begin", "tile_end")


@pytest.fixture(scope="module")
def api():
    from paper_2411_16816_b200 import api as _api
    return _api


@pytest.fixture(scope="module")
def op(oracle_lib):
    from oracle import oracle_py
    return oracle_py


@pytest.fixture()
def ctx(api):
    c = api.Context(0)
    yield c
    c.close()


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def assert_projection_bit_exact(gv, ov, sc=None):
    assert np.array_equal(gv.array("source_index"), ov.array("source_index"))
    for f in PROJ_FIELDS:
        a, b = gv.array(f), ov.array(f)
        assert a.shape == b.shape, f
        same = bits(a) == bits(b)
        assert same.all(), f"{f}: {np.count_nonzero(~same)} of {same.size} values differ bitwise (max abs {np.abs(a - b).max()})"
    assert_packed_record_bit_exact(gv, ov, sc)


def assert_packed_record_bit_exact(gv, ov, sc=None):
    """The record k_project STORED in HBM for the compositing kernels (geomA | geomB | geomC | 16 channel slots), read
    back as it lies — not the twin kernel's recomputation — against the oracle's make_splat (splat_oracle.hpp), in fp32
    arithmetic: b2 = conic01 + conic10, rho = det_ratio * opacity."""
    rec = gv.array("packed_record").reshape(-1, 26)
    src = ov.array("source_index")
    assert len(rec) == len(src)
    f32 = np.float32
    m, vel, con = ov.array("mean2d").reshape(-1, 2), ov.array("velocity").reshape(-1, 3), ov.array("conic").reshape(-1, 4)
    dr, dk, op_ = ov.array("det_ratio"), ov.array("depth_key"), ov.array("opacity")[src]
    want = np.zeros((len(src), 10), f32)
    want[:, 0:2], want[:, 2:4] = m, vel[:, :2]
    want[:, 4], want[:, 5], want[:, 6] = con[:, 0], (con[:, 1].astype(f32) + con[:, 2].astype(f32)), con[:, 3]
    want[:, 7] = dr.astype(f32) * op_.astype(f32)
    want[:, 8], want[:, 9] = dk, vel[:, 2]
    same = bits(rec[:, :10]) == bits(want)
    assert same.all(), f"packed record: {np.count_nonzero(~same)} geometry values differ bitwise (columns {np.unique(np.nonzero(~same)[1])})"
    if sc is not None:      # channel slots: camera rgb + features, lidar features, zero padded
        camera = gv.camera
        ch = np.zeros((len(src), 16), f32)
        o = 0
        if camera:
            ch[:, :3] = sc.color[src]
            o = 3
        ch[:, o:o + sc.d_f] = sc.feature[src]
        assert np.array_equal(bits(rec[:, 10:]), bits(ch)), "packed record: channel slots differ"


def assert_worklist_bit_exact(gv, ov):
    for f in INT_FIELDS:
        a, b = gv.array(f), ov.array(f)
        assert a.shape == b.shape, (f, a.shape, b.shape)
        assert np.array_equal(a, b), f"{f}: first mismatch at {np.flatnonzero(a != b)[:5]}"


def assert_render_close(gv, ov, lidar):
    assert np.array_equal(gv.array("n_contrib"), ov.array("n_contrib"))
    assert np.array_equal(gv.array("last_idx"), ov.array("last_idx"))
    b, ob = gv.array("blend").reshape(-1, 16), ov.array("blend").reshape(-1, 16)
    # identical op order => expect far better than the 1e-4 bar
    scale = np.maximum(np.abs(ob), 1e-3)
    assert (np.abs(b - ob) / scale).max() <= RENDER_RTOL
    assert np.abs(gv.array("alpha") - ov.array("alpha")).max() <= RENDER_RTOL
    assert np.abs(gv.array("t_final") - ov.array("t_final")).max() <= RENDER_RTOL


def grads_gate(ctx, og, sensor, n, what="", **kw):
    """tests/grad_gate.py: G1 (100 % of the rows within 1e-3 of the reference algorithm in fp32, minus the rows an input
    rule marks ill-conditioned) and G2 (vs fp64 on the rows without an fp32/fp64 forward flip)."""
    import grad_gate
    (g32, v32), (g64, v64) = og
    return grad_gate.grad_gate(ctx.grads(), g32, g64, v32, v64, sensor, n, what=what, **kw)


def assert_sensor_grads(gv, og):
    """SensorGrads (projection.hpp:207-222): all seven entries against the reference algorithm in fp32 (same forward
    bits) at 1e-3, and against fp64 at 5e-3 of the largest entry."""
    (_, v32), (_, v64) = og
    sg, s32, s64 = gv.sensor_grads().astype(np.float64), v32.array("sensor_grads").astype(np.float64), v64.array("sensor_grads")
    assert np.abs(sg - s32).max() <= GRAD_RTOL * np.abs(s32).max(), (sg, s32)
    assert np.abs(sg - s64).max() <= 5 * GRAD_RTOL * np.abs(s64).max(), (sg, s64)


def oracle_grads(op, sc, render, gb, ga):
    out = []
    for dt in (np.float32, np.float64):
        o = op.OracleScene(sc, dt)
        v = render(o)
        v.backward(gb, ga, workers=8)
        out.append((o.grads(), v))
    return out  # [(g32, view32), (g64, view64)]


# ---- config 1 of BASELINE.json: 10k Gaussians, 32-beam lidar, forward ---------------------------
def test_config1_lidar32_forward(ctx, op):
    sc = synth.make_scene(10000, seed=1)
    lid = synth.lidar32()
    rays = synth.grid_rays(lid)
    ctx.upload_scene(sc)
    gv = ctx.render_lidar(lid, rays, ST)
    ov = op.OracleScene(sc, np.float32).render_lidar(lid, rays, ST, workers=8)
    assert_projection_bit_exact(gv, ov, sc)
    assert_worklist_bit_exact(gv, ov)
    assert_render_close(gv, ov, True)
    st = gv.stats()
    assert st["n_visible"] == len(ov.array("source_index")) and st["n_intersections"] == len(ov.array("isect_tile"))
    # and against the fp64 oracle at the north-star tolerance
    o64 = op.OracleScene(sc, np.float64).render_lidar(lid, rays, ST, workers=8)
    nc_same = gv.array("n_contrib") == o64.array("n_contrib")
    b, ob = gv.array("blend").reshape(-1, 16)[nc_same], o64.array("blend").reshape(-1, 16)[nc_same]
    assert nc_same.mean() > 0.999
    # fp32 vs fp64 arithmetic: a sanity bound, the parity gate is the fp32 oracle above
    assert np.quantile(np.abs(b - ob) / np.maximum(np.abs(ob), 1e-2), 0.999) <= 1e-3


def _moving_lidar32():
    lid = synth.lidar32()
    lid.vel_lin, lid.vel_ang = np.array([12.0, 1.0, 0.0]), np.array([0.0, 0.02, 0.3])
    return lid


@pytest.mark.parametrize("n,seed", [(3000, 2), (20000, 3)])
def test_lidar_forward_backward(ctx, op, n, seed):
    sc = synth.make_scene(n, seed=seed, r_max=50.0, scale_mean=0.08)
    lid = _moving_lidar32() if seed == 2 else synth.lidar128()
    rays = synth.grid_rays(lid)
    ctx.upload_scene(sc)
    gv = ctx.render_lidar(lid, rays, ST)
    o32 = op.OracleScene(sc, np.float32)
    ov = o32.render_lidar(lid, rays, ST, workers=8)
    assert_projection_bit_exact(gv, ov)
    assert_worklist_bit_exact(gv, ov)
    assert_render_close(gv, ov, True)
    gb, ga = synth.upstream(gv.P, seed=seed)
    gb[:, 14:] = 0
    og = oracle_grads(op, sc, lambda o: o.render_lidar(lid, rays, ST, workers=8), gb, ga)
    ctx.zero_grads()
    gv.backward(gb, ga)
    grads_gate(ctx, og, lid, n, what="lidar ")
    assert_sensor_grads(gv, og)


@pytest.mark.parametrize("w,h,n,seed", [(320, 192, 4000, 4), (640, 360, 30000, 5), (100, 70, 800, 6)])
def test_camera_forward_backward(ctx, op, w, h, n, seed):
    sc = synth.make_scene(n, seed=seed, r_max=40.0, scale_mean=0.08)
    cam = synth.make_camera(width=w, height=h, time_offset=0.002)
    ctx.upload_scene(sc)
    gv = ctx.render_camera(cam, ST)
    ov = op.OracleScene(sc, np.float32).render_camera(cam, ST, workers=8)
    assert_projection_bit_exact(gv, ov)
    assert_worklist_bit_exact(gv, ov)
    assert_render_close(gv, ov, False)
    gb, ga = synth.upstream(gv.P, seed=seed)
    og = oracle_grads(op, sc, lambda o: o.render_camera(cam, ST, workers=8), gb, ga)
    (g32, ov32), (g64, ov64) = og
    ctx.zero_grads()
    gv.backward(gb, ga)
    grads_gate(ctx, og, cam, n, what="camera ")
    # SensorGrads are sums over all Gaussians, dominated by the ill-conditioned grazing ones: the bar is the
    # fp32 reference's own distance from the fp64 result
    sg, osg, osg32 = gv.sensor_grads(), ov64.array("sensor_grads"), ov32.array("sensor_grads")
    ref_err = np.abs(osg32 - osg).max()
    assert np.abs(sg - osg).max() <= GRAD_RTOL * np.abs(osg).max() + 5 * ref_err
    # backward accumulates (+=) like the reference: a second call doubles the gradients
    g1 = ctx.grads()
    gv.backward(gb, ga)
    g2 = ctx.grads()
    # (atomics => summation order differs run to run; the ill-conditioned grazing rows amplify that)
    for k in ("d_mean", "d_color", "d_feature", "d_opacity_logit"):
        a, b = g2[k].reshape(n, -1).astype(np.float64), 2 * g1[k].reshape(n, -1).astype(np.float64)
        rel = np.abs(a - b).max(1) / np.maximum(np.abs(b).max(1), 1e-3 * np.abs(b).max())
        assert np.quantile(rel, 0.95) <= 1e-4 and np.median(rel) <= 1e-5, (k, np.quantile(rel, 0.95))


def test_dynamic_scene_actors(ctx, op):
    """Moving actors (BASELINE config 4's ingredients): compose with interpolated actor poses,
    v_dyn, and the actor pose / velocity offset gradients (scene.hpp:292-305, 401-453)."""
    sc = synth.make_scene(6000, seed=7, n_actors=4, dynamic_fraction=0.3, r_max=30.0, scale_mean=0.1)
    for k, tr in enumerate(sc.tracks):           # park the actors in front of the camera
        tr.t[:] = np.array([8.0 + 3 * k, -3.0 + 2 * k, 1.0]) + np.outer(tr.stamps, [6.0, 1.0, 0.0])
    cam = synth.make_camera(width=320, height=192)
    t_scene = 0.03
    ctx.upload_scene(sc)
    for a in range(4):
        vl, va = ctx.actor_velocity(a)
        ovl, ova = op.OracleScene(sc, np.float64).actor_velocity(a)
        assert np.allclose(vl, ovl, atol=1e-12) and np.allclose(va, ova, atol=1e-12)
    gv = ctx.render_camera(cam, ST, t_scene=t_scene)
    ov = op.OracleScene(sc, np.float32).render_camera(cam, ST, t_scene=t_scene, workers=8)
    for f in ("mean_w", "vel_dyn_w", "opacity", "cov_w"):
        assert np.array_equal(bits(gv.array(f)), bits(ov.array(f))), f
    assert_projection_bit_exact(gv, ov)
    assert_worklist_bit_exact(gv, ov)
    assert_render_close(gv, ov, False)
    dyn = np.isin(gv.array("source_index"), np.nonzero(sc.actor_id)[0]).sum()
    assert dyn > 100
    gb, ga = synth.upstream(gv.P, seed=7)
    ogs = oracle_grads(op, sc, lambda o: o.render_camera(cam, ST, t_scene=t_scene, workers=8), gb, ga)
    (g32, _), (og, _) = ogs
    ctx.zero_grads()
    gv.backward(gb, ga)
    g = ctx.grads()
    grads_gate(ctx, ogs, cam, sc.n, what="dynamic ")
    for a in range(4):
        for k in ("d_pose_offset", "d_vel_offset"):
            x, y = g["actors"][a][k], og["actors"][a][k].reshape(g["actors"][a][k].shape)
            r = g32["actors"][a][k].reshape(x.shape)
            assert np.abs(x - y).max() <= 2e-3 * max(np.abs(y).max(), 1e-6) + 5 * np.abs(r - y).max(), (a, k)
    # lidar over the same dynamic scene
    lid = synth.lidar128()
    rays = synth.grid_rays(lid)
    gl = ctx.render_lidar(lid, rays, ST, t_scene=t_scene)
    ol = op.OracleScene(sc, np.float32).render_lidar(lid, rays, ST, t_scene=t_scene, workers=8)
    assert_projection_bit_exact(gl, ol)
    assert_worklist_bit_exact(gl, ol)
    assert_render_close(gl, ol, True)


def _golden_names():
    import golden_util as gu
    return gu.names()


@pytest.mark.parametrize("name", _golden_names())
def test_cuda_path_matches_reference_golden(ctx, op, name):
    """The sm_100a path against outputs of the reference's OWN code (unmodified headers compiled against the Eigen
    shim; tests/golden/ref_*.npz): fp32 kernels vs the reference's fp64 instantiation, so tolerances, not bits."""
    import golden_util as gu
    z, sc, sensor, st, t = gu.load(name)
    camera = hasattr(sensor, "fx")
    ctx.upload_scene(sc)
    gv = ctx.render_camera(sensor, st, t_scene=t) if camera else ctx.render_lidar(sensor, synth.grid_rays(sensor), st, t_scene=t)
    src = gv.array("source_index")
    common, gi, ri = np.intersect1d(src, z["source_index"], return_indices=True)
    assert len(common) >= 0.98 * len(z["source_index"]) and len(src) <= 1.02 * len(z["source_index"]) + 1
    dynamic = len(sc.tracks) > 0
    for f in gu.COMPOSED:
        w = 9 if f == "cov_w" else (1 if f == "opacity" else 3)
        assert gu.rel_err(gv.array(f), z["ref_" + f], floor=1e-3) <= (2e-3 if dynamic else 1e-4), f
    tol = 5e-3 if dynamic else 5e-4
    for f in gu.PROJ:
        w = gu.WIDTH[f]
        a, b = gv.array(f).reshape(-1, w)[gi].astype(np.float64), z["ref_" + f].reshape(-1, w)[ri]
        rowscale = np.maximum(np.abs(b).max(1), 1e-3 * np.abs(b).max())
        err = np.abs(a - b).max(1) / rowscale
        assert np.quantile(err, 0.98) <= tol and np.median(err) <= 1e-5, (f, np.quantile(err, 0.98), np.median(err))
    # whole backward chain: same upstream pixel gradients the fixture was made with
    gb, ga = synth.upstream(gv.P, seed=5)
    if not camera:
        gb[:, 14:] = 0
    ctx.zero_grads()
    gv.backward(gb, ga)
    g = ctx.grads()
    # the gate's G2 (tests/grad_gate.py) against the REFERENCE's values: rows no fp32/fp64 forward flip touches and the
    # input rule does not mark: 100 % within 5e-2, at most 10 % beyond 1e-3, group-level relative L2 <= 1e-3
    import grad_gate
    rays = None if camera else synth.grid_rays(sensor)
    ovs = [(op.OracleScene(sc, dt).render_camera(sensor, st, t_scene=t, workers=8) if camera else
            op.OracleScene(sc, dt).render_lidar(sensor, rays, st, t_scene=t, workers=8)) for dt in (np.float32, np.float64)]
    n_flips, fm = grad_gate.flip_mask(ovs[0], ovs[1])
    ok = ~(fm | grad_gate.ill_conditioned(ovs[1], sensor, sc.n))
    for k in ("d_mean", "d_scale_log", "d_quat", "d_opacity_logit"):
        a = g[k].reshape(sc.n, -1).astype(np.float64)
        b = z["ref_" + k].reshape(sc.n, -1)
        rowscale = np.maximum(np.abs(b).max(1), 1e-3 * np.abs(b).max())
        err = np.abs(a - b).max(1) / rowscale
        u = ok & (np.abs(b).max(1) > 0)
        msg = (f"{name} {k}: rows checked {u.sum()} of {(np.abs(b).max(1) > 0).sum()} live ({n_flips} flipped queries), beyond 1e-3: "
               f"{(err[u] > GRAD_RTOL).sum()}, worst {err[u].max(initial=0.0):.1e}")
        print(msg)
        assert err[u].max(initial=0.0) <= 5e-2 and (err[u] > GRAD_RTOL).sum() <= 0.10 * u.sum() + 1, msg
        assert np.linalg.norm((a - b)[ok]) <= 1e-3 * np.linalg.norm(b[ok]), msg
    sg = gv.sensor_grads()[:6].astype(np.float64)
    assert np.abs(sg - z["ref_sensor_grads"][:6]).max() <= 2e-2 * np.abs(z["ref_sensor_grads"][:6]).max()


def test_error_behaviour_matches_reference(ctx, api):
    sc = synth.make_scene(100, seed=8)
    sc.actor_id[17] = 5
    sc.actor_id[40] = 9
    ctx.upload_scene(sc)
    with pytest.raises(IndexError, match="unknown actor_id 5"):       # scene.hpp:297-298, first offender in index order
        ctx.render_camera(synth.make_camera(64, 64), ST)
    sc = synth.make_scene(100, seed=8)
    sc.tracks.append(ActorTrack(stamps=[], R=np.zeros((0, 3, 3)), t=np.zeros((0, 3))))
    ctx.upload_scene(sc)
    with pytest.raises(api.SplatError, match="actor track has no poses"):   # scene.hpp:242
        ctx.render_camera(synth.make_camera(64, 64), ST)
    sc = synth.make_scene(100, seed=8)
    ctx.upload_scene(sc)
    v = ctx.camera_view(synth.make_camera(64, 64), ST)
    with pytest.raises(api.SplatError, match="backward without saved forward state"):
        v.backward(np.zeros((64 * 64, 16), np.float32), np.zeros(64 * 64, np.float32))


def test_edge_cases_empty_and_culled(ctx, op):
    # empty scene => zeros
    empty = Scene(*[np.zeros((0, k), np.float32) for k in (3, 3, 4)], np.zeros(0, np.float32), np.zeros((0, 3), np.float32),
                  np.zeros((0, 13), np.float32), np.zeros(0, np.int32))
    ctx.upload_scene(empty)
    v = ctx.render_camera(synth.make_camera(64, 48), ST)
    assert np.all(v.array("blend") == 0) and np.all(v.array("alpha") == 0) and np.all(v.array("n_contrib") == 0)
    v.backward(np.ones((64 * 48, 16), np.float32), np.ones(64 * 48, np.float32))
    # everything behind the camera => all culled, nothing rendered
    sc = synth.make_scene(500, seed=9)
    sc.mean[:, 0] = -np.abs(sc.mean[:, 0]) - 1.0
    ctx.upload_scene(sc)
    v = ctx.render_camera(synth.make_camera(64, 48), ST)
    assert v.stats()["n_visible"] == 0 and v.stats()["n_intersections"] == 0
    assert np.all(v.array("blend") == 0)
    # ragged image size (last tile row/column partially filled) + zero upstream => zero grads
    sc = synth.make_scene(2000, seed=10, r_max=20.0, scale_mean=0.1)
    ctx.upload_scene(sc)
    cam = synth.make_camera(width=75, height=41)
    gv = ctx.render_camera(cam, ST)
    ov = op.OracleScene(sc, np.float32).render_camera(cam, ST)
    assert_worklist_bit_exact(gv, ov)
    assert_render_close(gv, ov, False)
    ctx.zero_grads()
    gv.backward(np.zeros((75 * 41, 16), np.float32), np.zeros(75 * 41, np.float32))
    assert all(np.all(x == 0) for k, x in ctx.grads().items() if k != "actors")


def test_azimuth_wrap_and_grazing(ctx, op):
    """Gaussians straddling azimuth 0 / 2pi and huge footprints covering the whole
    grid (no tan-FOV clamp in the reference, scene.hpp:112-117)."""
    rng = np.random.default_rng(3)
    n = 3000
    sc = synth.make_scene(n, seed=11, r_max=30.0, scale_mean=0.3)
    th = rng.uniform(-0.05, 0.05, n)
    r = rng.uniform(2.0, 25.0, n)
    sc.mean[:, 0] = (r * np.cos(th)).astype(np.float32)     # clustered around azimuth 0
    sc.mean[:, 1] = (r * np.sin(th)).astype(np.float32)
    sc.mean[:5, :2] *= 0.02                                 # a few almost on top of the sensor: full-circle AABBs
    lid = synth.lidar128()
    rays = synth.grid_rays(lid)
    ctx.upload_scene(sc)
    gv = ctx.render_lidar(lid, rays, ST)
    ov = op.OracleScene(sc, np.float32).render_lidar(lid, rays, ST, workers=8)
    rect = gv.array("rect").reshape(-1, 4)
    assert (rect[:, 0] < 0).any() and (rect[:, 1] > 57).any()      # both wrap branches exercised
    assert_projection_bit_exact(gv, ov)
    assert_worklist_bit_exact(gv, ov)
    assert_render_close(gv, ov, True)
    # camera: grazing depth => AABB over the whole tile grid
    sc2 = synth.make_scene(2000, seed=12, r_max=20.0)
    sc2.mean[:20, 0] = 0.06 + rng.uniform(0, 0.05, 20).astype(np.float32)   # z_cam ~ 0.06..0.11 m
    cam = synth.make_camera(width=256, height=144, position=(0.0, 0.0, 1.5))
    ctx.upload_scene(sc2)
    gc = ctx.render_camera(cam, ST)
    oc = op.OracleScene(sc2, np.float32).render_camera(cam, ST, workers=8)
    rect = gc.array("rect").reshape(-1, 4)
    assert ((rect[:, 1] - rect[:, 0]) * (rect[:, 3] - rect[:, 2])).max() == 16 * 9
    assert_projection_bit_exact(gc, oc)
    assert_worklist_bit_exact(gc, oc)
    assert_render_close(gc, oc, False)


def test_more_than_256_rays_per_tile(ctx, op):
    """a tile holding 257+ rays is rendered in additional passes."""
    sc = synth.make_scene(3000, seed=13, r_max=30.0, scale_mean=0.15)
    lid = synth.lidar32()
    rs = synth.grid_rays(lid)
    # duplicate the rays of every tile (512 per tile), tile-major
    T = len(rs.begin)
    parts, begin, end, cur = [], [], [], 0
    for t in range(T):
        seg = rs.rays[rs.begin[t]:rs.end[t]]
        seg = np.concatenate([seg, seg + np.array([1e-4, 0, 0], np.float32)])
        parts.append(seg)
        begin.append(cur)
        cur += len(seg)
        end.append(cur)
    from paper_2411_16816_b200.model import RaySet
    rs2 = RaySet(rays=np.concatenate(parts).astype(np.float32), begin=np.array(begin, np.int64), end=np.array(end, np.int64))
    ctx.upload_scene(sc)
    gv = ctx.render_lidar(lid, rs2, ST)
    ov = op.OracleScene(sc, np.float32).render_lidar(lid, rs2, ST, workers=8)
    assert_render_close(gv, ov, True)
    gb, ga = synth.upstream(gv.P, seed=3)
    gb[:, 14:] = 0
    og = oracle_grads(op, sc, lambda o: o.render_lidar(lid, rs2, ST, workers=8), gb, ga)
    ctx.zero_grads()
    gv.backward(gb, ga)
    grads_gate(ctx, og, lid, sc.n, what="multipass ")


_LIDAR_PAIR_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2411_16816_b200 import api, synth
from paper_2411_16816_b200.model import RasterSettings
sc = synth.make_scene(20000, seed=21, r_max=50.0, scale_mean=0.08)
lid = synth.lidar128()
lid.vel_lin = np.array([8.0, 1.0, 0.0])
rays = synth.grid_rays(lid)
ctx = api.Context(0)
ctx.upload_scene(sc)
v = ctx.render_lidar(lid, rays, RasterSettings())
gb, ga = synth.upstream(v.P, seed=21)
gb[:, 14:] = 0
ctx.zero_grads()
v.backward(gb, ga)
g = ctx.grads()
np.savez(sys.argv[1], blend=v.array("blend"), alpha=v.array("alpha"), n_contrib=v.array("n_contrib"), last_idx=v.array("last_idx"),
         hit_bits=v.array("hit_bits"),
         **{k: g[k] for k in ("d_mean", "d_scale_log", "d_quat", "d_opacity_logit", "d_feature")})
"""


@pytest.mark.gpu
def test_lidar_kernel_pairs_agree(tmp_path):
    """The lidar's own compositing kernels (raster_lidar.cu + k_raster_bwd_lidar: lane = entry prefilter, bit transpose,
    lane = ray walk; default for tiles of at most 256 rays) against the shared kernels (SPLATB200_LIDAR_V1=1), each in
    its own process: every forward output bit-identical (same per-ray blending order, same IEEE operations), gradients
    equal up to the order of the atomic additions."""
    import os
    import subprocess
    import sys as _sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for tag, env in (("v2", {}), ("v1", {"SPLATB200_LIDAR_V1": "1"})):
        out = str(tmp_path / f"{tag}.npz")
        e = dict(os.environ, **env)
        e.pop("SPLATB200_LIDAR_V1", None) if not env else None
        subprocess.run([_sys.executable, "-c", _LIDAR_PAIR_SCRIPT, out], cwd=root, env=e, check=True, timeout=600)
        outs.append(np.load(out))
    a, b = outs
    assert a["n_contrib"].sum() > 10000
    # hit_bits: which warps blended each list entry — the shared kernels' hit bytes, and the same thing derived from
    # the lidar pair's per-(entry, warp) ray masks
    for k in ("blend", "alpha", "n_contrib", "last_idx", "hit_bits"):
        assert np.array_equal(a[k], b[k]), f"{k}: the two kernel pairs differ"
    for k in ("d_mean", "d_scale_log", "d_quat", "d_opacity_logit", "d_feature"):
        scale = np.abs(b[k]).max()
        assert np.abs(a[k].astype(np.float64) - b[k]).max() <= 1e-4 * scale, k


@pytest.mark.gpu
def test_lidar_kernel_pairs_sweep():
    """scripts/lidar_pair_fuzz.py: seven scenes (sub-ray to tile-filling footprints, anisotropic, fast sensors, ragged ray
    sets) through the lidar kernel pair and through the shared kernels, one process each: every forward output and the
    hit bits bit-identical, gradients equal up to the order of the atomics."""
    import os
    import subprocess
    import sys as _sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([_sys.executable, os.path.join(root, "scripts", "lidar_pair_fuzz.py")], cwd=root, capture_output=True,
                       text=True, timeout=1500, env=dict(os.environ, PYTHONPATH=root))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "all identical" in r.stdout


def test_async_scene_upload_matches_blocking(ctx):
    """splatb200_scene_upload_async (geometry first, colour / features behind it on their own copy stream, projection and
    binning overlapping them; k_project + k_pack_feat instead of the fused k_project): bit-identical renders and
    worklists, identical gradients up to the order of the atomics, for a changed scene of the same shape."""
    sc = synth.make_scene(6000, seed=31, r_max=40.0, scale_mean=0.1)
    lid = synth.lidar32()
    rays = synth.grid_rays(lid)
    cam = synth.make_camera(width=320, height=192)
    ctx.set_view_streams(True)
    ctx.upload_scene(sc)
    vl, vc = ctx.lidar_view(lid, rays, ST), ctx.camera_view(cam, ST)
    sc2 = synth.make_scene(6000, seed=32, r_max=40.0, scale_mean=0.1).astype(np.float32)     # the next iteration's parameters

    def run():
        ctx.zero_grads()
        out = {}
        for name, v in (("l", vl), ("c", vc)):
            v.forward(0.0)
            gb, ga = synth.upstream(v.P, seed=5)
            if name == "l":
                gb[:, 14:] = 0
            v.backward(gb, ga)
            out[name] = {k: v.array(k).copy() for k in ("blend", "alpha", "n_contrib", "last_idx", "isect_src")}
        out["g"] = ctx.grads()
        return out

    ctx.upload_scene(sc2)
    ref = run()
    ctx.upload_scene(sc)               # something else in between
    ctx.upload_scene_async(sc2)
    got = run()
    ctx.sync()
    ctx.set_view_streams(False)
    for name in ("l", "c"):
        for k, a in ref[name].items():
            assert np.array_equal(a, got[name][k]), (name, k)
    # gradients: the same kernels on the same inputs; what differs is the order of the atomic additions, which only the
    # ill-conditioned (grazing) camera rows are sensitive to (tests/grad_gate.py): all but a fraction of a percent of the
    # rows agree to 1e-4 of the group's scale
    for k in ("d_mean", "d_scale_log", "d_quat", "d_opacity_logit", "d_color", "d_feature"):
        a, b = ref["g"][k].astype(np.float64).reshape(sc.n, -1), got["g"][k].astype(np.float64).reshape(sc.n, -1)
        bad = np.abs(a - b).max(axis=1) > 1e-4 * np.abs(a).max()
        assert bad.mean() <= 0.01, (k, bad.mean())


def test_multi_sensor_accumulation_and_reuse(ctx, op):
    """Several sensors over one scene accumulate into one SceneParamGrads; views are reusable across frames."""
    import grad_gate
    sc = synth.make_scene(5000, seed=14, r_max=40.0, scale_mean=0.1)
    ctx.upload_scene(sc)
    o64, o32 = op.OracleScene(sc, np.float64), op.OracleScene(sc, np.float32)
    cams = [synth.make_camera(width=160, height=96, yaw=k * np.pi / 3) for k in range(3)]
    view = ctx.camera_view(cams[0], ST)
    ctx.zero_grads()
    fm, ill = np.zeros(sc.n, bool), np.zeros(sc.n, bool)
    for k, cam in enumerate(cams):
        view.set_camera(cam)
        view.forward(0.0)
        gb, ga = synth.upstream(view.P, seed=20 + k)
        view.backward(gb, ga)
        vs = []
        for o in (o32, o64):
            ov = o.render_camera(cam, ST, workers=8)
            ov.backward(gb, ga, workers=8)
            vs.append(ov)
        if k < len(cams) - 1:       # masks of the earlier sensors (the gate adds the last one's itself)
            fm |= grad_gate.flip_mask(vs[0], vs[1])[1]
            ill |= grad_gate.ill_conditioned(vs[1], cam, sc.n)
    grad_gate.grad_gate(ctx.grads(), o32.grads(), o64.grads(), vs[0], vs[1], cams[-1], sc.n, what="multi-sensor ",
                        extra_mask=(fm, ill))


# ---- BASELINE.json full sizes ------------------------------------------------------------------------
def _worklist_invariants(v, n_tiles):
    """Size-independent properties of the sorted worklist: tiles ascending, depth ascending inside a
    tile, source index ascending among equal depths; tile ranges partition the list."""
    tile, depth, src = v.array("isect_tile"), v.array("isect_depth_bits"), v.array("isect_src")
    tb, te = v.array("tile_begin"), v.array("tile_end")
    assert len(tile) == v.stats()["n_intersections"]
    if len(tile) == 0:
        return
    dt = np.diff(tile)
    assert (dt >= 0).all()
    same_tile = dt == 0
    dd = np.diff(depth)
    assert (dd[same_tile] >= 0).all()
    ties = same_tile & (dd == 0)
    assert (np.diff(src)[ties] > 0).all()
    nonempty = te > tb
    assert int((te - tb).sum()) == len(tile)
    assert (tile[tb[nonempty]] == np.flatnonzero(nonempty)).all() and (tile[te[nonempty] - 1] == np.flatnonzero(nonempty)).all()
    assert tile.max() < n_tiles


@pytest.mark.parametrize("sensor", ["lidar128", "camera1080p"])
def test_full_size_1m_gaussians(ctx, op, sensor):
    """BASELINE configs 2/3 at the north-star size (1M Gaussians): worklist and contributor counts bit-exact against the
    oracle, plus the size-independent properties: sortedness, 0 <= alpha <= 1, backward linear in the upstream
    gradient, zero upstream => zero gradients, accumulation (+=)."""
    n = 1_000_000
    sc = synth.make_scene(n, seed=3)
    ctx.upload_scene(sc)
    if sensor == "lidar128":
        lid = synth.lidar128()
        rays = synth.grid_rays(lid)
        gv = ctx.render_lidar(lid, rays, ST)
        ov = op.OracleScene(sc, np.float32).render_lidar(lid, rays, ST, workers=op.hardware_threads())
    else:
        cam = synth.make_camera()
        gv = ctx.render_camera(cam, ST)
        ov = op.OracleScene(sc, np.float32).render_camera(cam, ST, workers=op.hardware_threads())
    st = gv.stats()
    _worklist_invariants(gv, st["tiles_x"] * st["tiles_y"])
    for f in ("source_index", "isect_tile", "isect_src", "tile_begin", "tile_end", "n_contrib", "last_idx"):
        assert np.array_equal(gv.array(f), ov.array(f)), f
    assert_render_close(gv, ov, sensor == "lidar128")
    a = gv.array("alpha")
    assert a.min() >= 0.0 and a.max() <= 1.0
    # backward: linearity / zero / accumulation
    gb, ga = synth.upstream(gv.P, seed=1)
    if sensor == "lidar128":
        gb[:, 14:] = 0
    ctx.zero_grads()
    gv.backward(np.zeros_like(gb), np.zeros_like(ga))
    assert all(np.all(x == 0) for k, x in ctx.grads().items() if k != "actors")
    gv.backward(gb, ga)
    g1 = ctx.grads()
    ctx.zero_grads()
    gv.backward(2.0 * gb, 2.0 * ga)
    g2 = ctx.grads()
    for k in ("d_mean", "d_scale_log", "d_quat", "d_opacity_logit", "d_color", "d_feature"):
        x, y = g2[k].reshape(n, -1).astype(np.float64), 2.0 * g1[k].reshape(n, -1).astype(np.float64)
        if np.abs(y).max() == 0:        # lidar renders no colour
            assert np.abs(x).max() == 0, k
            continue
        rel = np.abs(x - y).max(1) / np.maximum(np.abs(y).max(1), 1e-3 * np.abs(y).max())
        assert np.quantile(rel, 0.99) <= 1e-3 and np.isfinite(x).all(), (k, np.quantile(rel, 0.99))


# ---- gradient parity at the BASELINE sizes --------------------------------------------------
@pytest.mark.parametrize("near_plane", [None, 1.0])
def test_cfg2_camera_100k_forward_backward(ctx, op, near_plane):
    """BASELINE config 2: 100k Gaussians, 1920x1080 rolling-shutter camera, forward + backward, against the oracle at
    full size: projection, stored records, worklist and contributor counts bit-exact, render <= 1e-4, SceneParamGrads
    through the gradient gate. near_plane = None is synth-v1 as specified: ~2 % of the visible Gaussians lie at grazing
    depth and cover every tile (no tan-FOV clamp in the reference), so most pixels see an fp32/fp64 forward flip and G2
    has few rows left — G1 (100 % of the rows against the reference algorithm in fp32) carries that case. With
    near_plane = 1 m (the same code path; the grazing Gaussians are culled by the reference's own rule,
    projection.hpp:99) G2 covers >= 90 % of the live rows."""
    import dataclasses
    st = ST if near_plane is None else dataclasses.replace(ST, near_plane=near_plane)
    n = 100_000
    sc = synth.make_scene(n, seed=3)
    cam = synth.make_camera()
    ctx.upload_scene(sc)
    gv = ctx.render_camera(cam, st)
    W = op.hardware_threads()
    ov = op.OracleScene(sc, np.float32).render_camera(cam, st, workers=W)
    assert_projection_bit_exact(gv, ov, sc)
    assert_worklist_bit_exact(gv, ov)
    assert_render_close(gv, ov, False)
    gb, ga = synth.upstream(gv.P, seed=1)
    og = oracle_grads(op, sc, lambda o: o.render_camera(cam, st, workers=W), gb, ga)
    ctx.zero_grads()
    gv.backward(gb, ga)
    grads_gate(ctx, og, cam, n, what=f"cfg2 near_plane={near_plane} ", workers=W, max_ill_frac=0.03,
               max_flip_frac=None if near_plane is None else 0.10)
    if near_plane is not None:
        assert_sensor_grads(gv, og)


def test_cfg3_lidar128_1m_forward_backward(ctx, op):
    """BASELINE config 3: 1M Gaussians, 128-beam lidar with non-uniform elevation and rolling shutter, forward + backward
    incl. the feature channels standing in for intensity and ray-drop: SceneParamGrads and SensorGrads of the full-size
    sweep against the oracle (the worklist / contributor counts of this configuration are in
    test_full_size_1m_gaussians)."""
    n = 1_000_000
    sc = synth.make_scene(n, seed=3)
    lid = synth.lidar128()
    rays = synth.grid_rays(lid)
    ctx.upload_scene(sc)
    gv = ctx.render_lidar(lid, rays, ST)
    gb, ga = synth.upstream(gv.P, seed=1)
    gb[:, 14:] = 0
    W = op.hardware_threads()
    og = oracle_grads(op, sc, lambda o: o.render_lidar(lid, rays, ST, workers=W), gb, ga)
    assert np.array_equal(gv.array("n_contrib"), og[0][1].array("n_contrib"))
    ctx.zero_grads()
    gv.backward(gb, ga)
    grads_gate(ctx, og, lid, n, what="cfg3 ", workers=W, max_flip_frac=0.05)
    assert_sensor_grads(gv, og)


def test_cfg4_dynamic_3m_cropped_sensors_match_oracle(ctx, op):
    """BASELINE config 4's scene (3M Gaussians, 32 moving actors) against the oracle on sensors small enough for the CPU:
    a 480 x 270 camera of the rig (same field of view) and the 32-beam lidar. Everything the small dynamic test checks,
    at 3M: composed fields, projection, stored records, worklists and contributor counts bit-exact; render <= 1e-4;
    SceneParamGrads through the gate; actor pose / velocity offset gradients."""
    n = 3_000_000
    sc = synth.make_scene(n, seed=4, n_actors=32, dynamic_fraction=0.02)
    t_scene = 0.05
    ctx.upload_scene(sc)
    W = op.hardware_threads()
    cam = synth.make_camera(width=480, height=270, yaw=np.pi / 3.0)
    lid = synth.lidar32()
    lid.vel_lin, lid.vel_ang = np.array([12.0, 1.0, 0.0]), np.array([0.0, 0.02, 0.3])
    rays = synth.grid_rays(lid)
    for name, sensor in (("camera", cam), ("lidar", lid)):
        camera = name == "camera"
        gv = ctx.render_camera(cam, ST, t_scene=t_scene) if camera else ctx.render_lidar(lid, rays, ST, t_scene=t_scene)
        render = (lambda o: o.render_camera(cam, ST, t_scene=t_scene, workers=W)) if camera else \
                 (lambda o: o.render_lidar(lid, rays, ST, t_scene=t_scene, workers=W))
        gb, ga = synth.upstream(gv.P, seed=7)
        if not camera:
            gb[:, 14:] = 0
        og = oracle_grads(op, sc, render, gb, ga)
        ov = og[0][1]
        if camera:
            for f in ("mean_w", "vel_dyn_w", "opacity", "cov_w"):
                assert np.array_equal(bits(gv.array(f)), bits(ov.array(f))), f
        assert_projection_bit_exact(gv, ov, sc)
        assert_worklist_bit_exact(gv, ov)
        assert_render_close(gv, ov, not camera)
        dyn = np.isin(gv.array("source_index"), np.nonzero(sc.actor_id)[0]).sum()
        assert dyn > 100, dyn
        ctx.zero_grads()
        gv.backward(gb, ga)
        grads_gate(ctx, og, sensor, n, what=f"cfg4 {name} ", workers=W, max_ill_frac=0.03, max_flip_frac=None if camera else 0.05)
        g, (g32, _), (g64, _) = ctx.grads(), og[0], og[1]
        for a in range(len(sc.tracks)):
            for k in ("d_pose_offset", "d_vel_offset"):
                x, r, y = g["actors"][a][k], g32["actors"][a][k].reshape(g["actors"][a][k].shape), g64["actors"][a][k].reshape(g["actors"][a][k].shape)
                assert np.abs(x - y).max() <= 2e-3 * max(np.abs(y).max(), 1e-6) + 5 * np.abs(r - y).max(), (name, a, k)
        del gv, og, ov


@pytest.mark.parametrize("scale_mean,speed", [(0.01, 30.0), (0.3, 60.0), (1.5, 5.0)])
def test_per_warp_culling_is_sound(ctx, op, scale_mean, speed):
    """The compositing kernels drop (Gaussian, patch) pairs with a conservative bound before evaluating them
    (raster_common.cuh). Contributor counts and last-blended positions must stay bit-identical to the oracle, which
    evaluates every pair, across footprint sizes (sub-pixel to tile-filling, strongly anisotropic) and fast sensors
    (large rolling-shutter shifts)."""
    sc = synth.make_scene(6000, seed=int(scale_mean * 100) + 50, r_max=25.0, scale_mean=scale_mean)
    sc.scale_log[:, 0] += 1.5        # anisotropic: one long axis
    ctx.upload_scene(sc)
    cam = synth.make_camera(width=256, height=160, time_offset=0.004)
    cam.vel_lin, cam.vel_ang = np.array([2.0, 0.0, speed]), np.array([0.3, 0.5, 0.1])
    gv = ctx.render_camera(cam, ST)
    ov = op.OracleScene(sc, np.float32).render_camera(cam, ST, workers=8)
    assert_worklist_bit_exact(gv, ov)
    assert_render_close(gv, ov, False)
    lid = synth.lidar128()
    lid.vel_lin, lid.vel_ang = np.array([speed, 3.0, 0.0]), np.array([0.0, 0.05, 1.0])
    rays = synth.grid_rays(lid)
    gl = ctx.render_lidar(lid, rays, ST)
    ol = op.OracleScene(sc, np.float32).render_lidar(lid, rays, ST, workers=8)
    assert_worklist_bit_exact(gl, ol)
    assert_render_close(gl, ol, True)
    # and the backward pass revisits exactly those pairs: gradients agree with the fp64 oracle (checked where fp32 is
    # well conditioned: with 1 cm Gaussians the footprint is all dilation and the reference's own fp32 mode misses 1e-3
    # on 5-8% of the rows)
    if scale_mean < 0.1:
        return
    gb, ga = synth.upstream(gl.P, seed=9)
    gb[:, 14:] = 0
    og = oracle_grads(op, sc, lambda o: o.render_lidar(lid, rays, ST, workers=8), gb, ga)
    ctx.zero_grads()
    gl.backward(gb, ga)
    grads_gate(ctx, og, lid, sc.n, what=f"cull lidar s={scale_mean} ")


def test_near_singular_conics(api, op, monkeypatch):
    """Adversarial numerics (raster_common.cuh alpha_finish): needle Gaussians (one axis 1e-4 of the others) with almost
    no dilation give near-singular 2-D covariances, conic entries ~1e8 with cancelling terms, and quadratic forms whose
    fp32 evaluation is noise of either sign — including hugely negative ones, outside exp_bounded's proven range unless
    the argument is clamped. Contributor counts, last-blended positions and the blend must still follow the oracle bit for
    bit / to 1e-4; a record with non-finite fields is counted and never blended."""
    import dataclasses
    monkeypatch.setenv("SPLATB200_STATS", "1")
    st = dataclasses.replace(ST, dilation=1e-7)
    sc = synth.make_scene(4000, seed=41, r_max=25.0, scale_mean=0.3)
    sc.scale_log[:, 0] += 2.0
    sc.scale_log[:, 1] -= 9.0            # needles
    sc.opacity_logit[:] = 4.0
    sc.mean[7] = np.array([np.inf, 0.0, 0.0], np.float32)     # a Gaussian whose record is non-finite
    sc.mean[8] = np.array([np.nan, 2.0, 1.0], np.float32)
    c = api.Context(0)
    try:
        c.upload_scene(sc)
        cam = synth.make_camera(width=256, height=160)
        gv = c.render_camera(cam, st)
        ov = op.OracleScene(sc, np.float32).render_camera(cam, st, workers=8)
        assert_worklist_bit_exact(gv, ov)
        assert_render_close(gv, ov, False)
        qneg = 0
        lid = synth.lidar32()
        rays = synth.grid_rays(lid)
        gl = c.render_lidar(lid, rays, st)
        ol = op.OracleScene(sc, np.float32).render_lidar(lid, rays, st, workers=8)
        assert_worklist_bit_exact(gl, ol)
        assert_render_close(gl, ol, True)
        assert np.isfinite(gv.array("blend")).all() and np.isfinite(gl.array("blend")).all()
        assert gv.array("n_contrib").max() > 3
        src = set(gv.array("source_index").tolist()) | set(gl.array("source_index").tolist())
        assert 7 not in src and 8 not in src        # culled by the projection (non-finite depth), never staged
        assert gv.array("raster_stats")[4] == 0
    finally:
        c.close()


# ---- binning variants --------------------------------------------------------------------------------
def test_camera_one_level_binning_matches_two_level(api, op, monkeypatch):
    """Cameras bin in two levels (8x8-tile blocks sorted, then expanded into tile lists); SPLATB200_ONE_LEVEL selects the
    plain one-level sort. Both must produce the oracle's worklist bit for bit, on an image whose tile grid is not a
    multiple of the block size."""
    sc = synth.make_scene(12000, seed=21, r_max=40.0, scale_mean=0.1)
    cam = synth.make_camera(width=600, height=330, time_offset=0.001)   # 38 x 21 tiles -> 5 x 3 blocks, ragged
    ov = op.OracleScene(sc, np.float32).render_camera(cam, ST, workers=8)
    for one_level in (False, True):
        if one_level:
            monkeypatch.setenv("SPLATB200_ONE_LEVEL", "1")
        c = api.Context(0)
        try:
            c.upload_scene(sc)
            gv = c.render_camera(cam, ST)
            assert_worklist_bit_exact(gv, ov)
            assert_render_close(gv, ov, False)
        finally:
            c.close()


def test_large_tile_grid(ctx, op):
    """A 4K-wide image: 240 x 68 = 16,320 tiles (two 7-bit radix passes at block level would be one; the tile scan
    still fits shared memory) and a 5,120 x 2,880 one: 320 x 180 = 57,600 tiles, whose tile scan takes the
    global-memory path. Few Gaussians, so the oracle stays fast."""
    sc = synth.make_scene(1500, seed=22, r_max=30.0, scale_mean=0.2)
    ctx.upload_scene(sc)
    for w, h in ((3840, 1080), (5120, 2880)):
        cam = synth.make_camera(width=w, height=h)
        gv = ctx.render_camera(cam, ST)
        ov = op.OracleScene(sc, np.float32).render_camera(cam, ST, workers=8)
        assert_worklist_bit_exact(gv, ov)
        assert np.array_equal(gv.array("n_contrib"), ov.array("n_contrib"))


def test_backward_is_repeatable_after_new_forward(ctx, op):
    """The backward pass revisits the entries the forward pass marked (hit bytes): a second forward with another pose
    must re-mark them, and gradients must follow the new render (all but the ill-conditioned grazing rows within 1e-3
    of the fp64 oracle, exactly as for a fresh view)."""
    sc = synth.make_scene(6000, seed=23, r_max=40.0, scale_mean=0.1)
    ctx.upload_scene(sc)
    view = ctx.camera_view(synth.make_camera(width=320, height=192), ST)
    o64 = op.OracleScene(sc, np.float64)
    gb, ga = synth.upstream(view.P, seed=5)
    for yaw in (0.0, 0.7, 0.0):
        cam2 = synth.make_camera(width=320, height=192, yaw=yaw)
        view.set_camera(cam2)
        view.forward(0.0)
        ctx.zero_grads()
        view.backward(gb, ga)
        o64.zero_grads()
        ov = o64.render_camera(cam2, ST, workers=8)
        ov.backward(gb, ga, workers=8)
        o32 = op.OracleScene(sc, np.float32)
        ov32 = o32.render_camera(cam2, ST, workers=8)
        ov32.backward(gb, ga, workers=8)
        assert np.array_equal(view.array("n_contrib"), ov32.array("n_contrib"))
        grads_gate(ctx, [(o32.grads(), ov32), (o64.grads(), ov)], cam2, sc.n, what=f"yaw {yaw} ")


def test_config4_scale_dynamic_3m(ctx):
    """BASELINE config 4's size (3M Gaussians, 32 moving actors; one of the 6 cameras + the lidar of a frame): too large
    for the CPU oracle inside a test, so the size-independent properties are checked — worklist order and tile ranges,
    0 <= alpha <= 1, contributor counts consistent with the saved list positions, backward linear in the upstream
    gradient, zero upstream => zero gradients."""
    n = 3_000_000
    sc = synth.make_scene(n, seed=4, n_actors=32, dynamic_fraction=0.02)
    ctx.upload_scene(sc)
    lid = synth.lidar128()
    views = [("camera", ctx.camera_view(synth.make_camera(yaw=np.pi / 3.0), ST)), ("lidar", ctx.lidar_view(lid, synth.grid_rays(lid), ST))]
    for name, v in views:
        v.forward(0.05)
        st = v.stats()
        assert st["n_visible"] > 100_000 and st["n_intersections"] > st["n_visible"]
        _worklist_invariants(v, st["tiles_x"] * st["tiles_y"])
        a = v.array("alpha")
        assert a.min() >= 0.0 and a.max() <= 1.0 and np.isfinite(v.array("blend")).all()
        nc, li = v.array("n_contrib"), v.array("last_idx")
        assert (nc <= li).all() and ((nc == 0) == (li == 0)).all()
        gb, ga = synth.upstream(v.P, seed=9)
        if name == "lidar":
            gb[:, 14:] = 0
        ctx.zero_grads()
        v.backward(np.zeros_like(gb), np.zeros_like(ga))
        g0 = ctx.grads()
        assert all(np.count_nonzero(g0[k]) == 0 for k in ("d_mean", "d_color", "d_feature", "d_quat"))
        v.backward(gb, ga)
        g1 = {k: x.copy() for k, x in ctx.grads().items() if k != "actors"}
        ctx.zero_grads()
        v.backward(2.0 * gb, 2.0 * ga)
        g2 = ctx.grads()
        for k in ("d_mean", "d_opacity_logit", "d_color", "d_feature"):
            x, y = g2[k].reshape(n, -1).astype(np.float64), 2.0 * g1[k].reshape(n, -1).astype(np.float64)
            if np.abs(y).max() == 0:        # lidar renders no colour
                assert np.abs(x).max() == 0, k
                continue
            rel = np.abs(x - y).max(1) / np.maximum(np.abs(y).max(1), 1e-3 * np.abs(y).max())
            assert np.quantile(rel, 0.99) <= 1e-3 and np.isfinite(x).all(), (name, k, np.quantile(rel, 0.99))
        assert np.isfinite(g2["d_mean"]).all() and np.count_nonzero(g2["d_mean"]) > 0


def test_overlapped_host_buffer_calls(ctx):
    """download_async / backward_host_overlapped (copies on the library's own copy streams) give the same outputs and
    gradients as the synchronous host-buffer calls, over several steps with two views in flight."""
    import torch

    def pinned(shape, dtype):
        t = torch.empty(shape, dtype=dtype, pin_memory=True)
        return t, t.numpy()

    sc = synth.make_scene(20000, seed=31, r_max=40.0, scale_mean=0.1)
    ctx.upload_scene(sc)
    lid = synth.lidar32()
    vl = ctx.lidar_view(lid, synth.grid_rays(lid), ST)
    vc = ctx.camera_view(synth.make_camera(width=640, height=528), ST)
    keep, host = [], {}
    for name, v in (("l", vl), ("c", vc)):
        gb, ga = synth.upstream(v.P, seed=3)
        if name == "l":
            gb[:, 14:] = 0
        tb, vb = pinned((v.P, 16), torch.float32); ta, va = pinned((v.P,), torch.float32); tn, vn = pinned((v.P,), torch.int32)
        tgb, hgb = pinned(gb.shape, torch.float32); tga, hga = pinned(ga.shape, torch.float32)
        hgb[...] = gb; hga[...] = ga
        keep += [tb, ta, tn, tgb, tga]
        host[name] = (vb, va, vn, hgb, hga)
    # synchronous reference
    ctx.zero_grads()
    ref_out = {}
    for name, v in (("l", vl), ("c", vc)):
        v.forward(0.0)
        vb, va, vn, hgb, hga = host[name]
        v.download(vb, va, vn)
        ref_out[name] = (vb.copy(), va.copy(), vn.copy())
        v.backward_host_async(hgb, hga)
    g_ref = {k: x.copy() for k, x in ctx.grads().items() if k != "actors"}
    for step in range(5):
        ctx.zero_grads()
        for name, v in (("l", vl), ("c", vc)):
            vb, va, vn, _, _ = host[name]
            vb[...] = -1; va[...] = -1; vn[...] = -1
            if step < 2:
                v.forward(0.0)
                v.download_async(vb, va, vn)
            else:       # fused, banded forms (camera: 1, 3 and 8 bands over 33 tile rows)
                v.forward_to_host(0.0, vb, va, vn, bands=(1, 3, 8)[step - 2])
        for name, v in (("l", vl), ("c", vc)):
            if step < 2:
                v.backward_host_overlapped(host[name][3], host[name][4])
            else:
                v.backward_from_host(host[name][3], host[name][4])
        g = ctx.grads()          # synchronises the compute stream
        ctx.sync()
        for name in ("l", "c"):
            for a, b in zip(host[name][:3], ref_out[name]):
                assert np.array_equal(a, b), (step, name)
        for k, y in g_ref.items():
            x = g[k].astype(np.float64).reshape(sc.n, -1)
            y = y.astype(np.float64).reshape(sc.n, -1)
            rel = np.abs(x - y).max(1) / np.maximum(np.abs(y).max(1), 1e-3 * max(np.abs(y).max(), 1e-30))
            assert np.quantile(rel, 0.99) <= 1e-3, (step, k)


def test_view_streams_match_single_stream(ctx):
    """splatb200_ctx_set_view_streams: two views on their own streams produce the single-stream outputs bit for bit and
    the same accumulated gradients, over repeated frames (ordering against zero_grads / scene re-upload / download)."""
    sc = synth.make_scene(30000, seed=41, r_max=40.0, scale_mean=0.1)
    ctx.upload_scene(sc)
    lid = synth.lidar32()
    vl = ctx.lidar_view(lid, synth.grid_rays(lid), ST)
    vc = ctx.camera_view(synth.make_camera(width=640, height=360), ST)
    ups = {}
    for name, v in (("l", vl), ("c", vc)):
        gb, ga = synth.upstream(v.P, seed=5)
        if name == "l":
            gb[:, 14:] = 0
        ups[name] = (gb, ga)

    def frame():
        ctx.upload_scene(sc)
        ctx.zero_grads()
        for name, v in (("l", vl), ("c", vc)):
            v.forward(0.0)
            v.backward(*ups[name])
        ctx.join()
        g = {k: x.copy() for k, x in ctx.grads().items() if k != "actors"}
        return g, {n: (v.array("blend").copy(), v.array("n_contrib").copy()) for n, v in (("l", vl), ("c", vc))}

    g_ref, out_ref = frame()
    ctx.set_view_streams(True)
    try:
        for _ in range(4):
            g, out = frame()
            for n in ("l", "c"):
                assert np.array_equal(out[n][0], out_ref[n][0]) and np.array_equal(out[n][1], out_ref[n][1]), n
            for k, y in g_ref.items():
                x, y2 = g[k].astype(np.float64).reshape(sc.n, -1), y.astype(np.float64).reshape(sc.n, -1)
                rel = np.abs(x - y2).max(1) / np.maximum(np.abs(y2).max(1), 1e-3 * max(np.abs(y2).max(), 1e-30))
                assert np.quantile(rel, 0.99) <= 1e-3, k
    finally:
        ctx.set_view_streams(False)


@pytest.mark.parametrize("n", [0, 1, 2, 31, 4095, 4096, 4097, 8192, 100_003, 1_000_000])
def test_radix_sort_and_count_scan(ctx, n):
    """The hand-written onesweep radix sort + look-back scan against numpy on adversarial inputs: partial and exactly
    full 4,096-item tiles, all keys equal (stability = identity), two values, sorted / reversed, random 32-bit, keys that
    differ only in one byte."""
    rng = np.random.default_rng(n + 7)
    cases = {
        "random": rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32),
        "equal": np.full(n, 0x3f800000, np.uint32),
        "two": np.where(rng.random(n) < 0.5, 0xffffffff, 0x41200000).astype(np.uint32),
        "sorted": np.arange(n, dtype=np.uint32) * 3,
        "reversed": (np.arange(n, dtype=np.uint32)[::-1] * 5).copy(),
        "byte2": (rng.integers(0, 256, n, dtype=np.uint64).astype(np.uint32) << 16) | 0x40000000,
        "depths": np.abs(rng.normal(20.0, 15.0, n)).astype(np.float32).view(np.uint32),
    }
    counts = rng.integers(0, 1000, n, dtype=np.uint64).astype(np.uint32)   # totals stay below 2^30 (the per-view limit)
    for name, keys in cases.items():
        order, offsets = ctx.debug_depth_sort(keys, counts)
        ref = np.argsort(keys, kind="stable").astype(np.uint32)
        assert np.array_equal(order, ref), (name, n)
        ref_off = np.concatenate([[0], np.cumsum(counts[ref].astype(np.uint64))]).astype(np.uint64) & 0xffffffff
        assert np.array_equal(offsets.astype(np.uint64), ref_off), (name, n)


# ---- assign_points_to_tiles: the producer of the lidar views' rays -------------------------
@pytest.mark.parametrize("train", [False, True])
def test_assign_points_matches_oracle(ctx, op, train):
    """Per-point tile ids and (azimuth, elevation, t_l, range) bit-identical to the fp32 oracle, same tile-major order and
    slices, same rejected / dropped counts — moving sensor, real timestamps, non-finite points, an overfull tile."""
    lid = synth.lidar128()
    rng = np.random.default_rng(5)
    n = 250_000
    pts = rng.normal(0, 25, (n, 3)).astype(np.float32) + np.array([0, 0, 1.0], np.float32)
    pts[::5000] = np.nan
    pts[1234] = np.inf
    hot = pts[777] * np.linspace(1.0, 1.05, 600, dtype=np.float32)[:, None]     # 600 returns on one ray: an overfull tile
    pts = np.concatenate([pts, hot]).astype(np.float32)
    ts = (rng.uniform(-0.05, 0.05, len(pts)) + lid.timestamp).astype(np.float32)
    g = ctx.assign_points_to_tiles(lid, pts, ts, train=train, seed=11)
    o = op.assign_points_to_tiles(lid, pts, ts, train=train, seed=11, dtype=np.float32)
    assert np.array_equal(g["tile"], o["tile"])
    for k in ("phi", "omega", "t_l", "range"):
        assert np.array_equal(bits(g[k]), bits(o[k])), k
    assert g["rejected"] == o["rejected"] > 0 and g["dropped"] == o["dropped"]
    assert (g["dropped"] > 0) == train
    assert np.array_equal(g["order"], o["order"]) and np.array_equal(g["begin"], o["begin"]) and np.array_equal(g["end"], o["end"])
    counts = g["end"] - g["begin"]
    assert counts.max() > 256 if not train else counts.max() == 256


def test_render_from_assigned_points(ctx, op):
    """End to end on the input side: returns of a moving lidar -> assign_points_to_tiles -> view -> render, against the
    oracle fed with the oracle's own assignment (contributor counts bit-exact, outputs within 1e-4)."""
    sc = synth.make_scene(20000, seed=9, r_max=40.0, scale_mean=0.15)
    lid = synth.lidar128()
    rng = np.random.default_rng(6)
    pts = (rng.normal(0, 20, (60_000, 3)) + np.array([0, 0, 1.0])).astype(np.float32)
    ts = (rng.uniform(-0.05, 0.05, len(pts)) + lid.timestamp).astype(np.float32)
    g = ctx.assign_points_to_tiles(lid, pts, ts)
    o = op.assign_points_to_tiles(lid, pts, ts, dtype=np.float32)
    from paper_2411_16816_b200.model import RaySet
    ors = RaySet(rays=np.stack([o["phi"], o["omega"], o["t_l"]], 1)[o["order"]].astype(np.float32), begin=o["begin"], end=o["end"])
    assert np.array_equal(bits(g["rayset"].rays), bits(ors.rays))
    ctx.upload_scene(sc)
    gv = ctx.render_lidar(lid, g["rayset"], ST)
    ov = op.OracleScene(sc, np.float32).render_lidar(lid, ors, ST, workers=8)
    assert_render_close(gv, ov, True)


def test_view_set_rays_per_frame_sweeps(ctx, op):
    """One lidar view, a new sweep every frame (assign_points -> set_rays): sweeps of different sizes, growing past the
    initial capacity, each rendered and differentiated; outputs match the oracle, gradients match a fresh view."""
    sc = synth.make_scene(15000, seed=12, r_max=40.0, scale_mean=0.15)
    ctx.upload_scene(sc)
    lid = synth.lidar128()
    rng = np.random.default_rng(8)
    view = None
    for n_pts in (20_000, 8_000, 45_000):
        pts = (rng.normal(0, 20, (n_pts, 3)) + np.array([0, 0, 1.0])).astype(np.float32)
        ts = (rng.uniform(-0.05, 0.05, n_pts) + lid.timestamp).astype(np.float32)
        a = ctx.assign_points_to_tiles(lid, pts, ts)
        if view is None:
            view = ctx.lidar_view(lid, a["rayset"], ST)
        else:
            view.set_rays(a["rayset"])
        view.forward(0.0)
        ov = op.OracleScene(sc, np.float32).render_lidar(lid, a["rayset"], ST, workers=8)
        assert_render_close(view, ov, True)
        gb, ga = synth.upstream(view.P, seed=n_pts)
        gb[:, 14:] = 0
        ctx.zero_grads()
        view.backward(gb, ga)
        g = {k: x.copy() for k, x in ctx.grads().items() if k != "actors"}
        fresh = ctx.lidar_view(lid, a["rayset"], ST)
        fresh.forward(0.0)
        ctx.zero_grads()
        fresh.backward(gb, ga)
        g2 = ctx.grads()
        for k, y in g.items():
            x, y2 = g2[k].astype(np.float64).reshape(sc.n, -1), y.astype(np.float64).reshape(sc.n, -1)
            rel = np.abs(x - y2).max(1) / np.maximum(np.abs(y2).max(1), 1e-3 * max(np.abs(y2).max(), 1e-30))
            assert np.quantile(rel, 0.99) <= 1e-3, (n_pts, k)


# ---- line-of-sight channel ------------------------------------------------
def test_line_of_sight_channel(ctx, op):
    """los[q] = sum of alpha_i in front of the per-ray cut: bit-identical to the fp32 oracle (same additions in the same
    order); its upstream gradient reaches the parameters like the fp64 oracle's; switching the channel off restores the
    plain render; the cuts come from assign_points' measured ranges."""
    sc = synth.make_scene(20000, seed=14, r_max=40.0, scale_mean=0.15)
    ctx.upload_scene(sc)
    lid = synth.lidar128()
    rng = np.random.default_rng(9)
    pts = (rng.normal(0, 20, (50_000, 3)) + np.array([0, 0, 1.0])).astype(np.float32)
    ts = (rng.uniform(-0.05, 0.05, len(pts)) + lid.timestamp).astype(np.float32)
    a = ctx.assign_points_to_tiles(lid, pts, ts)
    rs = a["rayset"]
    cut = (a["range"][a["order"]] - 0.8).astype(np.float32)       # r_p - eps, in ray order
    view = ctx.lidar_view(lid, rs, ST)
    view.set_los(cut)
    view.forward(0.0)
    o32, o64 = op.OracleScene(sc, np.float32), op.OracleScene(sc, np.float64)
    ov32 = o32.render_lidar(lid, rs, ST, workers=8)
    ov32.set_los(cut, workers=8)
    los, olos = view.array("los"), ov32.array("los")
    assert np.count_nonzero(olos) > 1000
    assert np.array_equal(bits(los), bits(olos))
    assert_render_close(view, ov32, True)
    # backward: only the line-of-sight gradient
    g_los = rng.normal(size=view.P).astype(np.float32)
    zb, za = np.zeros((view.P, 16), np.float32), np.zeros(view.P, np.float32)
    ctx.zero_grads()
    view.set_los_grad(g_los)
    view.backward(zb, za)
    ovs = []
    for o in (o32, o64):
        o.zero_grads()
        ov = o.render_lidar(lid, rs, ST, workers=8)
        ov.set_los(cut, workers=8)
        ov.set_los_grad(g_los)
        ov.backward(zb, za, workers=8)
        ovs.append(ov)
    grads_gate(ctx, [(o32.grads(), ovs[0]), (o64.grads(), ovs[1])], lid, sc.n, what="los ")
    assert np.abs(ctx.grads()["d_opacity_logit"]).max() > 0
    # off again: no accumulator, no gradient from it
    view.set_los(None)
    view.forward(0.0)
    ctx.zero_grads()
    view.backward(zb, za)
    assert all(np.count_nonzero(x) == 0 for k, x in ctx.grads().items() if k != "actors")


# ---- lidar head ---------------------------------------------------------
def test_lidar_head_matches_oracle(ctx, op):
    """decode_lidar over a rendered sweep: intensity / ray-drop within 1e-4 of the fp32 oracle; weight gradients and the
    feature gradient (added into the compositing upstream buffer) within 1e-3 of the fp64 oracle; the combined backward
    — head + rasterizer — equals the rasterizer backward fed with the oracle's feature gradient."""
    import torch
    sc = synth.make_scene(15000, seed=16, r_max=40.0, scale_mean=0.15)
    ctx.upload_scene(sc)
    lid = synth.lidar128()
    rs = synth.grid_rays(lid)
    view = ctx.lidar_view(lid, rs, ST)
    view.forward(0.0)
    P, d_f = view.P, sc.d_f
    rng = np.random.default_rng(11)
    w = rng.normal(0, 0.3, op.lidar_head_params(d_f)).astype(np.float32)
    feat = view.array("blend").reshape(P, 16)[:, :d_f]
    sph = rs.rays[:, :2]
    y = view.lidar_head_forward(w)
    oy = op.lidar_head_forward(w, feat, sph, np.float32)
    assert y.min() > 0 and y.max() < 1
    assert np.abs(y - oy).max() <= RENDER_RTOL
    # the fused form: decoded in the compositing kernel's epilogue
    view.set_lidar_head(w)
    view.forward(0.0)
    yf = view.array("lidar_head").reshape(P, 2)
    assert np.abs(yf - oy).max() <= RENDER_RTOL and np.abs(yf - y).max() <= 1e-6
    assert np.array_equal(view.array("blend").reshape(P, 16)[:, :d_f], feat)
    view.set_lidar_head(None)
    view.forward(0.0)
    g_y = rng.normal(size=(P, 2)).astype(np.float32)
    g_up = torch.zeros((P, 16), dtype=torch.float32, device="cuda")
    g_up[:, 3] = 0.25                                   # some other upstream gradient of the render: must be kept
    gw = view.lidar_head_backward(w, g_y, g_up.data_ptr())
    ogw, ogf = op.lidar_head_backward(w, feat, sph, g_y, np.float64)
    assert np.abs(gw - ogw).max() <= GRAD_RTOL * np.abs(ogw).max()
    gf = g_up.cpu().numpy()
    exp = np.zeros((P, 16)); exp[:, :d_f] = ogf; exp[:, 3] += 0.25
    assert np.abs(gf - exp).max() <= GRAD_RTOL * np.abs(exp).max()
    # head + rasterizer backward in one go
    ga = torch.zeros(P, dtype=torch.float32, device="cuda")
    ctx.zero_grads()
    view.backward_device(g_up.data_ptr(), ga.data_ptr())
    g1 = {k: x.copy() for k, x in ctx.grads().items() if k != "actors"}
    ctx.zero_grads()
    view.backward(exp.astype(np.float32), np.zeros(P, np.float32))
    g2 = ctx.grads()
    for k, a in g1.items():
        b = g2[k]
        assert np.abs(a - b).max() <= 2e-3 * max(np.abs(b).max(), 1e-30), k


# ---- optimizer step -------------------------------------------------------
def test_optimizer_step_matches_oracle(ctx, op):
    """Adam on the resident scene from the resident gradients: five steps of render -> backward -> step follow the numpy
    oracle (fp32 arithmetic, 1e-5 relative on the parameters); a non-finite gradient skips exactly its group."""
    import torch
    cfg = {"lr_init": [1.6e-4, 5e-3, 1e-3, 5e-2, 2.5e-3, 2.5e-3], "lr_final": [1.6e-6, 5e-3, 1e-3, 5e-2, 2.5e-3, 2.5e-4],
           "warmup_steps": [0, 0, 0, 0, 0, 3], "total_steps": 10}
    sc = synth.make_scene(50_001, seed=18, r_max=40.0, scale_mean=0.1)
    ctx.upload_scene(sc)
    n = sc.n
    grads_t = torch.zeros(ctx.grads_size, dtype=torch.float32, device="cuda")
    ctx.bind_grads_device(grads_t.data_ptr(), ctx.grads_size)
    p = [np.ascontiguousarray(a, np.float32).reshape(n, -1).copy() for a in (sc.mean, sc.scale_log, sc.quat, sc.opacity_logit, sc.color, sc.feature)]
    m, v = [np.zeros_like(a) for a in p], [np.zeros_like(a) for a in p]
    widths = [3, 3, 4, 1, 3, sc.d_f]
    rng = np.random.default_rng(2)
    for step in range(5):
        g_all = (rng.normal(size=ctx.grads_size) * 10.0 ** rng.uniform(-4, 1)).astype(np.float32)
        if step == 3:
            g_all[3 * n * 2 + 17] = np.inf          # somewhere in the quat slice
        grads_t.copy_(torch.from_numpy(g_all))
        g, o = [], 0
        for w in widths:
            g.append(g_all[o:o + w * n].reshape(n, w)); o += w * n
        skipped = ctx.optimizer_step(cfg, step)
        oskipped = op.adam_step(p, g, m, v, cfg, step, np.float32)
        assert skipped == oskipped == ([2] if step == 3 else [])
        for a, b in zip(ctx.download_scene(), p):
            assert np.abs(a.reshape(b.shape) - b).max() <= 1e-5 * max(np.abs(b).max(), 1.0), step


def test_training_loop_reduces_the_loss(ctx):
    """Everything of the path chained: render (camera + lidar, views on their own streams) -> L2 loss against targets
    rendered from the unperturbed scene -> backward -> optimizer_step, 25 iterations on the resident scene. Appearance
    and opacity were perturbed; the loss must fall by an order of magnitude, geometry (learning rate ~0) must stay put and the appearance of the
    blended Gaussians must have moved."""
    rng = np.random.default_rng(4)
    truth = synth.make_scene(20_000, seed=19, r_max=40.0, scale_mean=0.12)
    lid = synth.lidar32()
    rays = synth.grid_rays(lid)
    cam = synth.make_camera(width=320, height=192)
    ctx.upload_scene(truth)
    vc, vl = ctx.camera_view(cam, ST), ctx.lidar_view(lid, rays, ST)
    targets = {}
    for name, v in (("c", vc), ("l", vl)):
        v.forward(0.0)
        targets[name] = v.array("blend").reshape(v.P, 16).copy()
    import copy
    start = copy.deepcopy(truth)
    start.color = truth.color + rng.normal(0, 0.3, truth.color.shape)
    start.feature = truth.feature + rng.normal(0, 0.3, truth.feature.shape)
    start.opacity_logit = truth.opacity_logit + rng.normal(0, 0.5, truth.opacity_logit.shape)
    ctx.upload_scene(start)
    ctx.set_view_streams(True)
    cfg = {"lr_init": [1e-12, 1e-12, 1e-12, 5e-2, 2e-2, 2e-2], "lr_final": [1e-12, 1e-12, 1e-12, 2e-2, 1e-2, 1e-2],
           "warmup_steps": [0] * 6, "total_steps": 25}
    losses = []
    try:
        for step in range(25):
            ctx.zero_grads()
            loss = 0.0
            for name, v in (("c", vc), ("l", vl)):
                v.forward(0.0)
                b = v.array("blend").reshape(v.P, 16)
                ch = 16 if name == "c" else 13             # lidar: features only (range slots carry no target here)
                d = np.zeros_like(b)
                d[:, :ch] = b[:, :ch] - targets[name][:, :ch]
                loss += 0.5 * float((d.astype(np.float64) ** 2).sum())
                v.backward(d, np.zeros(v.P, np.float32))
            losses.append(loss)
            assert ctx.optimizer_step(cfg, step) == []
    finally:
        ctx.set_view_streams(False)
    assert np.isfinite(losses).all() and losses[-1] < 0.1 * losses[0], (losses[0], losses[-1])
    mean, scale_log, quat, opl, color, feature = ctx.download_scene()
    assert np.array_equal(mean, np.asarray(start.mean, np.float32)) or np.abs(mean - start.mean).max() < 1e-6   # lr ~ 0: geometry stays
    vis = np.abs(feature - start.feature).max(1) > 1e-4                                                       # Gaussians the sensors blended
    assert vis.sum() > 200
    assert np.isfinite(feature).all() and np.isfinite(opl).all() and np.isfinite(color).all()


def test_optimizer_step_range_and_sharded_path(api, op):
    """optimizer_step_range on two consecutive shards == optimizer_step on the whole buffer (same context state otherwise),
    including an unaligned boundary; sharded_optimizer_step at world size 1 (no collective) == optimizer_step; a
    skip flag from 'another rank' leaves the group untouched."""
    import torch
    from paper_2411_16816_b200 import dist as sdist
    cfg = {"lr_init": [1.6e-4, 5e-3, 1e-3, 5e-2, 2.5e-3, 2.5e-3], "lr_final": [1.6e-6, 5e-3, 1e-3, 5e-2, 2.5e-3, 2.5e-4],
           "warmup_steps": [0] * 6, "total_steps": 10}
    sc = synth.make_scene(30_011, seed=21)
    g_all = (np.random.default_rng(3).normal(size=27 * sc.n) * 1e-2).astype(np.float32)
    results = []
    for mode in ("full", "two_shards", "sharded_world1", "skip_quat"):
        c = api.Context(0)
        try:
            c.upload_scene(sc)
            grads_t = torch.from_numpy(g_all.copy()).cuda()
            c.bind_grads_device(grads_t.data_ptr(), c.grads_size)
            for step in range(3):
                if mode == "full":
                    c.optimizer_step(cfg, step)
                elif mode == "two_shards":
                    cut = 13 * sc.n + 1                      # inside the color slice, not a multiple of 4
                    c.optimizer_step_range(cfg, step, 0, cut)
                    c.optimizer_step_range(cfg, step, cut, c.grads_size)
                elif mode == "sharded_world1":
                    sdist.sharded_optimizer_step(c, grads_t, None, cfg, step)
                else:
                    c.optimizer_step_range(cfg, step, 0, c.grads_size, skip_groups=[0, 0, 1, 0, 0, 0])
            results.append([a.copy() for a in c.download_scene()])
        finally:
            c.close()
    full, two, sh1, skipq = results
    for a, b, d in zip(full, two, sh1):
        assert np.array_equal(a, b) and np.array_equal(a, d)
    assert np.array_equal(skipq[2], np.asarray(sc.quat, np.float32)) and np.array_equal(skipq[0], full[0])


def test_library_nccl_collective_world1(api, op):
    """The C-ABI collective (splatb200_ctx_comm_init -> ncclCommInitRank, splatb200_allreduce_grads ->
    ncclAllReduce on the ctx stream after a join of the view streams, splatb200_sharded_optimizer_step) on the one GPU a
    test box has: a communicator of world size 1. The sum over one rank is the identity, so gradients (incl. the ActorGrad
    slots) must come back bit-identical, and the sharded step must equal the plain one. (Two ranks need two GPUs: NCCL
    refuses two ranks on one device; the two-rank host logic runs on gloo in tests/test_dist_gloo.py, and bench.py
    --gpus N drives this very call on N GPUs.)"""
    cfg = {"lr_init": [1.6e-4, 5e-3, 1e-3, 5e-2, 2.5e-3, 2.5e-3], "lr_final": [1.6e-6, 5e-3, 1e-3, 5e-2, 2.5e-3, 2.5e-4],
           "warmup_steps": [0] * 6, "total_steps": 10}
    sc = synth.make_scene(20_003, seed=31, n_actors=3, dynamic_fraction=0.2, r_max=30.0, scale_mean=0.1)
    for k, tr in enumerate(sc.tracks):
        tr.t[:] = np.array([8.0 + 3 * k, -3.0 + 2 * k, 1.0]) + np.outer(tr.stamps, [6.0, 1.0, 0.0])
    cam = synth.make_camera(width=320, height=192)
    import torch
    uid = api.nccl_unique_id()
    assert len(uid) == 128 and any(uid)
    c, c2 = api.Context(0), api.Context(0)
    try:
        for x in (c, c2):
            x.upload_scene(sc)
        assert c.comm_world == 0
        with pytest.raises(api.SplatError, match="without a communicator"):
            c.allreduce_grads()
        c.comm_init(uid, 0, 1)
        assert c.comm_world == 1
        grads_t = torch.zeros(c.grads_size, dtype=torch.float32, device="cuda")
        c.bind_grads_device(grads_t.data_ptr(), c.grads_size)
        c.set_view_streams(True)
        v = c.render_camera(cam, ST, t_scene=0.03)
        gb, ga = synth.upstream(v.P, seed=3)
        c.zero_grads()
        v.backward(gb, ga)
        g0 = c.grads()
        assert np.abs(g0["d_mean"]).max() > 0 and any(np.abs(a["d_pose_offset"]).max() > 0 for a in g0["actors"])
        c.allreduce_grads()          # ordered after the view's stream inside the library; the sum over one rank is the identity
        g1 = c.grads()
        for k in ("d_mean", "d_scale_log", "d_quat", "d_opacity_logit", "d_color", "d_feature"):
            assert np.array_equal(g0[k], g1[k]), k
        for a in range(3):
            for k in ("d_pose_offset", "d_vel_offset"):
                assert np.array_equal(g0["actors"][a][k], g1["actors"][a][k]), (a, k)
        # the sharded step on the communicator == the plain step on a second context fed the same gradient bits
        g2_t = grads_t.clone()
        c2.bind_grads_device(g2_t.data_ptr(), c2.grads_size)
        for step in range(2):
            assert c.sharded_optimizer_step(cfg, step) == []
            assert c2.optimizer_step(cfg, step) == []
        for a, b in zip(c.download_scene(), c2.download_scene()):
            assert np.array_equal(a, b)
        assert not np.array_equal(c.download_scene()[0], np.asarray(sc.mean, np.float32))
        c.comm_destroy()
        assert c.comm_world == 0
    finally:
        c.close()
        c2.close()


def _nccl_world2_worker(rank, uid, out_dir):
    """One rank of test_library_nccl_collective_world2 (its own process and its own GPU)."""
    import os
    import torch
    from paper_2411_16816_b200 import api as _api
    cfg = {"lr_init": [1.6e-4, 5e-3, 1e-3, 5e-2, 2.5e-3, 2.5e-3], "lr_final": [1.6e-6, 5e-3, 1e-3, 5e-2, 2.5e-3, 2.5e-4],
           "warmup_steps": [0] * 6, "total_steps": 10}
    torch.cuda.set_device(rank)
    sc = synth.make_scene(5_003, seed=31, r_max=30.0, scale_mean=0.1)   # 27 * 5003 floats: not a multiple of 2 * 4
    c = _api.Context(rank)
    try:
        c.upload_scene(sc)
        c.comm_init(uid, rank, 2)
        assert c.comm_world == 2
        g = np.random.default_rng(100 + rank).normal(size=c.grads_size).astype(np.float32)
        grads_t = torch.from_numpy(g.copy()).cuda()
        c.bind_grads_device(grads_t.data_ptr(), c.grads_size)
        c.allreduce_grads()
        c.sync()
        np.save(os.path.join(out_dir, f"sum_{rank}.npy"), grads_t.cpu().numpy())
        # second step's local gradients, reduced inside the sharded step (reduce-scatter -> Adam on the shard -> all-gather)
        grads_t.copy_(torch.from_numpy(g))
        skipped = c.sharded_optimizer_step(cfg, 0)
        assert skipped == []
        for k, a in enumerate(c.download_scene()):
            np.save(os.path.join(out_dir, f"param{k}_{rank}.npy"), a)
        c.comm_destroy()
    finally:
        c.close()


def test_library_nccl_collective_world2(api, tmp_path):
    """Two ranks on two GPUs through the library's own communicator (skipped on a one-GPU box: NCCL refuses two ranks
    on one device): the all-reduced gradient buffer is the same on both ranks and equals the fp32 sum of the two local
    buffers, and the sharded optimizer step (total not divisible by world * 4) leaves both ranks with the parameters
    an all-reduce followed by the plain step gives a single context."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import torch.multiprocessing as mp
    uid = api.nccl_unique_id()
    mp.spawn(_nccl_world2_worker, args=(uid, str(tmp_path)), nprocs=2, join=True)
    s0, s1 = np.load(tmp_path / "sum_0.npy"), np.load(tmp_path / "sum_1.npy")
    g0 = np.random.default_rng(100).normal(size=s0.size).astype(np.float32)
    g1 = np.random.default_rng(101).normal(size=s0.size).astype(np.float32)
    assert np.array_equal(s0, s1) and np.array_equal(s0, g0 + g1)     # two-operand fp32 sum: order-free, bit-exact
    cfg = {"lr_init": [1.6e-4, 5e-3, 1e-3, 5e-2, 2.5e-3, 2.5e-3], "lr_final": [1.6e-6, 5e-3, 1e-3, 5e-2, 2.5e-3, 2.5e-4],
           "warmup_steps": [0] * 6, "total_steps": 10}
    sc = synth.make_scene(5_003, seed=31, r_max=30.0, scale_mean=0.1)
    c = api.Context(0)
    try:
        c.upload_scene(sc)
        t = torch.from_numpy(g0 + g1).cuda()
        c.bind_grads_device(t.data_ptr(), c.grads_size)
        assert c.optimizer_step(cfg, 0) == []
        want = c.download_scene()
    finally:
        c.close()
    for k, a in enumerate(want):
        for r in range(2):
            assert np.array_equal(a, np.load(tmp_path / f"param{k}_{r}.npy")), (k, r)


# ---- camera ConvDecoder: tcgen05 / tf32 implicit-GEMM convolutions -----------------------
# tf32 operands (10-bit mantissa, rounded to nearest) with fp32 accumulation: 2^-11 relative per operand; over five
# layers the image agrees with the fp32 oracle to DEC_RTOL of the output scale.
DEC_RTOL = 3e-3


def _conv3x3_numpy(x, w, relu_in, res):
    H, W, _ = x.shape
    k = w[:9216].reshape(32, 3, 3, 32).astype(np.float64)
    xin = np.maximum(x, 0) if relu_in else x
    xp = np.pad(xin.astype(np.float64), ((1, 1), (1, 1), (0, 0)), mode="reflect")
    y = np.zeros((H, W, 32)) + w[9216:].astype(np.float64)
    for ky in range(3):
        for kx in range(3):
            y += xp[ky:ky + H, kx:kx + W, :] @ k[:, ky, kx, :].T
    return y + (0 if res is None else res)


@pytest.mark.gpu
@pytest.mark.parametrize("H,W", [(2, 2), (5, 131), (8, 128), (33, 300), (64, 640)])
def test_conv3x3_tensor_core_matches_numpy(ctx, H, W):
    """One decoder convolution (partial tiles in both directions, reflect padding, ReLU on the input, residual) against
    a float64 numpy evaluation, and bit-exactly on small integers (exact in tf32)."""
    rng = np.random.default_rng(H * 1000 + W)
    x = rng.normal(0, 1, (H, W, 32)).astype(np.float32)
    w = rng.normal(0, 0.1, 9248).astype(np.float32)
    res = rng.normal(0, 1, (H, W, 32)).astype(np.float32)
    for relu_in, r in ((False, None), (True, res)):
        y = ctx.debug_conv3x3(x, w, relu_in, r)
        ref = _conv3x3_numpy(x, w, relu_in, r)
        assert np.abs(y - ref).max() <= 2e-3 * np.abs(ref).max(), (relu_in, np.abs(y - ref).max(), np.abs(ref).max())
    # integers up to 2^10 are exact in tf32: bit-exact convolution
    xi = rng.integers(-8, 9, (H, W, 32)).astype(np.float32)
    wi = rng.integers(-4, 5, 9248).astype(np.float32)
    assert np.array_equal(ctx.debug_conv3x3(xi, wi), _conv3x3_numpy(xi, wi, False, None).astype(np.float32))


def _decoder_inputs(view, cam, d_f):
    blend = view.array("blend").reshape(cam.height, cam.width, 16)
    return blend[..., :3], blend[..., 3:3 + d_f], np.array([cam.fx, cam.fy, cam.cx, cam.cy], np.float32)


@pytest.mark.gpu
@pytest.mark.parametrize("w,h", [(320, 192), (203, 77)])
def test_decode_image_matches_oracle(ctx, op, w, h):
    sc = synth.make_scene(6000, seed=21, r_max=40.0, scale_mean=0.12)
    cam = synth.make_camera(width=w, height=h)
    ctx.upload_scene(sc)
    view = ctx.camera_view(cam, ST)
    view.forward(0.0)
    rgb, feat, intr = _decoder_inputs(view, cam, sc.d_f)
    rng = np.random.default_rng(5)
    params = rng.normal(0, 0.08, op.DEC_PARAMS).astype(np.float32)
    params[op.DEC_HEAD_OFFSET:] = rng.normal(0, 0.3, op.DEC_PARAMS - op.DEC_HEAD_OFFSET)
    emb = rng.normal(0, 1, 8).astype(np.float32)
    img = view.decode_image(params, emb).reshape(h, w, 3)
    ref = op.decoder_forward(params, rgb, feat, intr, emb, np.float32, workers=8)
    assert np.abs(img - ref).max() <= DEC_RTOL * max(1.0, np.abs(ref).max()), np.abs(img - ref).max()
    assert np.array_equal(view.array("decoded").reshape(h, w, 3), img)
    # zero-initialised head -> the decoder is the identity, exactly
    p0 = params.copy(); p0[op.DEC_HEAD_OFFSET:] = 0
    assert np.array_equal(view.decode_image(p0, emb).reshape(h, w, 3), rgb)
    # forced M = 2, b = 0.1
    p0[-6:] = [1, 1, 1, 0.1, 0.1, 0.1]
    assert np.allclose(view.decode_image(p0, emb).reshape(h, w, 3), 2 * rgb + np.float32(0.1), rtol=0, atol=1e-6)
    # a lidar view has no image to decode
    lv = ctx.lidar_view(synth.lidar32(), synth.grid_rays(synth.lidar32()), ST)
    lv.forward(0.0)
    with pytest.raises(Exception):
        lv.decode_image(params, emb)


@pytest.mark.gpu
@pytest.mark.parametrize("w,h,d_f", [(320, 192, 13), (203, 77, 13), (70, 50, 5)])
def test_decode_image_precise_mode_meets_fp32_bar(ctx, op, w, h, d_f):
    """splatb200_ctx_set_decoder_precise: the convolutions in split-tf32 (three tensor-core passes, hi*hi + lo*hi +
    hi*lo, fp32 accumulation). The image meets the north-star 1e-4 against the fp32 oracle, a single
    convolution agrees with float64 numpy to 2e-6, and the gradients of decode_image meet 1e-3 against the fp64 oracle
    backward evaluated from the ORACLE's own forward (not from the device's saved activations, which the tf32 mode
    needs because its ReLU masks differ)."""
    import torch
    rng = np.random.default_rng(11)
    ctx.set_decoder_precise(True)
    try:
        x = rng.normal(0, 1, (33, 150, 32)).astype(np.float32)
        wts = rng.normal(0, 0.1, 9248).astype(np.float32)
        res = rng.normal(0, 1, x.shape).astype(np.float32)
        for relu_in, r in ((False, None), (True, res)):
            y = ctx.debug_conv3x3(x, wts, relu_in, r)
            ref = _conv3x3_numpy(x, wts, relu_in, r)
            assert np.abs(y - ref).max() <= 2e-6 * np.abs(ref).max(), (relu_in, np.abs(y - ref).max() / np.abs(ref).max())
        gy = rng.normal(0, 1, x.shape).astype(np.float32)
        gx, gw = ctx.debug_conv3x3_backward(x, wts, gy, True)
        rgx, rgw = _conv3x3_backward_numpy(x, wts, True, gy)
        assert np.abs(gx - rgx).max() <= 1e-5 * np.abs(rgx).max() and np.abs(gw - rgw).max() <= 1e-5 * np.abs(rgw).max()

        sc = synth.make_scene(6000, seed=21, r_max=40.0, scale_mean=0.12, d_f=d_f)
        cam = synth.make_camera(width=w, height=h)
        ctx.upload_scene(sc)
        view = ctx.camera_view(cam, ST)
        view.forward(0.0)
        rgb, feat, intr = _decoder_inputs(view, cam, d_f)
        params = rng.normal(0, 0.08, op.DEC_PARAMS).astype(np.float32)
        params[op.DEC_HEAD_OFFSET:] = rng.normal(0, 0.3, op.DEC_PARAMS - op.DEC_HEAD_OFFSET)
        emb = rng.normal(0, 1, 8).astype(np.float32)
        img = view.decode_image(params, emb).reshape(h, w, 3)
        ref = op.decoder_forward(params, rgb, feat, intr, emb, np.float32, workers=8)
        assert np.abs(img - ref).max() <= 1e-4 * max(1.0, np.abs(ref).max()), np.abs(img - ref).max()
        p0 = params.copy(); p0[op.DEC_HEAD_OFFSET:] = 0                   # zero head = identity, exactly
        assert np.array_equal(view.decode_image(p0, emb).reshape(h, w, 3), rgb)
        # gradients against the fp64 oracle's own forward + backward. A ReLU whose fp32 pre-activation lies within
        # rounding of zero can still flip; with white-noise dL/dI such a flip is a full-size term, so the comparison
        # is made on a smooth upstream gradient (dL/dI = the image itself, an L2 loss against zero)
        view.decode_image(params, emb)
        g_image = ref.astype(np.float32)
        g_up = torch.zeros((view.P, 16), dtype=torch.float32, device="cuda")
        gp, ge = view.decode_image_backward(g_image, g_up.data_ptr())
        ogp, ogrgb, ogf, oge = op.decoder_backward(params, rgb, feat, intr, emb, g_image, np.float64)
        bounds = [l * op.DEC_CONV_PARAMS for l in range(6)] + [op.DEC_PARAMS]
        for l, (b, e) in enumerate(zip(bounds[:-1], bounds[1:])):
            err, scale = np.abs(gp[b:e] - ogp[b:e]).max(), np.abs(ogp[b:e]).max()
            assert err <= GRAD_RTOL * scale, (l, err, scale)
        assert np.abs(ge - oge).max() <= GRAD_RTOL * np.abs(oge).max()
        gb = g_up.cpu().numpy().reshape(h, w, 16)
        assert np.abs(gb[..., :3] - ogrgb).max() <= GRAD_RTOL * np.abs(ogrgb).max()
        # per-pixel feature gradients: of the ~8M rectified activations a handful lie within fp32 rounding of zero and
        # flip between the fp32 device forward and the fp64 oracle forward; each flip changes a 5 x 5 pixel
        # neighbourhood by O(1 %). Hence: relative L2 error, and all but 1e-3 of the entries within 1e-3
        d = np.abs(gb[..., 3:3 + d_f] - ogf)
        assert np.linalg.norm(d) <= GRAD_RTOL * np.linalg.norm(ogf), np.linalg.norm(d) / np.linalg.norm(ogf)
        assert (d > GRAD_RTOL * np.abs(ogf).max()).mean() <= 1e-3, (d > GRAD_RTOL * np.abs(ogf).max()).mean()
    finally:
        ctx.set_decoder_precise(False)


@pytest.mark.gpu
def test_decode_image_full_size_1080p(ctx, op):
    """The north-star camera (1920 x 1080): parity with the threaded fp32 oracle, run-to-run determinism, device time."""
    sc = synth.make_scene(200_000, seed=22)
    cam = synth.make_camera()
    ctx.upload_scene(sc)
    view = ctx.camera_view(cam, ST)
    view.forward(0.0)
    rgb, feat, intr = _decoder_inputs(view, cam, sc.d_f)
    rng = np.random.default_rng(6)
    params = rng.normal(0, 0.08, op.DEC_PARAMS).astype(np.float32)
    params[op.DEC_HEAD_OFFSET:] = rng.normal(0, 0.3, op.DEC_PARAMS - op.DEC_HEAD_OFFSET)
    emb = rng.normal(0, 1, 8).astype(np.float32)
    img, _ = view.decode_image(params, emb, timed=True)
    times = [view.decode_image(params, emb, download=False, timed=True)[1] for _ in range(5)]
    assert np.array_equal(view.array("decoded").reshape(-1, 3), img)
    ref = op.decoder_forward(params, rgb, feat, intr, emb, np.float32, workers=16)
    err = np.abs(img.reshape(ref.shape) - ref).max()
    print(f"decode_image 1920x1080: {min(times):.3f} ms on the device, max |err| {err:.2e} (scale {np.abs(ref).max():.2f})")
    assert err <= DEC_RTOL * max(1.0, np.abs(ref).max())


DEC_GRAD_RTOL = 5e-3   # tf32 operands in the gradient convolutions as well; relative to each tensor's largest entry


def _reflect_idx(i, n):
    i = np.abs(i)
    return np.where(i >= n, 2 * (n - 1) - i, i)


def _conv3x3_backward_numpy(x, w, relu_in, gy):
    H, W, _ = x.shape
    k = w[:9216].reshape(32, 3, 3, 32).astype(np.float64)
    xin = (np.maximum(x, 0) if relu_in else x).astype(np.float64)
    gy = gy.astype(np.float64)
    gx, gw = np.zeros((H, W, 32)), np.zeros((32, 3, 3, 32))
    for ky in range(3):
        ys = _reflect_idx(np.arange(H) + ky - 1, H)
        for kx in range(3):
            xs = _reflect_idx(np.arange(W) + kx - 1, W)
            gw[:, ky, kx, :] = np.einsum("hwo,hwi->oi", gy, xin[ys][:, xs])
            np.add.at(gx, (ys[:, None], xs[None, :]), gy @ k[:, ky, kx, :])
    if relu_in:
        gx *= x > 0
    return gx, np.concatenate([gw.ravel(), gy.sum((0, 1))])


@pytest.mark.parametrize("H,W", [(2, 2), (3, 3), (5, 131), (33, 300)])
def test_conv3x3_backward_matches_numpy(ctx, H, W):
    """Input and weight gradients of one decoder convolution (both tensor-core kernels; the adjoint of reflect padding
    on the borders, including the 3 x 3 image where both border preimages fold onto the centre)."""
    rng = np.random.default_rng(H * 1000 + W + 1)
    x = rng.normal(0, 1, (H, W, 32)).astype(np.float32)
    w = rng.normal(0, 0.1, 9248).astype(np.float32)
    gy = rng.normal(0, 1, (H, W, 32)).astype(np.float32)
    for relu_in in (False, True):
        gx, gw = ctx.debug_conv3x3_backward(x, w, gy, relu_in)
        rgx, rgw = _conv3x3_backward_numpy(x, w, relu_in, gy)
        assert np.abs(gx - rgx).max() <= 2e-3 * np.abs(rgx).max(), (relu_in, np.abs(gx - rgx).max(), np.abs(rgx).max())
        assert np.abs(gw - rgw).max() <= 2e-3 * np.abs(rgw).max(), (relu_in, np.abs(gw - rgw).max(), np.abs(rgw).max())
    # small integers: exact in tf32 and in the fp32 accumulators
    xi = rng.integers(-4, 5, (H, W, 32)).astype(np.float32)
    wi = rng.integers(-3, 4, 9248).astype(np.float32)
    gi = rng.integers(-2, 3, (H, W, 32)).astype(np.float32)
    gx, gw = ctx.debug_conv3x3_backward(xi, wi, gi, True)
    rgx, rgw = _conv3x3_backward_numpy(xi, wi, True, gi)
    assert np.array_equal(gx, rgx.astype(np.float32)) and np.array_equal(gw, rgw.astype(np.float32))


@pytest.mark.parametrize("w,h,d_f", [(96, 64, 13), (203, 77, 13), (70, 50, 5)])
def test_decode_image_backward_matches_oracle(ctx, op, w, h, d_f):
    """dL/dparams, dL/dembedding, dL/dF_rgb and dL/dfeature of decode_image against the fp64 oracle backward (pinned by
    finite differences, tests/test_oracle_kat.py); the feature gradient is added into the render's upstream buffer."""
    import torch
    sc = synth.make_scene(4000, seed=23, r_max=40.0, scale_mean=0.12, d_f=d_f)
    cam = synth.make_camera(width=w, height=h)
    ctx.upload_scene(sc)
    view = ctx.camera_view(cam, ST)
    view.forward(0.0)
    P = view.P
    rgb, feat, intr = _decoder_inputs(view, cam, d_f)
    rng = np.random.default_rng(7)
    params = rng.normal(0, 0.08, op.DEC_PARAMS).astype(np.float32)
    params[op.DEC_HEAD_OFFSET:] = rng.normal(0, 0.3, op.DEC_PARAMS - op.DEC_HEAD_OFFSET)
    emb = rng.normal(0, 1, 8).astype(np.float32)
    g_image = rng.normal(0, 1, (h, w, 3)).astype(np.float32)
    g_up = torch.zeros((P, 16), dtype=torch.float32, device="cuda")
    with pytest.raises(Exception):                      # no saved state yet
        view.decode_image_backward(g_image, g_up.data_ptr())
    view.decode_image(params, emb)
    g_up[:, 4] = 0.5                                    # another upstream gradient of the render: must be kept
    gp, ge = view.decode_image_backward(g_image, g_up.data_ptr())
    # The device gradient is the gradient of the device forward: its ReLU masks come from the tf32 activations, and
    # against white-noise dL/dI a mask flip on a near-zero activation is a full-size term of an incoherent sum. So the
    # oracle backward runs from the device's saved activations (forward parity is test_decode_image_matches_oracle).
    acts = np.stack([view.array(f"decoder_act{k}").reshape(h, w, 32) for k in range(6)])
    ogp, ogrgb, ogf, oge = op.decoder_backward_from_state(params, rgb, acts, d_f, g_image)
    names = [f"conv{l}" for l in range(5)] + ["head"]
    bounds = [l * op.DEC_CONV_PARAMS for l in range(6)] + [op.DEC_PARAMS]
    for name, b, e in zip(names, bounds[:-1], bounds[1:]):
        err, scale = np.abs(gp[b:e] - ogp[b:e]).max(), np.abs(ogp[b:e]).max()
        assert err <= DEC_GRAD_RTOL * scale, (name, err, scale)
    assert np.abs(ge - oge).max() <= DEC_GRAD_RTOL * np.abs(oge).max()
    gb = g_up.cpu().numpy().reshape(h, w, 16)
    exp = np.concatenate([ogrgb, ogf], axis=2); exp[..., 4] += 0.5
    assert np.abs(gb[..., :3] - exp[..., :3]).max() <= DEC_GRAD_RTOL * np.abs(exp[..., :3]).max()
    assert np.abs(gb[..., 3:3 + d_f] - exp[..., 3:]).max() <= DEC_GRAD_RTOL * np.abs(exp[..., 3:]).max()
    assert not gb[..., 3 + d_f:].any()                  # slots behind the features are not touched
    # decoder + rasterizer backward in one go: the buffer is the render's upstream gradient
    ga = torch.zeros(P, dtype=torch.float32, device="cuda")
    ctx.zero_grads()
    view.backward_device(g_up.data_ptr(), ga.data_ptr())
    assert np.isfinite(ctx.grads()["d_feature"]).all() and np.abs(ctx.grads()["d_feature"]).max() > 0
    # a new forward invalidates the saved activations
    view.forward(0.0)
    with pytest.raises(Exception):
        view.decode_image_backward(g_image, g_up.data_ptr())


def test_decode_image_backward_full_size_1080p(ctx, op):
    """1920 x 1080: linearity of the backward in dL/dimage, finite results, device time."""
    import torch
    sc = synth.make_scene(200_000, seed=22)
    cam = synth.make_camera()
    ctx.upload_scene(sc)
    view = ctx.camera_view(cam, ST)
    view.forward(0.0)
    rng = np.random.default_rng(8)
    params = rng.normal(0, 0.08, op.DEC_PARAMS).astype(np.float32)
    params[op.DEC_HEAD_OFFSET:] = rng.normal(0, 0.3, op.DEC_PARAMS - op.DEC_HEAD_OFFSET)
    emb = rng.normal(0, 1, 8).astype(np.float32)
    view.decode_image(params, emb, download=False)
    g_image = rng.normal(0, 1, (view.P, 3)).astype(np.float32)
    g1 = torch.zeros((view.P, 16), dtype=torch.float32, device="cuda")
    g2 = torch.zeros_like(g1)
    gp1, ge1, ms = view.decode_image_backward(g_image, g1.data_ptr(), timed=True)
    gp2, ge2, ms2 = view.decode_image_backward(2 * g_image, g2.data_ptr(), timed=True)
    print(f"decode_image backward 1920x1080: {min(ms, ms2):.3f} ms on the device")
    assert np.isfinite(gp1).all() and np.abs(gp1).max() > 0
    # power-of-two scaling is exact in every product; only the atomics' summation order differs between the runs
    assert np.abs(gp2 - 2 * gp1).max() <= 1e-4 * np.abs(gp1).max()
    assert np.abs(ge2 - 2 * ge1).max() <= 1e-4 * np.abs(ge1).max()
    assert torch.equal(g2, 2 * g1)


def test_files_to_render_spz1_and_lpc1(ctx, tmp_path):
    """The data formats either side of the path: a scene saved as SPZ1 and a sweep saved as
    LPC1, loaded back, give bit-identical renders / ray assignments to the in-memory originals."""
    from paper_2411_16816_b200 import io as sio
    sc = synth.make_scene(5000, seed=31, r_max=40.0, scale_mean=0.1, n_actors=2).astype(np.float32)
    cam = synth.make_camera(width=320, height=192)
    lid = synth.lidar128()
    sio.save_spz1(tmp_path / "s.spz1", sc, [cam], [lid])
    got = sio.load_spz1(tmp_path / "s.spz1")
    ctx.upload_scene(sc)
    a = ctx.render_camera(cam, ST).array("blend")
    ctx.upload_scene(got["scene"])
    b = ctx.render_camera(got["cameras"][0], ST).array("blend")
    assert np.array_equal(bits(a), bits(b)) and np.abs(a).max() > 0
    rng = np.random.default_rng(9)
    pts = rng.normal(0, 25, (20000, 3)).astype(np.float32) + np.array([0, 0, 1.0], np.float32)
    ts = (rng.uniform(-0.05, 0.05, len(pts)) + lid.timestamp).astype(np.float32)
    sio.save_lpc1(tmp_path / "w.lpc1", pts, rng.uniform(0, 1, len(pts)), ts, np.ones(len(pts)), "top", -0.05, 0.05)
    sweep = sio.load_lpc1(tmp_path / "w.lpc1")
    g0 = ctx.assign_points_to_tiles(lid, pts, ts, train=False, seed=1)
    g1 = ctx.assign_points_to_tiles(got["lidars"][0], sweep["xyz"], sweep["timestamps"], train=False, seed=1)
    assert np.array_equal(g0["tile"], g1["tile"]) and np.array_equal(g0["order"], g1["order"])
    for k in ("phi", "omega", "t_l", "range"):
        assert np.array_equal(bits(g0[k]), bits(g1[k])), k
