"""GPU-box diagnostic: per-Gaussian gradient error of the sm_100a path against the fp64 oracle, next to projected-input
features, so that an INPUT-derived conditioning criterion can be chosen for the gradient parity gate
(tests/test_gpu_parity.py). Writes gpurun_out/grad_probe_<name>.npz (offender rows + a random sample).

  PYTHONPATH=. python scripts/grad_cond_probe.py cam100k lidar1m cam30k lidar20k
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle_py as op  # noqa: E402
from paper_2411_16816_b200 import api, synth  # noqa: E402
from paper_2411_16816_b200.model import RasterSettings  # noqa: E402

ST = RasterSettings()
KEYS = ("d_mean", "d_scale_log", "d_quat", "d_opacity_logit", "d_color", "d_feature")


def case(name):
    if name.endswith("_np1"):
        sc, sen = case(name[:-4])
        return sc, sen + (1.0,)
    if name == "cam100k":
        return synth.make_scene(100_000, seed=3), ("camera", synth.make_camera())
    if name == "cam1m":
        return synth.make_scene(1_000_000, seed=3), ("camera", synth.make_camera())
    if name == "lidar1m":
        return synth.make_scene(1_000_000, seed=3), ("lidar", synth.lidar128())
    if name == "cam30k":
        return synth.make_scene(30000, seed=5, r_max=40.0, scale_mean=0.08), ("camera", synth.make_camera(width=640, height=360, time_offset=0.002))
    if name == "lidar20k":
        return synth.make_scene(20000, seed=3, r_max=50.0, scale_mean=0.08), ("lidar", synth.lidar128())
    raise SystemExit(name)


def main():
    ctx = api.Context(0)
    W = op.hardware_threads()
    for name in sys.argv[1:]:
        sc, sen = case(name)
        kind, sensor = sen[0], sen[1]
        ST = RasterSettings()
        if len(sen) > 2:
            ST.near_plane = sen[2]
        ctx.upload_scene(sc)
        if kind == "camera":
            gv = ctx.render_camera(sensor, ST)
            render = lambda o: o.render_camera(sensor, ST, workers=W)
        else:
            rays = synth.grid_rays(sensor)
            gv = ctx.render_lidar(sensor, rays, ST)
            render = lambda o: o.render_lidar(sensor, rays, ST, workers=W)
        gb, ga = synth.upstream(gv.P, seed=1)
        if kind == "lidar":
            gb[:, 14:] = 0
        ctx.zero_grads()
        gv.backward(gb, ga)
        g = ctx.grads()
        res = {}
        t0 = time.time()
        og, hashes, views, scenes = {}, {}, {}, {}
        for dt in (np.float32, np.float64):
            o = op.OracleScene(sc, dt)
            v = render(o)
            v.backward(gb, ga, workers=W)
            og[dt] = o.grads()
            hashes[dt] = v.contrib(want_hash=True, workers=W)[0]
            views[dt], scenes[dt] = v, o
            if dt == np.float64:
                src = v.array("source_index")
                feats = {f: v.array(f) for f in ("mean2d", "depth_key", "cov2d", "conic", "det_ratio", "rect", "velocity", "aabb")}
        flips = (hashes[np.float32] != hashes[np.float64]).astype(np.uint8)
        fmask = np.zeros(sc.n, bool)
        for dt in views:
            fmask |= views[dt].contrib(query_flag=flips, workers=W)[2].astype(bool)
        del views, scenes
        print(name, "oracle s", time.time() - t0, flush=True)
        n = sc.n
        err_gpu, err_ref, err_g32 = np.zeros((n, 6)), np.zeros((n, 6)), np.zeros((n, 6))
        print(f"  flipped queries {int(flips.sum())} of {len(flips)}; rows touched {int(fmask.sum())}", flush=True)
        rsc = np.zeros((n, 6))
        for j, k in enumerate(KEYS):
            a = np.asarray(g[k], np.float64).reshape(n, -1)
            b = np.asarray(og[np.float64][k], np.float64).reshape(n, -1)
            r = np.asarray(og[np.float32][k], np.float64).reshape(n, -1)
            scale = np.abs(b).max()
            if scale == 0:
                continue
            rowscale = np.maximum(np.abs(b).max(1), 1e-3 * scale)
            err_gpu[:, j] = np.abs(a - b).max(1) / rowscale
            err_ref[:, j] = np.abs(r - b).max(1) / rowscale
            rsc[:, j] = np.abs(b).max(1) / scale
            rs32 = np.maximum(np.abs(r).max(1), 1e-3 * np.abs(r).max())
            err_g32[:, j] = np.abs(a - r).max(1) / rs32
            um = ~fmask
            print(f"  {k}: vs fp32 oracle rows>1e-3 {(err_g32[:, j] > 1e-3).sum()} worst {err_g32[:, j].max():.2e} | outside flips: rows>1e-3 "
                  f"{(err_gpu[um, j] > 1e-3).sum()} worst {err_gpu[um, j].max():.2e} relL2 {np.linalg.norm((a - b)[um]) / np.linalg.norm(b[um]):.2e} "
                  f"maxabs/max {np.abs(a - b)[um].max() / scale:.2e} | all rows relL2 {np.linalg.norm(a - b) / np.linalg.norm(b):.2e}", flush=True)
            print(f"  {k}: rows>1e-3 gpu {(err_gpu[:, j] > 1e-3).sum()} ref32 {(err_ref[:, j] > 1e-3).sum()} live {(np.abs(b).max(1) > 0).sum()}"
                  f" worst gpu {err_gpu[:, j].max():.2e}", flush=True)
        # per-Gaussian features in source order
        F = {}
        for f, a in feats.items():
            w = a.size // len(src)
            full = np.zeros((n, w))
            full[src] = a.reshape(len(src), w)
            F[f] = full
        vis = np.zeros(n, bool)
        vis[src] = True
        bad = (err_gpu > 1e-3).any(1) | (err_g32 > 1e-4).any(1)
        rng = np.random.default_rng(0)
        sample = np.zeros(n, bool)
        sample[rng.choice(n, min(n, 60000), replace=False)] = True
        keep = np.flatnonzero(bad | (sample & vis))
        np.savez_compressed(f"gpurun_out/grad_probe_{name}.npz", idx=keep, err_gpu=err_gpu[keep].astype(np.float32),
                            err_ref=err_ref[keep].astype(np.float32), err_g32=err_g32[keep].astype(np.float32), fmask=fmask[keep], rowscale=rsc[keep].astype(np.float32),
                            n=n, n_vis=len(src), n_bad=int(bad.sum()), **{f: F[f][keep] for f in F})
        print(name, "visible", len(src), "bad rows", int(bad.sum()), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
