"""GPU-box probe of the end-to-end (host-buffer) frame: which part of the 10 ms is transfer, which is waiting.
  PYTHONPATH=. python scripts/e2e_probe.py"""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2411_16816_b200 import api, synth  # noqa: E402
from paper_2411_16816_b200.model import RasterSettings, Scene  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
st = RasterSettings()
with torch.cuda.stream(stream):
    ctx = api.Context(0, stream.cuda_stream)
    scene = synth.make_scene(1_000_000, seed=3)
    keep, arrs = [], []
    for a in (scene.mean, scene.scale_log, scene.quat, scene.opacity_logit, scene.color, scene.feature):
        t, v = bench.pinned(a.shape, torch.float32); v[...] = a; keep.append(t); arrs.append(v)
    t_id, v_id = bench.pinned(scene.actor_id.shape, torch.int32); v_id[...] = scene.actor_id
    pscene = Scene(*arrs, v_id, [])
    ctx.upload_scene(pscene)
    n_grad = ctx.grads_size
    lid, cam = bench.frame_sensors(0)
    rays = synth.grid_rays(lid)
    vl, vc = ctx.lidar_view(lid, rays, st), ctx.camera_view(cam, st)
    g_host, out_host = {}, {}
    for name, P, seed in (("l", vl.P, 11), ("c", vc.P, 12)):
        gb, ga = synth.upstream(P, seed=seed)
        tb, vb = bench.pinned(gb.shape, torch.float32); vb[...] = gb
        ta, va = bench.pinned(ga.shape, torch.float32); va[...] = ga
        g_host[name] = (tb, ta, vb, va)
        ob = bench.pinned((P, 16), torch.float32); oa = bench.pinned((P,), torch.float32); on = bench.pinned((P,), torch.int32)
        out_host[name] = (ob[1], oa[1], on[1], ob[0], oa[0], on[0])
    gh_t, gh = bench.pinned((n_grad,), torch.float32)
    n = 1_000_000
    gh_parts = [gh[0:3 * n], gh[3 * n:6 * n], gh[6 * n:10 * n], gh[10 * n:11 * n], gh[11 * n:14 * n], gh[14 * n:]]
    ctx.set_view_streams(True)
    pool = ThreadPoolExecutor(max_workers=2)

    def step(upload=True, download=True, bands=0, views=("l", "c")):
        if upload:
            ctx.upload_scene(pscene)
        ctx.zero_grads()

        def run_view(name, v):
            vb, va, vn = out_host[name][:3]
            v.forward_to_host(0.0, vb, va, vn, bands=bands)
            v.backward_from_host(g_host[name][2], g_host[name][3])
        fs = [pool.submit(run_view, name, v) for name, v in (("l", vl), ("c", vc)) if name in views]
        for f in fs:
            f.result()
        ctx.join()
        if download:
            ctx.grads_into(*gh_parts)
        ctx.sync()

    def timeit(label, **kw):
        for _ in range(2):
            step(**kw)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            step(**kw)
        torch.cuda.synchronize()
        print(f"{label:50s} {(time.perf_counter() - t0) * 100:.3f} ms", flush=True)

    g_dev = {}
    for name in ("l", "c"):
        g_dev[name] = (torch.from_numpy(np.ascontiguousarray(g_host[name][2])).to(dev), torch.from_numpy(np.ascontiguousarray(g_host[name][3])).to(dev))

    def step_dev(upload=False, download=False):
        """the device-resident frame bench.py times as `value`"""
        ctx.zero_grads()

        def run_view(name, v):
            v.forward(0.0)
            v.backward_device(g_dev[name][0].data_ptr(), g_dev[name][1].data_ptr())
        for f in [pool.submit(run_view, name, v) for name, v in (("l", vl), ("c", vc))]:
            f.result()
        ctx.join()
        ctx.sync()

    if os.environ.get("E2E_TRACE") == "dev":
        step = step_dev
    if os.environ.get("E2E_TRACE"):
        # timeline of one end-to-end step (CUPTI through torch.profiler): every kernel and copy with its stream, start
        # and duration, relative to the step's first activity -> gpurun_out/e2e_trace.txt
        from torch.profiler import ProfilerActivity, profile
        kw = dict(upload=os.environ["E2E_TRACE"] != "mid", download=os.environ["E2E_TRACE"] != "mid")
        for _ in range(3):
            step(**kw)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
            for _ in range(3):          # the first profiled steps pay CUPTI's lazy set-up: keep the last one
                step(**kw)
                torch.cuda.synchronize()
        prof.export_chrome_trace("gpurun_out/e2e_trace.json")
        import json
        ev = [e for e in json.load(open("gpurun_out/e2e_trace.json"))["traceEvents"]
              if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset", "cuda_runtime", "cuda_driver")]
        ev.sort(key=lambda e: e["ts"])
        big = [e for e in ev if e["cat"] == "gpu_memset" and e.get("args", {}).get("bytes", 0) > 50_000_000]
        last0 = big[-1]["ts"] - 400.0       # zero_grads of the last step (its host call starts a little earlier)
        ev = [e for e in ev if e["ts"] >= last0]
        t0 = ev[0]["ts"]
        with open("gpurun_out/e2e_trace.txt", "w") as f:
            for e in ev:
                a = e.get("args", {})
                f.write("%9.1f %8.1f %s s%-3s %s %s\n" % (e["ts"] - t0, e["dur"], "host t%s" % e.get("tid") if e["cat"].startswith("cuda_") else "gpu", a.get("stream", "?"), e["name"][:60].replace("\n", " "),
                                                     a.get("bytes", "")))
        os.remove("gpurun_out/e2e_trace.json")
        print("trace written:", len(ev), "activities, span %.3f ms" % ((ev[-1]["ts"] + ev[-1]["dur"] - t0) / 1e3))
        sys.exit(0)
    timeit("full e2e, 4 bands")
    timeit("full e2e, 8 bands", bands=8)
    timeit("full e2e, 2 bands", bands=2)
    timeit("no scene upload", upload=False)
    timeit("no grads download", download=False)
    timeit("neither", upload=False, download=False)
    timeit("neither, camera only", upload=False, download=False, views=("c",))
    timeit("neither, lidar only", upload=False, download=False, views=("l",))
    t0 = time.perf_counter()
    for _ in range(10):
        ctx.upload_scene(pscene)
    torch.cuda.synchronize()
    print(f"scene upload alone {(time.perf_counter() - t0) * 100:.3f} ms")
    t0 = time.perf_counter()
    for _ in range(10):
        ctx.grads_into(*gh_parts)
    torch.cuda.synchronize()
    print(f"grads download alone {(time.perf_counter() - t0) * 100:.3f} ms")
