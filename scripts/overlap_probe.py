"""GPU box: where does the frame's time go when the two sensors share the GPU? Wall-clock over 30 iterations between
two ctx.sync() calls, device-resident inputs, north-star frame.   PYTHONPATH=. python scripts/overlap_probe.py"""
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2411_16816_b200 import api, synth  # noqa: E402
from paper_2411_16816_b200.model import RasterSettings  # noqa: E402

st = RasterSettings()
ctx = api.Context(0)
ctx.upload_scene(synth.make_scene(1_000_000, seed=3))
lid = synth.lidar128()
vl = ctx.lidar_view(lid, synth.grid_rays(lid), st)
vc = ctx.camera_view(synth.make_camera(), st)
g = {}
for name, v, seed in (("l", vl, 11), ("c", vc, 12)):
    gb, ga = synth.upstream(v.P, seed=seed)
    if name == "l":
        gb[:, 14:] = 0
    g[name] = (torch.from_numpy(gb).cuda(), torch.from_numpy(ga).cuda())
torch.cuda.synchronize()
pool = ThreadPoolExecutor(max_workers=2)


def run(v, k):
    v.forward(0.0)
    v.backward_device(g[k][0].data_ptr(), g[k][1].data_ptr())


def timed(fn, n=30):
    for _ in range(3):
        fn()
    ctx.sync()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    ctx.sync()
    return (time.perf_counter() - t0) / n * 1e3


def both_threads():
    ctx.zero_grads()
    for fu in [pool.submit(run, vl, "l"), pool.submit(run, vc, "c")]:
        fu.result()
    ctx.join()


def both_seq():
    ctx.zero_grads()
    run(vl, "l")
    run(vc, "c")
    ctx.join()


def both_seq_nozero():
    run(vl, "l")
    run(vc, "c")


def fwd_then_bwd():
    """all forwards first, then all backwards (one host thread)"""
    ctx.zero_grads()
    vl.forward(0.0)
    vc.forward(0.0)
    vl.backward_device(g["l"][0].data_ptr(), g["l"][1].data_ptr())
    vc.backward_device(g["c"][0].data_ptr(), g["c"][1].data_ptr())
    ctx.join()


for streams in (True, False):
    ctx.set_view_streams(streams)
    print(f"view streams {streams}:", flush=True)
    print(f"  lidar alone            {timed(lambda: run(vl, 'l')):.3f} ms")
    print(f"  camera alone           {timed(lambda: run(vc, 'c')):.3f} ms")
    print(f"  both, one host thread  {timed(both_seq):.3f} ms")
    print(f"  same, no zero/join     {timed(both_seq_nozero):.3f} ms")
    print(f"  forwards then backwards {timed(fwd_then_bwd):.3f} ms")
    print(f"  both, a thread per view {timed(both_threads):.3f} ms", flush=True)
