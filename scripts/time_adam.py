"""optimizer_step at the north-star size: ms per step and HBM fraction (28 B per parameter: g, m, v, p in; m, v, p out,
plus one more read of g by the finiteness check)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_16816_b200 import api, synth
cfg = {"lr_init": [1.6e-4, 5e-3, 1e-3, 5e-2, 2.5e-3, 2.5e-3], "lr_final": [1.6e-6, 5e-3, 1e-3, 5e-2, 2.5e-3, 2.5e-4],
       "warmup_steps": [0] * 6, "total_steps": 30000}
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    ctx = api.Context(0, stream.cuda_stream)
    sc = synth.make_scene(1_000_000, seed=3)
    ctx.upload_scene(sc)
    g = torch.randn(ctx.grads_size, dtype=torch.float32, device="cuda") * 1e-3
    ctx.bind_grads_device(g.data_ptr(), ctx.grads_size)
    for s in range(3):
        ctx.optimizer_step(cfg, s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 20
    e0.record(stream)
    for s in range(K):
        ctx.L.splatb200_optimizer_step(ctx.h, None, 0, None) if False else ctx.optimizer_step(cfg, 3 + s)
    e1.record(stream)
    stream.synchronize()
    ms = e0.elapsed_time(e1) / K
    bytes_ = 32 * ctx.grads_size
    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
    print(json.dumps({"optimizer_step_ms": ms, "bytes": bytes_, "GBps": bytes_ / ms / 1e6, "frac_of_hbm_peak": bytes_ / ms / 1e6 / peak}))
