"""Times decode_image forward + backward (ConvDecoder) on the north-star camera (1920 x 1080).
Usage (GPU box): PYTHONPATH=. python scripts/time_decoder.py [reps]"""
import sys

import numpy as np
import torch

from paper_2411_16816_b200 import api, synth
from paper_2411_16816_b200.model import RasterSettings

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
ctx = api.Context(0)
sc = synth.make_scene(200_000, seed=22)
cam = synth.make_camera()
ctx.upload_scene(sc)
view = ctx.camera_view(cam, RasterSettings())
view.forward(0.0)
rng = np.random.default_rng(6)
n = ctx.L.splatb200_conv_decoder_params()
params = rng.normal(0, 0.08, n).astype(np.float32)
emb = rng.normal(0, 1, 8).astype(np.float32)
g_image = rng.normal(0, 1, (view.P, 3)).astype(np.float32)
g_up = torch.zeros((view.P, 16), dtype=torch.float32, device="cuda")
fwd, bwd = [], []
for _ in range(reps):
    fwd.append(view.decode_image(params, emb, download=False, timed=True)[1])
    bwd.append(view.decode_image_backward(g_image, g_up.data_ptr(), timed=True)[2])
P = view.P
flops_conv = 2.0 * P * 9 * 32 * 32
print(f"decode_image 1920x1080: forward {min(fwd):.3f} ms (5 convolutions = {5 * flops_conv / 1e9:.0f} GFLOP -> "
      f"{5 * flops_conv / min(fwd) / 1e9:.0f} TFLOP/s tf32), backward {min(bwd):.3f} ms "
      f"({10 * flops_conv / min(bwd) / 1e9:.0f} TFLOP/s)")
