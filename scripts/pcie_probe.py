"""GPU-box probe: PCIe bandwidth of pinned copies one way and both ways at once (bounds the end-to-end frame).
  python scripts/pcie_probe.py"""
import torch

MB = 141
n = MB * (1 << 20) // 4
h_up = torch.empty(n, dtype=torch.float32).pin_memory()
h_dn = torch.empty(n, dtype=torch.float32).pin_memory()
d_up = torch.empty(n, dtype=torch.float32, device="cuda")
d_dn = torch.ones(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(up, dn, chunks=1, reps=10):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    c = n // chunks
    for _ in range(reps):
        for k in range(chunks):
            if up:
                with torch.cuda.stream(s1):
                    d_up[k * c:(k + 1) * c].copy_(h_up[k * c:(k + 1) * c], non_blocking=True)
            if dn:
                with torch.cuda.stream(s2):
                    h_dn[k * c:(k + 1) * c].copy_(d_dn[k * c:(k + 1) * c], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return ms, MB * 1.048576 / ms


for chunks in (1, 8):
    for up, dn, name in ((1, 0, "H2D alone"), (0, 1, "D2H alone"), (1, 1, "both at once")):
        run(up, dn, chunks, 2)
        ms, gbs = run(up, dn, chunks)
        print(f"{name:14s} {chunks} chunk(s): {ms:.3f} ms per {MB} MB per direction = {gbs:.1f} GB/s per direction", flush=True)
