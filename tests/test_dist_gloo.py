"""The N > 1 path on CPU: world_size-2 gloo. Each rank renders its share of a multi-frame batch (the CPU oracle stands in
for the kernels, which need a GPU), the SceneParamGrads buffers are all-reduced, and the result must equal the
single-process sum over all frames; frame assignment must be a partition."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_16816_b200 import dist as sdist

KEYS = ("d_mean", "d_scale_log", "d_quat", "d_opacity_logit", "d_color", "d_feature")
N_FRAMES = 5


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _frame_grads(frame):
    """flat 27*N buffer in the ABI's layout [d_mean 3N | d_scale_log 3N | d_quat 4N | d_opacity_logit N | d_color 3N | d_feature 13N]"""
    import bench
    from oracle import oracle_py as op
    from paper_2411_16816_b200 import synth
    from paper_2411_16816_b200.model import RasterSettings
    sc = synth.make_scene(600, seed=41, r_max=30.0, scale_mean=0.1)
    o = op.OracleScene(sc, np.float64)
    lid, cam = bench.frame_sensors(frame)
    cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy = 96, 64, 50.0, 50.0, 48.0, 32.0
    lid32 = synth.lidar32(position=(1.5 * frame, 0.0, 1.8))
    st = RasterSettings()
    v = o.render_camera(cam, st)
    gb, ga = synth.upstream(v.P, seed=frame)
    v.backward(gb, ga)
    rays = synth.grid_rays(lid32)
    v = o.render_lidar(lid32, rays, st)
    gb, ga = synth.upstream(v.P, seed=100 + frame)
    gb[:, 14:] = 0
    v.backward(gb, ga)
    g = o.grads()
    return np.concatenate([np.asarray(g[k], np.float64).ravel() for k in KEYS])


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = sdist.assign_frames(N_FRAMES, world, rank)
        buf = None
        for f in mine:
            g = _frame_grads(f)
            buf = g if buf is None else buf + g            # backward accumulates (+=) across a rank's frames
        t = torch.from_numpy(buf.copy())
        sdist.allreduce_grads(t)
        ms = sdist.max_over_ranks(10.0 * (rank + 1))
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), t.numpy())
        np.save(os.path.join(out_dir, f"ms{rank}.npy"), np.array([ms]))
        np.save(os.path.join(out_dir, f"frames{rank}.npy"), np.array(mine))
    finally:
        dist.destroy_process_group()


def test_frame_assignment_is_a_partition():
    for world in (1, 2, 4, 8):
        for n in (0, 1, 7, 64):
            seen = sorted(f for r in range(world) for f in sdist.assign_frames(n, world, r))
            assert seen == list(range(n))
            sizes = [len(sdist.assign_frames(n, world, r)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    costs = [5, 1, 1, 1, 4, 4, 1, 1]
    parts = [sdist.assign_frames(8, 2, r, costs) for r in range(2)]
    assert sorted(parts[0] + parts[1]) == list(range(8))
    loads = [sum(costs[f] for f in p) for p in parts]
    assert abs(loads[0] - loads[1]) <= 1            # cost-balanced (LPT)
    with pytest.raises(ValueError):
        sdist.assign_frames(4, 2, 2)


def test_two_rank_allreduce_equals_single_process(tmp_path, oracle_lib):
    world = 2
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    single = sum(_frame_grads(f) for f in range(N_FRAMES))
    r0, r1 = np.load(tmp_path / "rank0.npy"), np.load(tmp_path / "rank1.npy")
    assert np.array_equal(r0, r1)                                       # every rank holds the same reduced buffer
    assert np.allclose(r0, single, rtol=1e-12, atol=1e-12 * np.abs(single).max())
    assert np.abs(single).max() > 0
    assert float(np.load(tmp_path / "ms0.npy")[0]) == 20.0 == float(np.load(tmp_path / "ms1.npy")[0])   # MAX over ranks
    f0, f1 = np.load(tmp_path / "frames0.npy"), np.load(tmp_path / "frames1.npy")
    assert sorted(list(f0) + list(f1)) == list(range(N_FRAMES))
