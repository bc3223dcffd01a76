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


# ---- sharded optimizer step: reduce-scatter -> Adam on the shard -> all-gather -----------------
class _NumpyAdamCtx:
    """Stands in for the CUDA context on CPU: the two calls sharded_optimizer_step makes, on flat numpy views of torch
    tensors, with the oracle's Adam (the kernel itself is covered by the GPU tests)."""

    def __init__(self, params_flat, grads, n, d_f):
        self.p, self.g = params_flat.numpy(), grads.numpy()
        self.m, self.v = np.zeros_like(self.p), np.zeros_like(self.p)
        w = [3, 3, 4, 1, 3, d_f]
        self.begin = np.concatenate([[0], np.cumsum([x * n for x in w])])

    comm_world = 0      # no library communicator on CPU: the torch.distributed (gloo) branch is under test

    def join(self):
        pass

    def sync(self):
        pass

    def _slices(self, lo, hi):
        for k in range(6):
            a, b = max(self.begin[k], lo), min(self.begin[k + 1], hi)
            if b > a:
                yield k, int(a), int(b)

    def grads_nonfinite_range(self, lo, hi):
        f = [0] * 6
        for k, a, b in self._slices(lo, hi):
            f[k] = int(not np.isfinite(self.g[a:b]).all())
        return f

    def optimizer_step_range(self, cfg, step, lo, hi, skip_groups=None):
        from oracle import oracle_py as op
        t1 = step + 1.0
        bc1, bc2 = 1.0 / (1.0 - 0.9 ** t1), 1.0 / (1.0 - 0.999 ** t1)
        for k, a, b in self._slices(lo, hi):
            if skip_groups and skip_groups[k]:
                continue
            g = self.g[a:b]
            self.m[a:b] = 0.9 * self.m[a:b] + 0.1 * g
            self.v[a:b] = 0.999 * self.v[a:b] + 0.001 * g * g
            self.p[a:b] -= op.adam_lr(cfg, k, step) * (self.m[a:b] * bc1) / (np.sqrt(self.v[a:b] * bc2) + 1e-15)
        return []


_CFG = {"lr_init": [1.6e-4, 5e-3, 1e-3, 5e-2, 2.5e-3, 2.5e-3], "lr_final": [1.6e-6, 5e-3, 1e-3, 5e-2, 2.5e-3, 2.5e-4],
        "warmup_steps": [0, 0, 0, 0, 0, 2], "total_steps": 10}


def _sharded_worker(rank, world, port, out_dir, n, d_f):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        total = (14 + d_f) * n
        rng = np.random.default_rng(7)                       # same initial parameters everywhere (replicated scene)
        params = torch.from_numpy(rng.normal(size=total))
        ctx = None
        skipped_log = []
        for step in range(4):
            g = np.random.default_rng(100 * step + rank).normal(size=total)   # this rank's local gradients
            if step == 2 and rank == 1:
                g[3 * n + 5] = np.inf                         # a non-finite value in rank 1's scale_log gradients
            grads = torch.from_numpy(g)
            if ctx is None:
                ctx = _NumpyAdamCtx(params, grads, n, d_f)
            ctx.g = grads.numpy()
            skipped_log.append(sdist.sharded_optimizer_step(ctx, grads, params, _CFG, step))
        np.save(os.path.join(out_dir, f"params_{rank}.npy"), params.numpy())
        np.save(os.path.join(out_dir, f"skipped_{rank}.npy"), np.array([len(s) for s in skipped_log]))
    finally:
        dist.destroy_process_group()


def test_sharded_optimizer_step_equals_allreduce_then_step(tmp_path):
    """world_size 2 on gloo: reduce-scatter -> step on the shard -> all-gather gives every rank the parameters that
    all-reduce -> full step gives (total not divisible by the world size: padded shards), moments are only touched on
    the owning shard, and a non-finite gradient on ONE rank skips the group on BOTH."""
    from oracle import oracle_py as op
    n, d_f, world = 37, 13, 2
    total = (14 + d_f) * n
    port = _free_port()
    mp.spawn(_sharded_worker, args=(world, port, str(tmp_path), n, d_f), nprocs=world, join=True)
    # single-process reference: sum of the ranks' gradients, full Adam
    rng = np.random.default_rng(7)
    p = rng.normal(size=total)
    w = [3, 3, 4, 1, 3, d_f]
    begin = np.concatenate([[0], np.cumsum([x * n for x in w])])
    split = lambda a: [a[begin[k]:begin[k + 1]] for k in range(6)]
    params, m, v = split(p), split(np.zeros(total)), split(np.zeros(total))
    for step in range(4):
        g = sum(np.random.default_rng(100 * step + r).normal(size=total) for r in range(world))
        if step == 2:
            g[3 * n + 5] = np.inf
        skipped = op.adam_step(params, split(g), m, v, _CFG, step, np.float64)
        assert skipped == ([1] if step == 2 else [])
    ref = np.concatenate(params)
    for r in range(world):
        got = np.load(tmp_path / f"params_{r}.npy")
        assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), r
        assert list(np.load(tmp_path / f"skipped_{r}.npy")) == [0, 0, 1, 0]
    lo0, hi0 = sdist.shard_range(total, world, 0)
    lo1, hi1 = sdist.shard_range(total, world, 1)
    assert lo0 == 0 and hi0 == lo1 and hi1 == total and hi0 % 4 == 0
