"""SPZ1 / LPC1: round trips are bit-exact in fp32, malformed files are rejected. CPU only."""
import numpy as np
import pytest

from paper_2411_16816_b200 import io as sio
from paper_2411_16816_b200 import synth


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def test_spz1_round_trip_is_bit_exact(tmp_path):
    sc = synth.make_scene(500, seed=3, n_actors=3).astype(np.float32)
    sc.mean[7, 1] = np.float32(-0.0)                      # sign of zero and a denormal survive
    sc.color[9, 2] = np.float32(1e-42)
    cams = [synth.make_camera(width=320, height=192, yaw=0.3), synth.make_camera()]
    lids = [synth.lidar128()]
    rng = np.random.default_rng(0)
    if sc.tracks:
        sc.tracks[0].box_size = np.array([4.5, 1.9, 1.6])     # ActorTrack::box_size (scene.hpp:51) travels with the track
    weights = {"conv_decoder": rng.normal(size=46438).astype(np.float32), "lidar_head": rng.normal(size=610).astype(np.float32)}
    embs = [rng.normal(size=8).astype(np.float32) for _ in cams]
    p = tmp_path / "scene.spz1"
    sio.save_spz1(p, sc, cams, lids, weights, embs)
    got = sio.load_spz1(p)
    g = got["scene"]
    for k in ("mean", "scale_log", "quat", "opacity_logit", "color", "feature", "actor_id"):
        a, b = getattr(sc, k), getattr(g, k)
        assert a.shape == b.shape and a.dtype == b.dtype and np.array_equal(_bits(a), _bits(b)), k
    assert len(g.tracks) == 3
    for a, b in zip(sc.tracks, g.tracks):
        for k in ("stamps", "R", "t", "pose_offset", "vel_lin", "vel_ang", "vel_offset", "box_size"):
            assert np.array_equal(getattr(a, k), getattr(b, k)), k      # doubles through JSON repr: exact
        assert a.init_velocity_from_poses == b.init_velocity_from_poses
    for a, b in zip(cams, got["cameras"]):
        assert np.array_equal(a.packed(np.float64), b.packed(np.float64))
    for a, b in zip(embs, got["embeddings"]):
        assert np.array_equal(a, b)
    assert np.array_equal(lids[0].elevation_channels, got["lidars"][0].elevation_channels)
    assert lids[0].azimuth_resolution == got["lidars"][0].azimuth_resolution
    for k, v in weights.items():
        assert np.array_equal(_bits(v), _bits(got["weights"][k]))
    # load -> save reproduces the file byte for byte
    p2 = tmp_path / "again.spz1"
    sio.save_spz1(p2, g, got["cameras"], got["lidars"], got["weights"], got["embeddings"])
    assert p.read_bytes() == p2.read_bytes()


def test_spz1_empty_scene_and_malformed_files(tmp_path):
    sc = synth.make_scene(0, seed=1).astype(np.float32)
    p = tmp_path / "empty.spz1"
    sio.save_spz1(p, sc)
    g = sio.load_spz1(p)["scene"]
    assert g.n == 0 and g.feature.shape == (0, 13)
    full = tmp_path / "full.spz1"
    sio.save_spz1(full, synth.make_scene(50, seed=2).astype(np.float32))
    raw = full.read_bytes()
    for name, data in (("trunc", raw[:-5]), ("extra", raw + b"x"), ("magic", b"SPZ2" + raw[4:]), ("hdr", raw[:12])):
        q = tmp_path / f"{name}.spz1"
        q.write_bytes(data)
        with pytest.raises(sio.FormatError):
            sio.load_spz1(q)
    with pytest.raises(sio.FormatError):
        sio.load_lpc1(full)


def test_lpc1_round_trip_and_validation(tmp_path):
    rng = np.random.default_rng(4)
    n = 1000
    xyz = rng.normal(0, 20, (n, 3)).astype(np.float32)
    inten = rng.uniform(0, 1, n).astype(np.float32)
    stamps = np.sort(rng.uniform(10.0, 10.1, n)).astype(np.float32)
    valid = rng.uniform(size=n) > 0.1
    p = tmp_path / "sweep.lpc1"
    sio.save_lpc1(p, xyz, inten, stamps, valid, "lidar_top", 10.0, 10.1)
    g = sio.load_lpc1(p)
    assert np.array_equal(_bits(g["xyz"]), _bits(xyz)) and np.array_equal(_bits(g["intensity"]), _bits(inten))
    assert np.array_equal(_bits(g["timestamps"]), _bits(stamps)) and np.array_equal(g["valid"], valid)
    assert (g["sensor_id"], g["sweep_start"], g["sweep_end"]) == ("lidar_top", 10.0, 10.1)
    assert p.stat().st_size == len(p.read_bytes()) and p.read_bytes()[-n:] == valid.astype(np.uint8).tobytes()
    bad = inten.copy(); bad[valid.argmax()] = 1.5
    with pytest.raises(sio.FormatError):
        sio.save_lpc1(tmp_path / "bad.lpc1", xyz, bad, stamps, valid, "l", 0.0, 0.1)
    (tmp_path / "trunc.lpc1").write_bytes(p.read_bytes()[:-1])
    with pytest.raises(sio.FormatError):
        sio.load_lpc1(tmp_path / "trunc.lpc1")
    sio.save_lpc1(tmp_path / "none.lpc1", np.zeros((0, 3)), [], [], [], "l", 0.0, 0.0)
    assert sio.load_lpc1(tmp_path / "none.lpc1")["xyz"].shape == (0, 3)
