"""On-disk formats either side of the hot path: SPZ1 scenes and LPC1 lidar sweeps.

The reference ships no I/O code; the formats are SPEC.md:93 (SPZ1: "a structured-text header (JSON-style: counts, D_f,
actor tracks, sensor models) followed by little-endian 32-bit-float binary blocks in declared order (means, scale_logs,
quaternions, opacity_logits, colors, features, actor_ids as 32-bit ints). Round-trip must be bit-exact in fast mode"),
SPEC.md:401 ("Weights serialized inside the SPZ1 scene file as named float blocks") and SPEC.md:252 (LPC1:
"structured-text header (count, sensor id, sweep start/end times) + binary little-endian 32-bit floats: x, y, z,
intensity, timestamp per point; intensity in [0,1]; a validity flag byte per point for ray-drop ground truth").
What SPEC leaves open is fixed here: the file starts with the ASCII line `<MAGIC> <header bytes>\\n`, then the UTF-8 JSON
header of exactly that many bytes, then the blocks, each exactly as long as the header declares, nothing after them.

Host-side only (numpy): the loaded arrays go to `Context.upload_scene` / `Context.assign_points_to_tiles` unchanged.
"""
import json
from typing import Dict, Optional, Sequence

import numpy as np

from .model import ActorTrack, CameraModel, LidarModel, Scene

SPZ1_BLOCKS = ("mean", "scale_log", "quat", "opacity_logit", "color", "feature")   # declared order, then actor_id


class FormatError(ValueError):
    pass


def _write(path, magic: str, header: dict, blocks: Sequence[np.ndarray]):
    h = json.dumps(header, sort_keys=True).encode("utf-8")
    with open(path, "wb") as f:
        f.write(f"{magic} {len(h)}\n".encode("ascii"))
        f.write(h)
        for b in blocks:
            f.write(np.ascontiguousarray(b).tobytes())


def _read_header(f, magic: str) -> dict:
    line = f.readline(64)
    parts = line.split()
    if len(parts) != 2 or parts[0] != magic.encode("ascii") or not parts[1].isdigit() or not line.endswith(b"\n"):
        raise FormatError(f"not a {magic} file")
    n = int(parts[1])
    h = f.read(n)
    if len(h) != n:
        raise FormatError(f"{magic}: truncated header")
    try:
        return json.loads(h.decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as e:
        raise FormatError(f"{magic}: bad header ({e})") from None


def _read_block(f, dtype, count: int, what: str) -> np.ndarray:
    nbytes = int(count) * np.dtype(dtype).itemsize
    raw = f.read(nbytes)
    if len(raw) != nbytes:
        raise FormatError(f"truncated block {what}: {len(raw)} of {nbytes} bytes")
    return np.frombuffer(raw, dtype=dtype).copy()


def _f32(a):
    return np.ascontiguousarray(a, dtype="<f4")


def _vec(a):
    return [float(x) for x in np.asarray(a, np.float64).ravel()]


def _camera_header(c: CameraModel, embedding=None) -> dict:
    return {"fx": c.fx, "fy": c.fy, "cx": c.cx, "cy": c.cy, "width": int(c.width), "height": int(c.height), "R": _vec(c.R),
            "t": _vec(c.t), "vel_lin": _vec(c.vel_lin), "vel_ang": _vec(c.vel_ang), "shutter_duration": c.shutter_duration,
            "time_offset": c.time_offset, "timestamp": c.timestamp,
            "embedding": _vec(np.zeros(8) if embedding is None else embedding)}


def _lidar_header(l: LidarModel) -> dict:
    return {"elevation_channels": _vec(l.elevation_channels), "azimuth_resolution": l.azimuth_resolution,
            "scan_duration": l.scan_duration, "beam_divergence_h": l.beam_divergence_h, "beam_divergence_v": l.beam_divergence_v,
            "R": _vec(l.R), "t": _vec(l.t), "vel_lin": _vec(l.vel_lin), "vel_ang": _vec(l.vel_ang), "timestamp": l.timestamp,
            "max_range": l.max_range}


def _track_header(t: ActorTrack) -> dict:
    return {"stamps": _vec(t.stamps), "R": _vec(t.R), "t": _vec(t.t), "pose_offset": _vec(t.pose_offset), "vel_lin": _vec(t.vel_lin),
            "vel_ang": _vec(t.vel_ang), "vel_offset": _vec(t.vel_offset), "init_velocity_from_poses": bool(t.init_velocity_from_poses),
            "box_size": _vec(t.box_size)}


def save_spz1(path, scene: Scene, cameras: Sequence[CameraModel] = (), lidars: Sequence[LidarModel] = (),
              weights: Optional[Dict[str, np.ndarray]] = None, embeddings: Optional[Sequence[np.ndarray]] = None):
    """Scene (GaussianSet + actor tracks), sensor models and named float blocks (decoder weights) -> one SPZ1 file.
    The float blocks hold the scene's values rounded to fp32 — the library's own precision ("fast mode")."""
    weights = dict(weights or {})
    header = {"format": "SPZ1", "count": int(scene.n), "d_f": int(scene.d_f),
              "blocks": [*SPZ1_BLOCKS, "actor_id"],
              "actor_tracks": [_track_header(t) for t in scene.tracks],
              "cameras": [_camera_header(c, None if embeddings is None else embeddings[k]) for k, c in enumerate(cameras)],
              "lidars": [_lidar_header(l) for l in lidars],
              "weights": [{"name": k, "count": int(np.asarray(v).size)} for k, v in weights.items()]}
    blocks = [_f32(getattr(scene, k)) for k in SPZ1_BLOCKS] + [np.ascontiguousarray(scene.actor_id, dtype="<i4")]
    blocks += [_f32(v) for v in weights.values()]
    _write(path, "SPZ1", header, blocks)


def load_spz1(path) -> dict:
    """-> {"scene": Scene (fp32 arrays), "cameras": [...], "embeddings": [...], "lidars": [...], "weights": {name: fp32}}"""
    with open(path, "rb") as f:
        h = _read_header(f, "SPZ1")
        try:
            n, d_f = int(h["count"]), int(h["d_f"])
            if h.get("format") != "SPZ1" or h["blocks"] != [*SPZ1_BLOCKS, "actor_id"] or n < 0 or d_f < 0:
                raise KeyError("blocks")
            width = {"mean": 3, "scale_log": 3, "quat": 4, "opacity_logit": 1, "color": 3, "feature": d_f}
            arrays = {}
            for k in SPZ1_BLOCKS:
                a = _read_block(f, "<f4", n * width[k], k)
                arrays[k] = a.reshape(n, width[k]) if k != "opacity_logit" else a
            actor_id = _read_block(f, "<i4", n, "actor_id")
            weights = {w["name"]: _read_block(f, "<f4", int(w["count"]), w["name"]) for w in h["weights"]}
            if f.read(1):
                raise FormatError("SPZ1: bytes after the last declared block")
            tracks = [ActorTrack(stamps=np.array(t["stamps"]), R=np.array(t["R"]), t=np.array(t["t"]),
                                 pose_offset=np.array(t["pose_offset"]), vel_lin=np.array(t["vel_lin"]),
                                 vel_ang=np.array(t["vel_ang"]), vel_offset=np.array(t["vel_offset"]),
                                 init_velocity_from_poses=bool(t["init_velocity_from_poses"]),
                                 box_size=np.array(t.get("box_size", [0.0, 0.0, 0.0]))) for t in h["actor_tracks"]]
            cams, embs = [], []
            for c in h["cameras"]:
                cams.append(CameraModel(fx=c["fx"], fy=c["fy"], cx=c["cx"], cy=c["cy"], width=c["width"], height=c["height"],
                                        R=np.array(c["R"]).reshape(3, 3), t=np.array(c["t"]), vel_lin=np.array(c["vel_lin"]),
                                        vel_ang=np.array(c["vel_ang"]), shutter_duration=c["shutter_duration"],
                                        time_offset=c["time_offset"], timestamp=c["timestamp"]))
                embs.append(np.array(c["embedding"], np.float32))
            lids = [LidarModel(elevation_channels=np.array(l["elevation_channels"]), azimuth_resolution=l["azimuth_resolution"],
                               scan_duration=l["scan_duration"], beam_divergence_h=l["beam_divergence_h"],
                               beam_divergence_v=l["beam_divergence_v"], R=np.array(l["R"]).reshape(3, 3), t=np.array(l["t"]),
                               vel_lin=np.array(l["vel_lin"]), vel_ang=np.array(l["vel_ang"]), timestamp=l["timestamp"],
                               max_range=l["max_range"]) for l in h["lidars"]]
        except (KeyError, TypeError, ValueError) as e:
            if isinstance(e, FormatError):
                raise
            raise FormatError(f"SPZ1: bad header field ({e})") from None
    scene = Scene(arrays["mean"], arrays["scale_log"], arrays["quat"], arrays["opacity_logit"], arrays["color"],
                  arrays["feature"], actor_id, tracks)
    return {"scene": scene, "cameras": cams, "embeddings": embs, "lidars": lids, "weights": weights}


def save_lpc1(path, xyz, intensity, timestamps, valid, sensor_id: str, sweep_start: float, sweep_end: float):
    """One lidar sweep: per point x, y, z, intensity in [0, 1], capture timestamp (fp32), then one validity byte per
    point (0: the beam returned nothing — ray-drop ground truth)."""
    xyz = _f32(xyz).reshape(-1, 3)
    n = len(xyz)
    inten, stamps = _f32(intensity).reshape(n), _f32(timestamps).reshape(n)
    flags = np.ascontiguousarray(np.asarray(valid).reshape(n) != 0, dtype=np.uint8)
    live = inten[flags != 0]
    if live.size and (not np.isfinite(live).all() or live.min() < 0.0 or live.max() > 1.0):
        raise FormatError("LPC1: intensity outside [0, 1]")
    header = {"format": "LPC1", "count": n, "sensor_id": str(sensor_id), "sweep_start": float(sweep_start),
              "sweep_end": float(sweep_end), "fields": ["x", "y", "z", "intensity", "timestamp"]}
    _write(path, "LPC1", header, [np.concatenate([xyz, inten[:, None], stamps[:, None]], axis=1), flags])


def load_lpc1(path) -> dict:
    """-> {"xyz" (n,3), "intensity" (n,), "timestamps" (n,), "valid" (n,) bool, "sensor_id", "sweep_start", "sweep_end"};
    xyz and timestamps are what `Context.assign_points_to_tiles` takes."""
    with open(path, "rb") as f:
        h = _read_header(f, "LPC1")
        try:
            n = int(h["count"])
            if h.get("format") != "LPC1" or n < 0 or h["fields"] != ["x", "y", "z", "intensity", "timestamp"]:
                raise KeyError("fields")
            sensor_id, t0, t1 = str(h["sensor_id"]), float(h["sweep_start"]), float(h["sweep_end"])
        except (KeyError, TypeError, ValueError) as e:
            raise FormatError(f"LPC1: bad header field ({e})") from None
        pts = _read_block(f, "<f4", 5 * n, "points").reshape(n, 5)
        flags = _read_block(f, np.uint8, n, "validity")
        if f.read(1):
            raise FormatError("LPC1: bytes after the last declared block")
    return {"xyz": pts[:, :3].copy(), "intensity": pts[:, 3].copy(), "timestamps": pts[:, 4].copy(), "valid": flags != 0,
            "sensor_id": sensor_id, "sweep_start": t0, "sweep_end": t1}
