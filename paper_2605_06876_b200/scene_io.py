"""Binary scene and camera files for large fixtures.

The reference stores scenes and cameras as ``repr`` text (ref/scene.py:279-381),
which parses 1-8M Gaussians at a few MB/s.  The binary v1 files hold the same
float64 values as little-endian structure-of-arrays blocks, so a load is one
read per field and a scene goes to the device as ``GaussianTensors`` without a
per-Gaussian Python object.  The text format itself is not re-implemented here
(SURVEY.md §2 marks it out of scope); tests/golden/make_io_golden.py converts
files written and parsed by the reference into these binary fixtures.

  scene:   b"ADPSSCN1" | u64 N | u32 K | u32 0 | f64 extent |
           f64 mu[N,3] | scale[N,3] | rot[N,4] | opacity[N] | sh_dc[N,3] | sh_rest[N,K,3]
  cameras: b"ADPSCAM1" | u64 M | f64 rows[M,16] (r_c2w 9, center 3, f_x f_y p_x p_y)
           | i64 size[M,2] (width, height)

Invariants are checked vectorised with the reference's rules
(ref/scene.py:54-128) on every load.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .types import Camera, Gaussian3D, InvariantError, Scene

SCENE_MAGIC = b"ADPSSCN1"
CAMERA_MAGIC = b"ADPSCAM1"


class SceneFormatError(ValueError):
    """A scene or camera file is malformed (ref/scene.py:43-44)."""


@dataclass
class SceneArrays:
    """A scene as float64 structure of arrays (uniform SH-rest count K)."""

    mu: np.ndarray        # [N,3]
    scale: np.ndarray     # [N,3]
    rot: np.ndarray       # [N,4] (w,x,y,z)
    opacity: np.ndarray   # [N]
    sh_dc: np.ndarray     # [N,3]
    sh_rest: np.ndarray   # [N,K,3]
    extent: float

    def __len__(self):
        return int(self.mu.shape[0])

    def fields(self):
        return (self.mu, self.scale, self.rot, self.opacity, self.sh_dc, self.sh_rest)


def check_invariants(a: SceneArrays, where: str = "") -> None:
    """The reference's per-Gaussian invariants (ref/scene.py:54-81, 131-144), vectorised;
    the first offending Gaussian is reported as the reference reports it."""
    if not a.extent > 0:
        raise InvariantError("scene extent must be > 0")
    if a.sh_rest.shape[1] > 15:
        raise InvariantError("sh_rest exceeds degree-3 coefficient count")
    bad_rot = np.abs(np.linalg.norm(a.rot, axis=1) - 1.0) > 1e-9
    bad_scale = ~np.all(a.scale > 0, axis=1)
    bad_op = ~((a.opacity > 0.0) & (a.opacity < 1.0))
    bad = bad_rot | bad_scale | bad_op
    if not bad.any():
        return
    i = int(np.argmax(bad))
    if bad_rot[i]:
        msg = f"rot quaternion not unit: {a.rot[i]}"
    elif bad_scale[i]:
        msg = f"scale components must be > 0: {a.scale[i]}"
    else:
        msg = f"opacity must lie in (0,1): {a.opacity[i]}"
    loc = f"{where}: " if where else ""
    raise InvariantError(f"{loc}Gaussian {i}: {msg}")


# ---------------------------------------------------------------- conversions
def scene_to_arrays(scene) -> SceneArrays:
    """Reference-style ``Scene`` (list of Gaussian3D) -> SoA; every Gaussian must
    carry the same number of SH-rest terms."""
    gs = scene.gaussians
    ks = {len(g.sh_rest) for g in gs}
    if len(ks) > 1:
        raise SceneFormatError(f"ragged sh_rest counts {sorted(ks)}: the SoA layout needs one K")
    k = ks.pop() if ks else 0
    n = len(gs)
    rest = np.zeros((n, k, 3))
    for i, g in enumerate(gs):
        for j, c in enumerate(g.sh_rest):
            rest[i, j] = c
    return SceneArrays(np.array([g.mu for g in gs], dtype=np.float64).reshape(n, 3),
                       np.array([g.scale for g in gs], dtype=np.float64).reshape(n, 3),
                       np.array([g.rot for g in gs], dtype=np.float64).reshape(n, 4),
                       np.array([g.opacity for g in gs], dtype=np.float64).reshape(n),
                       np.array([g.sh_dc for g in gs], dtype=np.float64).reshape(n, 3),
                       rest, float(scene.extent))


def arrays_to_scene(a: SceneArrays) -> Scene:
    gs = [Gaussian3D(mu=a.mu[i], scale=a.scale[i], rot=a.rot[i], opacity=float(a.opacity[i]),
                     sh_dc=a.sh_dc[i], sh_rest=tuple(a.sh_rest[i])) for i in range(len(a))]
    return Scene(gaussians=gs, extent=a.extent)


def scene_tensors(a: SceneArrays, device="cuda"):
    """SceneArrays -> (operator.GaussianTensors fp32 on ``device``, extent)."""
    from .operator import GaussianTensors   # needs torch + the extension
    return GaussianTensors.from_numpy(a.mu, a.scale, a.rot, a.opacity, a.sh_dc,
                                      a.sh_rest if a.sh_rest.shape[1] else None, device=device), a.extent


def _camera(vals):
    return Camera(r_c2w=np.array(vals[0:9]).reshape(3, 3), center=vals[9:12], f_x=vals[12], f_y=vals[13],
                  p_x=vals[14], p_y=vals[15], width=int(vals[16]), height=int(vals[17]))


# ---------------------------------------------------------------- binary v1
_SCENE_HDR = struct.Struct("<8sQIId")
_CAM_HDR = struct.Struct("<8sQ")


def save_scene_bin(scene, path) -> None:
    """Write the binary v1 scene (a Scene or SceneArrays)."""
    a = scene if isinstance(scene, SceneArrays) else scene_to_arrays(scene)
    n, k = len(a), int(a.sh_rest.shape[1])
    with open(path, "wb") as f:
        f.write(_SCENE_HDR.pack(SCENE_MAGIC, n, k, 0, float(a.extent)))
        for x in a.fields():
            f.write(np.ascontiguousarray(x, dtype="<f8").tobytes())


def load_scene_bin(path) -> SceneArrays:
    """Read a binary v1 scene into SoA arrays; raises SceneFormatError on a bad
    magic or a truncated file, InvariantError on invalid Gaussians."""
    raw = Path(path).read_bytes()
    if len(raw) < _SCENE_HDR.size:
        raise SceneFormatError(f"{path}: truncated header")
    magic, n, k, _, extent = _SCENE_HDR.unpack_from(raw, 0)
    if magic != SCENE_MAGIC:
        raise SceneFormatError(f"{path}: not a binary v1 scene (magic {magic!r})")
    if n == 0:
        raise SceneFormatError(f"{path}: scene contains no Gaussians")
    widths = (3, 3, 4, 1, 3, 3 * k)
    need = _SCENE_HDR.size + 8 * n * sum(widths)
    if len(raw) != need:
        raise SceneFormatError(f"{path}: {len(raw)} bytes, expected {need} for N={n}, K={k} (truncated?)")
    out, off = [], _SCENE_HDR.size
    for w in widths:
        out.append(np.frombuffer(raw, dtype="<f8", count=n * w, offset=off).astype(np.float64))
        off += 8 * n * w
    a = SceneArrays(out[0].reshape(n, 3), out[1].reshape(n, 3), out[2].reshape(n, 4), out[3],
                    out[4].reshape(n, 3), out[5].reshape(n, k, 3), float(extent))
    check_invariants(a, str(path))
    return a


def save_cameras_bin(cameras, path) -> None:
    rows = np.array([[*c.r_c2w.ravel(), *c.center, c.f_x, c.f_y, c.p_x, c.p_y] for c in cameras],
                    dtype="<f8").reshape(len(cameras), 16)
    size = np.array([[c.width, c.height] for c in cameras], dtype="<i8").reshape(len(cameras), 2)
    with open(path, "wb") as f:
        f.write(_CAM_HDR.pack(CAMERA_MAGIC, len(cameras)))
        f.write(rows.tobytes())
        f.write(size.tobytes())


def load_cameras_bin(path) -> list:
    raw = Path(path).read_bytes()
    if len(raw) < _CAM_HDR.size:
        raise SceneFormatError(f"{path}: truncated header")
    magic, m = _CAM_HDR.unpack_from(raw, 0)
    if magic != CAMERA_MAGIC:
        raise SceneFormatError(f"{path}: not a binary v1 camera file (magic {magic!r})")
    need = _CAM_HDR.size + m * (16 + 2) * 8
    if len(raw) != need:
        raise SceneFormatError(f"{path}: {len(raw)} bytes, expected {need} for M={m} (truncated?)")
    rows = np.frombuffer(raw, dtype="<f8", count=16 * m, offset=_CAM_HDR.size).reshape(m, 16)
    size = np.frombuffer(raw, dtype="<i8", count=2 * m, offset=_CAM_HDR.size + 128 * m).reshape(m, 2)
    cameras = []
    for i in range(m):
        try:
            cameras.append(_camera([*rows[i], *size[i]]))
        except InvariantError as exc:
            raise InvariantError(f"{path}: camera {i}: {exc}") from exc
    return cameras
