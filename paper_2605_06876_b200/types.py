"""Host-side mirror of the reference's operator types.

Same names, fields, defaults, validation and exceptions as the reference
package so a caller can switch imports:

* ``Gaussian3D``, ``Camera``, ``Scene``, ``AdpSplitConfig``  ref/scene.py:54-180
* ``DensifyStats``, ``CandidateRecord``, ``SplitReport``     ref/adc.py:30-70
* ``InvariantError``                                         ref/scene.py:39-40
* ``DegenerateRayError``                                     ref/child_init.py:24-25

The operator (``operator.py``) is duck-typed: objects of the reference
package itself are accepted too.
"""

from __future__ import annotations

from dataclasses import dataclass, field, fields, replace

import numpy as np


class InvariantError(ValueError):
    """A domain-type invariant was violated."""


class DegenerateRayError(ValueError):
    """The Mahalanobis quadratic along the ray is numerically singular."""


def _vec(x, n, name):
    a = np.asarray(x, dtype=np.float64)
    if a.shape != (n,):
        raise InvariantError(f"{name} must be a {n}-vector, got shape {a.shape}")
    return a


@dataclass(frozen=True)
class Gaussian3D:
    """One anisotropic splat (ref/scene.py:54-81): unit quaternion (w,x,y,z),
    positive scales, opacity in (0,1), SH colour (DC + up to 15 rest terms)."""

    mu: np.ndarray
    scale: np.ndarray
    rot: np.ndarray
    opacity: float
    sh_dc: np.ndarray
    sh_rest: tuple = ()

    def __post_init__(self):
        object.__setattr__(self, "mu", _vec(self.mu, 3, "mu"))
        object.__setattr__(self, "scale", _vec(self.scale, 3, "scale"))
        object.__setattr__(self, "rot", _vec(self.rot, 4, "rot"))
        object.__setattr__(self, "sh_dc", _vec(self.sh_dc, 3, "sh_dc"))
        object.__setattr__(self, "sh_rest", tuple(_vec(c, 3, "sh_rest") for c in self.sh_rest))
        object.__setattr__(self, "opacity", float(self.opacity))
        if abs(np.linalg.norm(self.rot) - 1.0) > 1e-9:
            raise InvariantError(f"rot quaternion not unit: {self.rot}")
        if not np.all(self.scale > 0):
            raise InvariantError(f"scale components must be > 0: {self.scale}")
        if not (0.0 < self.opacity < 1.0):
            raise InvariantError(f"opacity must lie in (0,1): {self.opacity}")
        if len(self.sh_rest) > 15:
            raise InvariantError("sh_rest exceeds degree-3 coefficient count")


@dataclass(frozen=True)
class Camera:
    """Pinhole view; r_c2w columns are right, down, forward (ref/scene.py:84-128)."""

    r_c2w: np.ndarray
    center: np.ndarray
    f_x: float
    f_y: float
    p_x: float
    p_y: float
    width: int
    height: int

    def __post_init__(self):
        r = np.asarray(self.r_c2w, dtype=np.float64)
        if r.shape != (3, 3):
            raise InvariantError(f"r_c2w must be 3x3, got {r.shape}")
        if np.max(np.abs(r.T @ r - np.eye(3))) >= 1e-8:
            raise InvariantError("r_c2w is not orthonormal")
        object.__setattr__(self, "r_c2w", r)
        object.__setattr__(self, "center", _vec(self.center, 3, "center"))
        for name in ("f_x", "f_y", "p_x", "p_y"):
            object.__setattr__(self, name, float(getattr(self, name)))
        object.__setattr__(self, "width", int(self.width))
        object.__setattr__(self, "height", int(self.height))
        if self.f_x <= 0 or self.f_y <= 0:
            raise InvariantError("focal lengths must be positive")
        if not (0 <= self.p_x < self.width and 0 <= self.p_y < self.height):
            raise InvariantError("principal point outside image")

    @property
    def right(self):
        return self.r_c2w[:, 0]

    @property
    def down(self):
        return self.r_c2w[:, 1]

    @property
    def forward(self):
        return self.r_c2w[:, 2]


@dataclass
class Scene:
    """Ordered Gaussians plus the bounding-sphere radius (ref/scene.py:131-144)."""

    gaussians: list
    extent: float

    def __post_init__(self):
        self.extent = float(self.extent)
        if self.extent <= 0:
            raise InvariantError("scene extent must be > 0")

    def __len__(self):
        return len(self.gaussians)


@dataclass
class AdpSplitConfig:
    """Operator hyper-parameters, paper defaults (ref/scene.py:147-180)."""

    tau_l1: float = 0.1
    r_erode: int = 2
    m_min: int = 5
    l_bands: int = 3
    n_max: int = 19
    v_views: int = 20
    gamma_d: float = 2.0
    gamma_c: float = 0.15
    tau_g: float = 0.0002
    tau_s: float = 0.01
    eta: float = 1.6
    t_interval: int = 100
    eps: float = 1e-9

    def __post_init__(self):
        if not (0.0 < self.tau_l1 < 1.0):
            raise InvariantError("tau_l1 must lie in (0,1)")
        if self.l_bands < 1 or self.n_max < 1 or self.v_views < 1:
            raise InvariantError("l_bands, n_max, v_views must be >= 1")
        if self.gamma_d < 0 or self.gamma_c < 0:
            raise InvariantError("gamma_d, gamma_c must be >= 0")
        if self.eta <= 0 or self.eps <= 0:
            raise InvariantError("eta and eps must be > 0")

    def with_overrides(self, overrides: dict) -> "AdpSplitConfig":
        known = {f.name for f in fields(self)}
        bad = set(overrides) - known
        if bad:
            raise KeyError(f"unknown config fields: {sorted(bad)}")
        return replace(self, **overrides)


@dataclass
class DensifyStats:
    """Accumulated viewspace-gradient norms and visibility counts (ref/adc.py:30-46)."""

    grad_accum: np.ndarray
    denom: np.ndarray

    @classmethod
    def zeros(cls, n: int) -> "DensifyStats":
        return cls(grad_accum=np.zeros(n), denom=np.zeros(n))

    def g(self) -> np.ndarray:
        out = np.zeros_like(self.grad_accum)
        seen = self.denom > 0
        out[seen] = self.grad_accum[seen] / self.denom[seen]
        return out


@dataclass
class CandidateRecord:
    """Per split-candidate outcome (ref/adc.py:49-57)."""

    index: int
    regions_per_view: list
    proposals: int = 0
    merged: int = 0
    children_inserted: int = 0
    fallback: bool = False
    reset: bool = False


@dataclass
class SplitReport:
    """Step report (ref/adc.py:60-70); index_map[new] = old index or -1."""

    count_before: int
    count_after: int = 0
    clones: list = field(default_factory=list)
    candidates: list = field(default_factory=list)
    sampled_views: list = field(default_factory=list)
    merge_edges: int = 0
    index_map: np.ndarray = None
    reset_indices: list = field(default_factory=list)
