"""B200-native AdpSplit split operator (arXiv 2605.06876), drop-in for the
reference package's ``adpsplit_step`` (ref/adc.py:143-245).

Public API mirrors the reference (ref/__init__.py): ``adpsplit_step``,
``vanilla_densify``, ``remap_stats_ref`` (ref ``remap_stats``),
``render``, ``DensifyStats``, ``SplitReport``, ``CandidateRecord``,
``AdpSplitConfig``, ``Gaussian3D``, ``Camera``, ``Scene`` plus the tensor
API ``densify_step`` / ``render_views`` / ``GaussianTensors`` / ``Plan``.
"""

from .types import (AdpSplitConfig, Camera, CandidateRecord, DegenerateRayError, DensifyStats,
                    Gaussian3D, InvariantError, Scene, SplitReport)

__version__ = "0.2.0"

_OPS = ("adpsplit_step", "render", "densify_step", "render_views", "GaussianTensors", "Plan",
        "StepResult", "sample_views", "camera_rows", "accumulate_stats_", "default_plan",
        "vanilla_densify", "vanilla_densify_step", "remap_stats", "remap_stats_ref", "remap_rows", "prune")


def __getattr__(name):
    # the operator needs torch + libadps.so; import lazily so the types stay usable anywhere
    if name in _OPS:
        from . import operator as _op
        return getattr(_op, name)
    raise AttributeError(name)


__all__ = ["AdpSplitConfig", "Camera", "CandidateRecord", "DegenerateRayError", "DensifyStats",
           "Gaussian3D", "InvariantError", "Scene", "SplitReport", *_OPS]
