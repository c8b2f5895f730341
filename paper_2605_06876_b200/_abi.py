"""ctypes binding of the C ABI in include/adps.h (libadps.so, built in-tree).

This is the only place Python touches the native library.  There is no
fallback: if the library is missing or CUDA is unavailable the import of the
operator API raises.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ADPS_LIB") or os.path.join(HERE, "libadps.so")   # ADPS_LIB: dev variants

ADPS_OK, ADPS_INVALID_ARG, ADPS_V_TOO_LARGE, ADPS_DEGENERATE_RAY = 0, 1, 2, 3
ADPS_CUDA_ERROR, ADPS_OOM, ADPS_BAD_STATE, ADPS_INTERNAL = 4, 5, 6, 7
CASE_SPLIT, CASE_FALLBACK, CASE_RESET = 0, 1, 2
PARAM_LARGE_THRESHOLD, PARAM_TILE_PATH, PARAM_DEFERRED_TILES = 1, 2, 3
PARAM_NORMALS_CONSUMED, PARAM_NORMALS_STATUS, PARAM_RAW_CACHE = 4, 5, 6
PARAM_RENDER_BINNING, PARAM_RENDER_PAIR_CAP, PARAM_CAP_HUGE = 12, 13, 14
BUF_DOM_FLAG, BUF_REGIONS, BUF_PROPOSALS, BUF_VALID = 1, 2, 3, 4
BUF_CAND_MERGED, BUF_CAND_INS, BUF_CHILDREN, BUF_LO, BUF_THRESHOLDS = 5, 6, 7, 8, 9

vp = C.c_void_p


class Gaussians(C.Structure):
    _fields_ = [("mu", vp), ("scale", vp), ("rot", vp), ("opacity", vp), ("sh_dc", vp),
                ("sh_rest", vp), ("sh_rest_k", C.c_int32)]


class GaussiansOut(C.Structure):
    _fields_ = [("mu", vp), ("scale", vp), ("rot", vp), ("opacity", vp), ("sh_dc", vp),
                ("sh_rest", vp), ("sh_rest_k", C.c_int32)]


class Config(C.Structure):
    _fields_ = [("tau_l1", C.c_double), ("r_erode", C.c_int32), ("m_min", C.c_int32),
                ("l_bands", C.c_int32), ("n_max", C.c_int32), ("v_views", C.c_int32),
                ("reserved0", C.c_int32), ("gamma_d", C.c_double), ("gamma_c", C.c_double),
                ("tau_g", C.c_double), ("tau_s", C.c_double), ("eta", C.c_double),
                ("eps", C.c_double)]


class Counts(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "n_before", "n_out", "n_keep", "n_split", "n_clone", "n_fallback", "n_reset",
        "n_children", "n_inserted", "n_regions", "n_proposals", "merge_edges", "n_partials")] + \
        [("degenerate_ray", C.c_int32), ("reserved1", C.c_int32)]

    def as_dict(self):
        d = dict(zip(_COUNTS_NAMES, _COUNTS_FMT.unpack(bytes(self))))   # one copy, not a getattr per field
        del d["reserved1"]
        return d


_COUNTS_FMT = __import__("struct").Struct("=13q2i")
_COUNTS_NAMES = tuple(f for f, _ in Counts._fields_)
assert _COUNTS_FMT.size == C.sizeof(Counts)


class Report(C.Structure):
    _fields_ = [("cand_index", vp), ("cand_case", vp), ("cand_proposals", vp), ("cand_merged", vp),
                ("regions_per_view", vp), ("clone_index", vp), ("n_views", C.c_int32)]


ABI_VERSION = 3

EXPORTS = (
    "adps_abi_version", "adps_last_error", "adps_plan_create", "adps_plan_destroy", "adps_render",
    "adps_step_phase1", "adps_step_phase1_begin", "adps_step_phase1_end", "adps_step_phase2", "adps_get_report", "adps_get_regions",
    "adps_set_debug_records", "adps_set_debug_maps", "adps_set_timing", "adps_get_timing",
    "adps_accumulate_stats", "adps_get_launch_count", "adps_set_param", "adps_get_param", "adps_normals_pcg64",
    "adps_set_view_sharding", "adps_get_buffer", "adps_step_phase1_refresh", "adps_step_phase1_local",
    "adps_step_phase1_import", "adps_step_phase1_merge", "adps_vanilla_phase1", "adps_reset_flags",
    "adps_remap_rows", "adps_set_parent_sharding", "adps_get_shard", "adps_step_phase1_finish",
    "adps_copy_report", "adps_accumulate_stats_f64", "adps_prune_index", "adps_render_stats",
    "adps_render_fused", "adps_check_guards", "adps_step_capacity", "adps_step_phase1_end_emit",
)

_lib = None


def load(path: str = LIB_PATH):
    """Load libadps.so and declare every exported signature (no GPU needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run __graft_entry__.build() "
                          "(python -m paper_2605_06876_b200.build_ext)")
    lib = C.CDLL(path)
    st = C.c_int
    lib.adps_abi_version.restype = C.c_int
    lib.adps_last_error.restype = C.c_char_p
    lib.adps_plan_create.argtypes = [C.POINTER(vp), C.c_int32, C.c_int64, C.c_int32, C.c_int32, C.c_int32]
    lib.adps_plan_destroy.argtypes = [vp]
    lib.adps_render.argtypes = [vp, vp, C.POINTER(Gaussians), C.c_int64, vp, C.c_int32, vp, vp, vp]
    lib.adps_check_guards.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
    lib.adps_render_fused.argtypes = [vp, vp, C.POINTER(Gaussians), C.c_int64, C.c_double, vp, vp,
                                      C.POINTER(Config), vp, C.c_int32, vp, vp, vp, vp]
    lib.adps_render_stats.argtypes = [vp, vp, C.POINTER(Gaussians), C.c_int64, vp, C.c_int32, vp, vp, vp, vp,
                                      C.POINTER(C.c_uint64)]
    lib.adps_step_phase1.argtypes = [vp, vp, C.POINTER(Gaussians), C.c_int64, C.c_double, vp, vp,
                                     C.POINTER(Config), vp, C.c_int32, vp, vp, vp, C.POINTER(Counts)]
    lib.adps_step_phase1_begin.argtypes = lib.adps_step_phase1.argtypes
    lib.adps_step_phase1_end.argtypes = [vp, vp, C.POINTER(Counts)]
    lib.adps_step_phase2.argtypes = [vp, vp, C.POINTER(Gaussians), vp, C.POINTER(GaussiansOut), vp, vp, vp]
    lib.adps_step_capacity.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    lib.adps_step_phase1_end_emit.argtypes = [vp, vp, C.POINTER(Gaussians), vp, C.POINTER(GaussiansOut), vp, vp, vp,
                                              C.c_int64, C.c_int64, vp, C.POINTER(Counts)]
    lib.adps_get_report.argtypes = [vp, C.POINTER(Report)]
    lib.adps_copy_report.argtypes = [vp, vp, vp, C.c_int64, C.c_int64]
    lib.adps_get_regions.argtypes = [vp] + [C.POINTER(vp)] * 5 + [C.POINTER(C.c_int64)]
    lib.adps_set_debug_records.argtypes = [vp, C.c_int32]
    lib.adps_set_debug_maps.argtypes = [vp, vp, vp]
    lib.adps_set_timing.argtypes = [vp, C.c_int32]
    lib.adps_get_timing.argtypes = [vp, C.POINTER(C.c_double), C.c_int32, C.POINTER(C.c_int32),
                                    C.POINTER(C.c_char_p)]
    lib.adps_accumulate_stats.argtypes = [vp, vp, vp, vp, vp, C.c_int64]
    lib.adps_accumulate_stats_f64.argtypes = [vp, vp, vp, vp, vp, C.c_int64]
    lib.adps_prune_index.argtypes = [vp, vp, vp, vp, C.c_int64, C.c_double, vp, C.POINTER(C.c_int64),
                                     C.POINTER(C.c_int64)]
    lib.adps_get_launch_count.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    lib.adps_set_param.argtypes = [vp, C.c_int32, C.c_int64]
    lib.adps_get_param.argtypes = [vp, C.c_int32, C.POINTER(C.c_int64)]
    lib.adps_set_view_sharding.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32]
    lib.adps_get_buffer.argtypes = [vp, C.c_int32, C.POINTER(vp), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    lib.adps_step_phase1_refresh.argtypes = [vp, vp, C.POINTER(Counts)]
    lib.adps_step_phase1_local.argtypes = [vp, vp, C.POINTER(C.c_int64)]
    lib.adps_step_phase1_import.argtypes = [vp, vp, vp, vp, vp, C.c_int64]
    lib.adps_step_phase1_merge.argtypes = [vp, vp, C.POINTER(Counts)]
    lib.adps_vanilla_phase1.argtypes = [vp, vp, C.POINTER(Gaussians), C.c_int64, C.c_double, vp, vp,
                                        C.POINTER(Config), C.c_int32, C.POINTER(Counts)]
    lib.adps_reset_flags.argtypes = [vp, vp, vp, C.c_int32]
    lib.adps_set_parent_sharding.argtypes = [vp, C.c_int32, C.c_int32]
    lib.adps_get_shard.argtypes = [vp] + [C.POINTER(C.c_int64)] * 4
    lib.adps_step_phase1_finish.argtypes = [vp, vp, C.c_int64, C.c_int64, C.POINTER(Counts)]
    lib.adps_remap_rows.argtypes = [vp, vp, C.c_int64, vp, vp, C.c_int64, vp]
    lib.adps_normals_pcg64.argtypes = [vp, vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_int64, vp,
                                       C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
    for name in EXPORTS:
        fn = getattr(lib, name)
        if name not in ("adps_abi_version", "adps_last_error"):
            fn.restype = st
    if lib.adps_abi_version() != ABI_VERSION:
        raise ImportError("libadps.so ABI version mismatch")
    _lib = lib
    return lib


class AdpsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"adps status {status}: {msg}")
        self.status = status


def check(status: int):
    """Map status codes onto the reference's exception types (include/adps.h)."""
    if status == ADPS_OK:
        return
    msg = _lib.adps_last_error().decode(errors="replace") if _lib else "?"
    from .types import DegenerateRayError
    if status in (ADPS_INVALID_ARG, ADPS_V_TOO_LARGE):
        raise ValueError(msg)
    if status == ADPS_DEGENERATE_RAY:
        raise DegenerateRayError(msg)
    raise AdpsError(status, msg)
