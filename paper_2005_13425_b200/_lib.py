"""ctypes binding of libsem.so, the sm_100a C-ABI declared in include/sem.h.

There is deliberately no CPU fallback: if the shared library is missing or
cannot be loaded, every operation raises ``SemLibraryError``.  Build it with
``python -m paper_2005_13425_b200.build`` (or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SEM_LIBRARY", os.path.join(_HERE, "libsem.so"))


class SemLibraryError(RuntimeError):
    """libsem.so is unavailable or a call into it failed."""


class sem_cg_state(ctypes.Structure):
    """Mirror of `sem_cg_state` in include/sem.h (device-resident CG scalars)."""

    _fields_ = [
        ("rtz", ctypes.c_double),
        ("rtz_old", ctypes.c_double),
        ("pap", ctypes.c_double),
        ("alpha", ctypes.c_double),
        ("beta", ctypes.c_double),
        ("tolerance", ctypes.c_double),
        ("it", ctypes.c_int32),
        ("max_iterations", ctypes.c_int32),
        ("iterations_run", ctypes.c_int32),
        ("stop", ctypes.c_int32),
        ("breakdown_it", ctypes.c_int32),
        ("x_pending", ctypes.c_int32),
        ("local_sum", ctypes.c_double),
    ]


_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f64 = ctypes.c_double
_dp = ctypes.POINTER(ctypes.c_double)

# name -> (restype, argtypes); the single source of truth for the binding and
# for the "every declared symbol is exported" test.
SIGNATURES = {
    "sem_abi_version": (ctypes.c_int, []),
    "sem_last_error": (ctypes.c_char_p, []),
    "sem_min_points": (ctypes.c_int, []),
    "sem_fallback_count": (ctypes.c_int64, []),
    "sem_max_points": (ctypes.c_int, []),
    "sem_ax": (ctypes.c_int, [_vp, _vp, _dp, _dp, _vp, _i64, _i32, _vp]),
    "sem_ax_variant": (ctypes.c_int, [_vp, _vp, _dp, _dp, _vp, _i64, _i32, _i32, _vp]),
    "sem_ax_reference": (ctypes.c_int, [_vp, _vp, _dp, _dp, _vp, _vp, _vp, _vp, _i64, _i32, _vp]),
    "sem_ax_scratch": (ctypes.c_int, [_vp, _vp, _dp, _vp, _i64, _i32, _vp]),
    "sem_ax_num_variants": (ctypes.c_int, [_i32]),
    "sem_ax_host": (ctypes.c_int, [_vp, _vp, _dp, _dp, _vp, _i64, _i32, _vp, _vp, _i64, _vp]),
    "sem_dssum_box": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp]),
    "sem_mask_box": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _vp]),
    "sem_dssum_csr": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _vp]),
    "sem_mask_array": (ctypes.c_int, [_vp, _vp, _vp, _i64, _vp]),
    "sem_consistent_box": (ctypes.c_int, [_vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "sem_apply_global": (ctypes.c_int, [_vp, _vp, _dp, _dp, _vp, _vp, _i32, _i32, _i32, _i32,
                                        _vp]),
    "sem_add2s1": (ctypes.c_int, [_vp, _vp, _f64, _i64, _vp]),
    "sem_add2s2": (ctypes.c_int, [_vp, _vp, _f64, _i64, _vp]),
    "sem_reduce_scratch_bytes": (ctypes.c_int64, []),
    "sem_glsc3": (ctypes.c_int, [_vp, _vp, _vp, _i64, _vp, _vp, _vp]),
    "sem_glsc3_box": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp]),
    "sem_cg_init": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _f64, _i32, _i32, _i32,
                                   _i32, _vp, _vp]),
    "sem_cg_run": (ctypes.c_int, [_vp, _dp, _dp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32,
                                  _i32, _i32, _vp, _vp]),
    "sem_cg_run_at": (ctypes.c_int, [_vp, _dp, _dp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32,
                                     _i32, _i32, _i32, _i32, _vp, _vp]),
    "sem_cg_finalize": (ctypes.c_int, [_vp, _vp, _vp, _i64, _vp]),
    "sem_cg_run_phases": (ctypes.c_int, [_vp, _dp, _dp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32,
                                         _i32, _i32, _i32, _vp, _dp, _vp]),
    "sem_slab_plane_top": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _vp]),
    "sem_slab_plane_bottom": (ctypes.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp]),
    "sem_dssum_slab": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32,
                                      _i32, _vp]),
    "sem_mask_slab": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp]),
    "sem_glsc3_slab": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp,
                                      _vp]),
    "sem_cg_init_slab": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _f64, _i32, _i32,
                                        _i32, _i32, _i32, _i32, _vp, _vp]),
    "sem_cg_ax_slab": (ctypes.c_int, [_vp, _vp, _vp, _vp, _dp, _dp, _vp, _i64, _i32, _vp, _vp,
                                      _vp, _vp, _i32, _vp]),
    "sem_cg_settle_slab": (ctypes.c_int, [_vp, _i64, _vp, _i32, _vp]),
    "sem_cg_update_slab": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32,
                                          _i32, _vp, _vp]),
    "sem_cg_update_slab_alpha": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32,
                                                _i32, _i32, _i32, _i32, _vp, _vp]),
    "sem_cg_finish": (ctypes.c_int, [_vp, _vp, _i32, _i32, _vp, _vp]),
    "sem_random_field": (ctypes.c_int, [_vp, _i64, ctypes.c_uint64, _vp]),
    "sem_box_geom": (ctypes.c_int, [_vp, _i64, _i32, _dp, _f64, _vp]),
    "sem_stream_copy": (ctypes.c_int, [_vp, _vp, _i64, _vp]),
    "sem_l2_props": (ctypes.c_int, [ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "sem_l2_window": (ctypes.c_int, [_vp, _i64, _f64, _i64, _vp]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load libsem.so once; raise SemLibraryError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise SemLibraryError(
            f"libsem.so not found at {LIB_PATH}; build it with "
            "`python -m paper_2005_13425_b200.build` (no CPU fallback exists)")
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:  # pragma: no cover - environment dependent
        raise SemLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.sem_abi_version() != 1:
        raise SemLibraryError("libsem ABI version mismatch")
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().sem_last_error()
        text = msg.decode() if msg else ""
        if rc == 1001:
            raise ValueError(f"{what}: {text}")
        raise SemLibraryError(f"{what} failed (code {rc}): {text}")
