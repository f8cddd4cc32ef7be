"""ctypes binding of libemm.so (include/emm.h).

The product path has no CPU fallback: if the shared library is missing the
import fails loudly.  Build it with `python -m paper_2507_10069_b200.build`.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EMM_LIB_PATH") or os.path.join(_HERE, "libemm.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not found: the B200 extension is not built "
        "(run `python -m paper_2507_10069_b200.build`); there is no CPU fallback")

lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
vp, cp = C.c_void_p, C.c_char_p
P = C.POINTER

_SIGS = {
    "emm_last_error": (cp, []),
    "emm_version": (C.c_int, []),
    # image pool
    "emm_pool_create": (C.c_int, [i64, P(vp)]),
    "emm_pool_destroy": (C.c_int, [vp]),
    "emm_pool_lookup": (C.c_int, [vp, cp, f64, P(i64)]),
    "emm_pool_insert": (C.c_int, [vp, cp, i64, f64, i64, P(i32)]),
    "emm_pool_info": (C.c_int, [vp, P(i64)]),
    "emm_pool_take_evicted": (C.c_int, [vp, C.c_char_p, i64, P(i64)]),
    # prefix tree
    "emm_tree_create": (C.c_int, [i64, P(vp)]),
    "emm_tree_destroy": (C.c_int, [vp]),
    "emm_tree_match": (C.c_int, [vp, vp, vp, i64, f64, P(i64), P(u64)]),
    "emm_tree_release": (C.c_int, [vp, u64]),
    "emm_tree_insert": (C.c_int, [vp, vp, vp, i64, f64, P(i64)]),
    "emm_tree_evict": (C.c_int, [vp, i64, f64, P(i64)]),
    "emm_tree_info": (C.c_int, [vp, P(i64)]),
    "emm_tree_eviction_log": (C.c_int, [vp, i64, i64, vp, vp, vp]),
    "emm_tree_nodes": (C.c_int, [vp, i64, i64, P(i64), P(i64), vp, vp, vp, vp, vp, vp, vp,
                                 vp]),
    "emm_tree_handle_entries": (C.c_int, [vp, u64, P(i64)]),
    # unified cache
    "emm_cache_create": (C.c_int, [i64, f64, P(vp)]),
    "emm_cache_destroy": (C.c_int, [vp]),
    "emm_cache_parts": (C.c_int, [vp, P(vp), P(vp)]),
    "emm_cache_image_lookup": (C.c_int, [vp, cp, f64, P(i64)]),
    "emm_cache_image_insert": (C.c_int, [vp, cp, i64, f64, i64, P(i32)]),
    "emm_cache_match_prefix": (C.c_int, [vp, vp, vp, i64, f64, P(i64), P(u64)]),
    "emm_cache_match_prefix_lazy": (C.c_int, [vp, vp, i64, i64, f64, P(i64), P(u64), P(i32)]),
    "emm_cache_insert_prefix": (C.c_int, [vp, vp, vp, i64, f64, P(i64)]),
    "emm_cache_release": (C.c_int, [vp, u64]),
    "emm_cache_stats": (C.c_int, [vp, P(i64)]),
    "emm_prefix_hashes_host": (C.c_int, [vp, vp, i64, vp, vp]),
    # scheduler host loop (host_sched.cpp)
    "emm_sched_set_float_sum": (C.c_int, [C.c_int]),
    "emm_estimator_create": (C.c_int, [vp, f64, f64, P(vp)]),
    "emm_estimator_destroy": (C.c_int, [vp]),
    "emm_estimator_service_seconds": (C.c_int, [vp, i64, i64, i64, P(f64)]),
    "emm_estimator_observe": (C.c_int, [vp, f64, i64, i64, i64]),
    "emm_estimator_avg_required": (C.c_int, [vp, f64, P(i64)]),
    "emm_estimator_peak_required": (C.c_int, [vp, f64, P(i64)]),
    "emm_estimator_required": (C.c_int, [vp, f64, P(i64), P(i64)]),
    "emm_estimator_len": (C.c_int, [vp, P(i64)]),
    "emm_assign_idle": (C.c_int, [vp, vp, vp, i64, i64, vp]),
    "emm_place_reservations": (C.c_int, [vp, i64, vp, i64, vp, P(i32)]),
    "emm_allocate_prefill": (C.c_int, [vp, f64, i64, vp, i64, vp, i64, vp, i64, vp, i64, i64,
                                       i64, i64, vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                       vp]),
}

_OPTIONAL = {}


def _declare(sigs, required=True):
    for name, (res, args) in sigs.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            if required:
                raise ImportError(f"libemm.so does not export {name}")
            continue
        fn.restype = res
        fn.argtypes = args


_declare(_SIGS)


class EmmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"emm error {code}: {msg}")
        self.code = code


EMM_E_RELEASE_WITHOUT_MATCH = 2


def check(code: int) -> None:
    if code != 0:
        msg = lib.emm_last_error().decode("utf-8", "replace")
        raise EmmError(code, msg)


def declare_more(sigs):
    """Register additional signatures (device entry points)."""
    _declare(sigs)


def exported_symbols() -> list[str]:
    return list(_SIGS)
