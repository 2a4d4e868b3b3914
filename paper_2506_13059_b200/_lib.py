"""ctypes binding of libmpattn.so (the C ABI declared in include/mpattn.h).

The product path has no fallback: if the library is missing or a call fails, a Python
exception is raised (`MpattnError`, or the reference's own exception types where the
reference raises them).
"""

from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MPATTN_LIB") or os.path.join(_HERE, "libmpattn.so")  # override: experiments only

MPA_F32, MPA_BF16, MPA_F64 = 0, 1, 2
MPA_ERR_ARG, MPA_ERR_UNSUPPORTED = 1001, 1002

_vp, _i32, _i64, _f32, _f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_float, C.c_double


class MpattnError(RuntimeError):
    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} failed ({code}): {msg}")
        self.code = code


class MpaCache(C.Structure):
    _fields_ = [("k_rot", _vp), ("k_raw", _vp), ("v", _vp), ("dtype", _i32), ("n_ledgers", _i32),
                ("tcap", _i32), ("head_dim", _i32), ("block_table", _vp), ("page_size", _i32),
                ("pages_per_seq", _i32), ("n_pages", _i32), ("n_kv_heads", _i32)]


class MpaLevel(C.Structure):
    _fields_ = [("kc", _vp), ("vc", _vp), ("size", _vp), ("count", _vp), ("off", _vp), ("idx", _vp),
                ("cap", _i32), ("idx_cap", _i32), ("dtype", _i32), ("n_ledgers", _i32)]


class MpaKm(C.Structure):
    _fields_ = [("n_prob", _i32), ("d", _i32), ("pts", _vp), ("pts_dtype", _i32), ("tcap", _i32), ("pts64", _vp),
                ("wts", _vp), ("rows64_cap", _i32), ("n_max", _i32), ("k_max", _i32), ("min_iters", _i32),
                ("prob_l", _vp), ("prob_start", _vp), ("prob_n", _vp), ("prob_k", _vp), ("pt_off", _vp),
                ("c_off", _vp), ("assign", _vp), ("prev", _vp), ("p2", _vp), ("cent", _vp), ("c2", _vp),
                ("count", _vp), ("order", _vp), ("cstart", _vp), ("state", _vp), ("flag", _vp),
                ("pts_rows", _i64), ("sum_n", _i32), ("sum_k", _i32), ("tc_ws", _vp), ("tc_ws_bytes", _i64),
                ("dirty", _vp)]


_KM = C.POINTER(MpaKm)

_SIGS = {
    "mpa_kv_write": [C.POINTER(MpaCache), _vp, _vp, _vp, C.c_int, _vp, _vp],
    "mpa_stage3": [_vp, _vp, C.c_longlong, _vp, _vp, C.c_longlong, _vp, _vp, C.c_longlong, _vp],
    "mpa_decode_step_rebind": [_vp, _vp, _vp, _vp, _vp],
    "mpa_step_host": [_vp, _vp, _vp, C.c_longlong, _vp, C.c_longlong, _vp, C.c_longlong, _vp, _vp, C.c_longlong,
                      _vp],
    "mpa_kv_append": [C.POINTER(MpaCache), _vp, _vp, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp],
    "mpa_rotate_queries": [_vp, C.c_int, C.c_int, C.c_int, _vp, C.c_int, _vp, _f32, _vp, _vp, _vp],
    "mpa_centroid_logits": [_vp, C.c_int, C.c_int, C.c_int, C.POINTER(MpaLevel), _vp, _vp, C.c_int, _vp, _vp,
                            _vp, C.c_int, _vp, C.c_int, _vp, _vp, _vp],
    "mpa_select": [_vp, C.c_int, _vp, _vp, C.c_int, _vp, C.c_int, _vp, _vp, _vp, _vp, C.c_int, _vp, C.c_int,
                   _vp, _vp, _vp, _vp, C.c_int, _vp],
    "mpa_select_worklist": [C.POINTER(MpaLevel), C.POINTER(MpaLevel), C.c_int, _vp, _vp, _vp, _vp, C.c_int, _vp, _vp,
                            _vp, _vp, _vp, _vp, _vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, C.c_int, _vp, _vp,
                            C.c_int, _vp, C.c_int, _vp],
    "mpa_decode_step_fits": [C.c_int, C.c_int, C.c_int],
    "mpa_decode_step": [_vp, _vp, _vp, C.POINTER(MpaCache), _vp, _vp, C.c_int, C.c_int, C.POINTER(MpaLevel), _vp,
                        _vp, _vp, _vp, _vp, _vp, C.c_int, _vp, _vp, _vp, C.c_int, _vp, C.c_int, _vp, _vp, C.c_int,
                        _vp],
    "mpa_ref_rotate": [_vp, _vp, C.c_int, C.c_int, _vp, _vp, _vp],
    "mpa_ref_logits": [_vp, _vp, C.c_int, C.c_int, C.c_int, _vp, _vp],
    "mpa_ref_partial": [_vp, _vp, _vp, C.c_int, C.c_int, _vp, _vp, _vp],
    "mpa_ref_group_scores": [_vp, _vp, C.c_int, C.c_int, _vp, _vp, _vp],
    "mpa_ref_nearest": [_vp, _vp, C.c_int, C.c_int, C.c_int, _vp, _vp],
    "mpa_ref_seg_stats": [_vp, _vp, _vp, _vp, C.c_int, C.c_int, _vp, _vp, _vp, _vp],
    "mpa_hier_candidates": [C.POINTER(MpaLevel), _vp, C.c_int, _vp, _vp, C.c_int, _vp],
    "mpa_head_norms": [_vp, C.c_int, _vp, C.c_int, C.c_int, _vp, _vp],
    "mpa_merge_norms": [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp],
    "mpa_select_worklist_sharded": [C.POINTER(MpaLevel), C.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, C.c_int,
                                    C.c_int, _vp, _vp, _vp, C.c_int, _vp, _vp, C.c_int, _vp, C.c_int, _vp, _vp,
                                    _vp, _vp, C.c_int, _vp, _vp],
    "mpa_global_cut": [_vp, _vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp],
    "mpa_sparse_decode_partials": [C.POINTER(MpaCache), _vp, C.c_int, C.c_int, _vp, _vp, C.c_int, _vp, _vp, _vp,
                                   C.c_int, _vp, C.c_int, _vp, C.c_int, C.c_int, _vp, C.c_size_t, _vp, _vp],
    "mpa_merge_rank_partials": [_vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp],
    "mpa_km_lloyd": [_KM, C.POINTER(_i32), _vp],
    "mpa_km_means": [_KM, _vp],
    "mpa_km_count_nonempty": [_KM, _vp, _vp],
    "mpa_km_write_level": [_KM, C.POINTER(MpaCache), _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _i32, _i32, _vp],
    "mpa_km_assign_from_level": [_KM, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp],
    "mpa_km_seq_assign": [_KM, _vp, C.c_int, _vp, _vp],
    "mpa_sparse_decode": [C.POINTER(MpaCache), _vp, C.c_int, C.c_int, _vp, _vp, C.c_int, _vp, _vp, _vp,
                          C.c_int, _vp, C.c_int, _vp, C.c_int, C.c_int, _vp, C.c_size_t, _vp, _vp],
}

# symbols that include/mpattn.h declares (checked by tests/test_abi.py)
EXPORTED = ["mpa_last_error", "mpa_version", "mpa_sparse_decode_workspace", "mpa_km_tc_workspace", *_SIGS]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2506_13059_b200.build` "
                          "(or __graft_entry__.build())")
    lib = C.CDLL(LIB_PATH)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    lib.mpa_km_tc_workspace.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int]
    lib.mpa_km_tc_workspace.restype = C.c_size_t
    lib.mpa_sparse_decode_workspace.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
    lib.mpa_sparse_decode_workspace.restype = C.c_size_t
    lib.mpa_last_error.restype = C.c_char_p
    lib.mpa_version.restype = C.c_char_p
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


def call(name: str, *args) -> None:
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        raise MpattnError(name, rc, lib().mpa_last_error().decode())


def ptr(t) -> int | None:
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return MPA_F32
    if dt == torch.bfloat16:
        return MPA_BF16
    raise ValueError(f"unsupported cache dtype {dt} (float32 or bfloat16)")
