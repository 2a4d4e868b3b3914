"""CPU checks of the C-ABI boundary: libmpattn.so loads, exports every function that
include/mpattn.h declares, and reports argument errors through mpa_last_error without a GPU."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mpattn.h")
LIB = os.path.join(ROOT, "paper_2506_13059_b200", "libmpattn.so")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mpa_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2506_13059_b200.build import build
        build(verbose=False)
    return ctypes.CDLL(LIB)


def test_header_declares_entry_points():
    names = declared()
    for must in ("mpa_kv_write", "mpa_rotate_queries", "mpa_centroid_logits", "mpa_select",
                 "mpa_sparse_decode", "mpa_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_2506_13059_b200 import _lib
    assert sorted(_lib.EXPORTED) == declared()


def test_argument_errors_without_gpu(lib):
    lib.mpa_last_error.restype = ctypes.c_char_p
    lib.mpa_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.mpa_version()
    rc = lib.mpa_select(None, 4, None, None, 0, None, 0, None, None, None, None, 0, None, 1, None, None, None,
                        None, 0, None)
    assert rc == 1001
    assert b"null argument" in lib.mpa_last_error()
    rc = lib.mpa_sparse_decode(None, None, 8, 4, None, None, 0, None, None, None, 0, None, 0, None, 0, 1,
                               None, ctypes.c_size_t(0), None, None)
    assert rc == 1001


def test_new_entry_points_reject_bad_arguments(lib):
    lib.mpa_last_error.restype = ctypes.c_char_p
    ll = ctypes.c_longlong
    # step-input staging: sizes must be multiples of 4 floats, buffers 16-byte aligned
    rc = lib.mpa_stage3(ctypes.c_void_p(64), ctypes.c_void_p(64), ll(6), None, None, ll(0), None, None, ll(0), None)
    assert rc == 1001 and b"multiple of 4" in lib.mpa_last_error()
    rc = lib.mpa_stage3(ctypes.c_void_p(68), ctypes.c_void_p(64), ll(8), None, None, ll(0), None, None, ll(0), None)
    assert rc == 1001 and b"aligned" in lib.mpa_last_error()
    # logits: neither q_lk nor (q_raw, cs_lk)
    rc = lib.mpa_centroid_logits(None, 8, 4, 128, None, None, None, 0, None, None, None, 0, None, 0, None, None, None)
    assert rc == 1001 and b"null argument" in lib.mpa_last_error()


def test_paged_cache_geometry_is_validated(lib):
    # a paged mpa_cache is checked before any launch: page size a power of two, enough pages per
    # sequence for tcap, kv-heads dividing the ledgers
    from paper_2506_13059_b200._lib import MpaCache

    lib.mpa_last_error.restype = ctypes.c_char_p
    dummy = ctypes.c_void_p(256)
    bt = ctypes.c_void_p(512)

    def cache(page_size, pages_per_seq, n_kv_heads=2):
        return MpaCache(dummy, dummy, dummy, 2, 4, 100, 128, bt, page_size, pages_per_seq, 8, n_kv_heads)

    k = ctypes.c_void_p(1024)
    for c, msg in ((cache(24, 8), b"power of two"), (cache(16, 2), b"tcap"), (cache(16, 8, 3), b"geometry")):
        rc = lib.mpa_kv_write(ctypes.byref(c), k, k, k, 1, k, None)
        assert rc == 1001 and msg in lib.mpa_last_error(), lib.mpa_last_error()
