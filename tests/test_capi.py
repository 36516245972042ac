"""CPU: the C-ABI library loads, exports every symbol include/trim_gpu.h
declares, and rejects bad arguments with the reference's error classes
without touching a GPU. No compute calls (there is no GPU here)."""
import ctypes as C
import re

import numpy as np
import pytest

from paper_2508_17828_b200 import _lib


def declared_functions():
    src = open(_lib.HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(trim_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_expected_surface():
    fns = declared_functions()
    for f in ("trim_index_create", "trim_search_knn", "trim_search_range",
              "trim_search_baseline_ivfpq", "trim_merge_topk_device", "trim_last_error"):
        assert f in fns


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing
    # and the binding covers them all
    assert set(declared_functions()) <= set(_lib.SIGNATURES)


def test_abi_version():
    assert _lib.load().trim_abi_version() == 2


def _desc(**kw):
    d = _lib.TrimIndexDesc()
    d.dim, d.m, d.ksub, d.nlist, d.code_stride = 8, 2, 16, 1, 2
    for k, v in kw.items():
        setattr(d, k, v)
    return d


@pytest.mark.parametrize("kw,exc", [
    (dict(dim=0), _lib.DataError),
    (dict(m=0), _lib.InvalidArgument),
    (dict(m=9), _lib.InvalidArgument),
    (dict(ksub=300), _lib.InvalidArgument),
    (dict(nlist=0), _lib.InvalidArgument),
    (dict(code_stride=1), _lib.InvalidArgument),
])
def test_index_create_validation(kw, exc):
    lib = _lib.load()
    d = _desc(**kw)
    h = C.c_void_p()
    with pytest.raises(exc):
        _lib.check(lib.trim_index_create(C.byref(d), C.byref(h)))


def test_no_cpu_fallback_without_gpu():
    """With arrays present but no device, creation fails loudly (TRIM_ECUDA)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = _lib.load()
    sub = np.array([4, 4], np.uint32)
    cent = np.zeros(16 * 8, np.float32)
    coarse = np.zeros(8, np.float32)
    offs = np.array([0, 0], np.uint64)
    d = _desc(sub_dims=sub.ctypes.data, centroids=cent.ctypes.data, coarse=coarse.ctypes.data,
              list_offsets=offs.ctypes.data)
    h = C.c_void_p()
    with pytest.raises(_lib.CudaError):
        _lib.check(lib.trim_index_create(C.byref(d), C.byref(h)))


def test_search_argument_errors_before_device():
    lib = _lib.load()
    q = np.zeros(8, np.float32)
    out = np.zeros(16, np.uint32)
    # null index
    with pytest.raises(_lib.InvalidArgument):
        _lib.check(lib.trim_search_knn(None, q.ctypes.data, 1, 5, 1, 0.0, out.ctypes.data,
                                       out.ctypes.data, None))
    with pytest.raises(_lib.InvalidArgument):
        _lib.check(lib.trim_merge_topk_device(None, None, 0, 1, 1, None, None, 0, None))
