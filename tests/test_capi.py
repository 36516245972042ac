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
    assert _lib.load().trim_abi_version() == 3 == _lib.ABI_VERSION


def test_struct_layouts_match_the_header(tmp_path):
    """The ctypes mirrors of trim_index_desc / trim_index_info / trim_graph_desc /
    trim_counters have the C sizes and field offsets (a C probe compiled
    against include/trim_gpu.h)."""
    import os
    import subprocess
    structs = {"trim_index_desc": _lib.TrimIndexDesc, "trim_index_info": _lib.TrimIndexInfo,
               "trim_graph_desc": _lib.TrimGraphDesc, "trim_counters": _lib.TrimCounters}
    lines = ["#include <stdio.h>", "#include <stddef.h>", f'#include "{_lib.HEADER}"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'printf("{name} sizeof %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{name} {f} %zu\\n", offsetof({name}, {f}));')
    lines.append("return 0; }")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-std=c11", "-o", str(exe), str(src)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for name, cls in structs.items():
        assert got[(name, "sizeof")] == C.sizeof(cls), name
        for f, _ in cls._fields_:
            assert got[(name, f)] == getattr(cls, f).offset, (name, f)


@pytest.mark.parametrize("kw", [dict(ndevices=2, shard_mode=1), dict(ndevices=1, shard_mode=7)])
def test_multi_device_descriptor_validation(kw):
    """ndevices > 0 without devices[] or with an unknown shard_mode is rejected
    before any device work (TRIM_EINVAL) — or TRIM_ECUDA first when there is no
    GPU at all (no CPU fallback)."""
    lib = _lib.load()
    sub = np.array([4, 4], np.uint32)
    z = np.zeros(16 * 8, np.float32)
    offs = np.array([0, 0], np.uint64)
    d = _desc(sub_dims=sub.ctypes.data, centroids=z.ctypes.data, coarse=z.ctypes.data,
              list_offsets=offs.ctypes.data, **kw)
    h = C.c_void_p()
    rc = lib.trim_index_create(C.byref(d), C.byref(h))
    assert rc in (_lib.TRIM_EINVAL, _lib.TRIM_ECUDA)


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
