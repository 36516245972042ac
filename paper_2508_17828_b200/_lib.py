"""ctypes binding of libtrim_b200.so (the C ABI in include/trim_gpu.h).

The library is built in-tree by ``__graft_entry__.build()`` /
``make -C paper_2508_17828_b200/csrc``. There is no Python or CPU fallback:
if the library is missing this module raises ImportError, and every search
returns TRIM_ECUDA when no GPU is present.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# TRIM_B200_LIB selects another build of the library (the perf-probe build
# libtrim_b200_tl.so, profiles/knn_timeline.py); default: the production build.
LIB_PATH = os.environ.get("TRIM_B200_LIB") or os.path.join(HERE, "libtrim_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "trim_gpu.h")

TRIM_OK, TRIM_EINVAL, TRIM_EDATA, TRIM_ECUDA, TRIM_ENCCL, TRIM_ENOMEM = range(6)
TRIM_MEM_HOST, TRIM_MEM_DEVICE = 0, 1
TRIM_SHARD_SINGLE, TRIM_SHARD_ID, TRIM_SHARD_REPLICAS = 0, 1, 2
ABI_VERSION = 3

_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_f32p = C.POINTER(C.c_float)


class TrimCounters(C.Structure):
    _fields_ = [("dc", C.c_uint64), ("edc", C.c_uint64), ("pruned", C.c_uint64),
                ("evaluated", C.c_uint64), ("hops", C.c_uint64), ("coarse_dc", C.c_uint64)]


class TrimIndexDesc(C.Structure):
    _fields_ = [
        ("dim", C.c_uint32), ("m", C.c_uint32), ("ksub", C.c_uint32),
        ("sub_dims", C.c_void_p), ("centroids", C.c_void_p),
        ("nlist", C.c_uint32), ("coarse", C.c_void_p),
        ("list_offsets", C.c_void_p), ("list_ids", C.c_void_p), ("list_codes", C.c_void_p),
        ("code_stride", C.c_uint32), ("list_lx", C.c_void_p),
        ("n", C.c_uint64), ("vectors", C.c_void_p),
        ("id_base", C.c_uint64), ("device", C.c_int), ("memory", C.c_int),
        # ABI 3: multi-device layout (trim_shard_mode)
        ("devices", C.c_void_p), ("ndevices", C.c_uint32), ("shard_mode", C.c_int),
    ]


class TrimIndexInfo(C.Structure):
    _fields_ = [("dim", C.c_uint32), ("m", C.c_uint32), ("ksub", C.c_uint32),
                ("nlist", C.c_uint32), ("n", C.c_uint64), ("total_entries", C.c_uint64),
                ("id_base", C.c_uint64), ("max_list_size", C.c_uint64),
                ("device_bytes", C.c_uint64), ("device", C.c_int), ("range_query_tile", C.c_uint32),
                ("ndevices", C.c_uint32), ("shard_mode", C.c_uint32), ("nccl", C.c_uint32)]


class TrimGraphDesc(C.Structure):
    _fields_ = [
        ("n", C.c_uint64), ("dim", C.c_uint32), ("m", C.c_uint32), ("ksub", C.c_uint32),
        ("sub_dims", C.c_void_p), ("centroids", C.c_void_p), ("codes", C.c_void_p),
        ("code_stride", C.c_uint32), ("lx", C.c_void_p), ("vectors", C.c_void_p),
        ("levels", C.c_uint32), ("entry", C.c_uint32), ("offsets", C.c_void_p),
        ("nbr_base", C.c_void_p), ("nbrs", C.c_void_p), ("total_nbrs", C.c_uint64),
        ("device", C.c_int), ("memory", C.c_int),
    ]


# name -> (restype, argtypes); must cover every function include/trim_gpu.h declares
SIGNATURES = {
    "trim_last_error": (C.c_char_p, []),
    "trim_abi_version": (C.c_int, []),
    "trim_index_create": (C.c_int, [C.POINTER(TrimIndexDesc), C.POINTER(C.c_void_p)]),
    "trim_index_destroy": (C.c_int, [C.c_void_p]),
    "trim_index_get_info": (C.c_int, [C.c_void_p, C.POINTER(TrimIndexInfo)]),
    "trim_index_skip_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.c_int]),
    "trim_probe_launches": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_uint32)]),
    "trim_search_knn": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32,
                                  C.c_float, C.c_void_p, C.c_void_p, C.c_void_p]),
    "trim_search_range": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint32,
                                    C.c_float, C.c_void_p, C.POINTER(_u32p), C.POINTER(_f32p),
                                    C.c_void_p]),
    "trim_search_baseline_ivfpq": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32,
                                             C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p,
                                             C.c_void_p]),
    "trim_search_knn_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32,
                                         C.c_uint32, C.c_float, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p]),
    "trim_probe_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p,
                                    C.c_void_p]),
    "trim_search_range_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint32,
                                            C.c_float, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_void_p]),
    "trim_ground_truth_knn": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p]),
    "trim_search_knn_preassigned_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32,
                                                     C.c_void_p, C.c_uint32, C.c_float, C.c_void_p,
                                                     C.c_void_p, C.c_void_p, C.c_void_p,
                                                     C.c_void_p]),
    "trim_build_lut": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "trim_probe": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p]),
    "trim_merge_topk_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64,
                                         C.c_uint32, C.c_void_p, C.c_void_p, C.c_int,
                                         C.c_void_p]),
    "trim_free": (None, [C.c_void_p]),
    # TRIM filter over an HNSW graph
    "trim_graph_create": (C.c_int, [C.POINTER(TrimGraphDesc), C.POINTER(C.c_void_p)]),
    "trim_graph_destroy": (C.c_int, [C.c_void_p]),
    "trim_graph_search_knn": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32,
                                        C.c_float, C.c_void_p, C.c_void_p, C.c_void_p]),
    "trim_graph_search_knn_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32,
                                               C.c_float, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "trim_graph_search_range": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint32,
                                          C.c_float, C.c_void_p, C.POINTER(_u32p), C.POINTER(_f32p),
                                          C.c_void_p]),
    # device-side index build
    "trim_synth_normal_device": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_void_p, C.c_int,
                                           C.c_void_p]),
    "trim_synth_blobs_device": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64,
                                          C.c_float, C.c_uint64, C.c_void_p, C.c_int, C.c_void_p]),
    "trim_synth_uniform_device": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_int,
                                            C.c_void_p, C.c_int, C.c_void_p]),
    "trim_sample_rows": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p]),
    "trim_assign_device": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p, C.c_uint32,
                                     C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "trim_kmeans_device": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                     C.c_uint64, C.c_void_p, C.c_int]),
    "trim_pq_train_device": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                       C.c_uint32, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p,
                                       C.c_int]),
    "trim_pq_encode_device": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p,
                                        C.c_int, C.c_void_p]),
    "trim_ivf_lists_device": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p,
                                        C.c_int, C.c_void_p]),
}


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference (TRIM_EINVAL)."""


class DataError(RuntimeError):
    """trimsearch::DataError (core/io_util.hpp:13-16) (TRIM_EDATA)."""


class CudaError(RuntimeError):
    """CUDA failure or no device (TRIM_ECUDA). There is no CPU fallback."""


_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the TRIM GPU path has no CPU fallback)")
    lib = C.CDLL(path)
    if lib.trim_abi_version() != ABI_VERSION:
        raise ImportError(f"{path}: ABI {lib.trim_abi_version()}, this binding speaks {ABI_VERSION}: rebuild it")
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc == TRIM_OK:
        return
    msg = load().trim_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what and not msg.startswith(what) else msg
    if rc == TRIM_EINVAL:
        raise InvalidArgument(text)
    if rc == TRIM_EDATA:
        raise DataError(text)
    if rc == TRIM_ECUDA:
        raise CudaError(text)
    if rc == TRIM_ENOMEM:
        raise MemoryError(text)
    raise RuntimeError(f"trim rc={rc}: {text}")
