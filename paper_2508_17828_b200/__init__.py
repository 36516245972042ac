"""B200-native TRIM candidate filter (arXiv 2508.17828).

The hot path of the reference (proj/include/trimsearch/ivf/ivf.hpp:193-347 —
per-query PQ LUT, ADC, γ-relaxed triangle bound, prune, exact L2 of the
survivors, top-k / range merge) as hand-written sm_100a CUDA behind the C ABI
in include/trim_gpu.h. See DESIGN.md.
"""
from .ivf import (  # noqa: F401
    CudaError,
    DataError,
    GpuIvfIndex,
    InvalidArgument,
    IvfArrays,
    IvfResult,
    PruningProfile,
    SearchCounters,
    build_distance_table,
    probe_order,
    search_baseline_ivfpq,
    search_baseline_ivfpq_batch,
    search_trim_ivf_knn,
    search_trim_ivf_knn_batch,
    search_trim_ivf_knn_device,
    search_trim_ivf_range,
    search_trim_ivf_range_batch,
    search_trim_ivf_range_device,
)
from . import formats  # noqa: F401  (reference on-disk formats)
from . import graph  # noqa: F401  (TRIM filter over an HNSW graph)

__version__ = "0.1.0"
