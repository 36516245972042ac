// trim_launch.h — per-(m, ksub) kernel launchers. Each specialization lives in
// its own translation unit (trim_inst.cu built once per M by the Makefile) so
// the template instantiations compile in parallel.
#pragma once

#include <cuda_runtime.h>

#include "trim_common.cuh"

namespace trimgpu {

struct KnnParams;
struct RangeParams;
struct BlParams;
struct GraphDev;
struct GraphParams;

// trim_graph.cu: trim_graph_kernel<S> (candidate queue capacity 32*S).
cudaError_t launch_graph(const GraphDev& g, const GraphParams& p, uint32_t S, size_t smem,
                         cudaStream_t st);

#define TRIM_DECLARE_LAUNCHERS(MV)                                                                \
    cudaError_t launch_knn_##MV(const DevIndex& ix, const KnnParams& p, size_t smem,             \
                                cudaStream_t st);                                                 \
    cudaError_t launch_knn_seg_##MV(const DevIndex& ix, const KnnParams& p, size_t smem,         \
                                    cudaStream_t st);                                             \
    cudaError_t launch_range_##MV(const DevIndex& ix, const RangeParams& p, dim3 grid, size_t smem,\
                                  cudaStream_t st);                                               \
    cudaError_t launch_range_flat_##MV(const DevIndex& ix, const RangeParams& p, dim3 grid,        \
                                       size_t smem, uint32_t qt, cudaStream_t st);                 \
    cudaError_t launch_bl_est_##MV(const DevIndex& ix, const BlParams& p, dim3 grid, size_t smem,  \
                                   cudaStream_t st);

TRIM_DECLARE_LAUNCHERS(16)
TRIM_DECLARE_LAUNCHERS(32)
TRIM_DECLARE_LAUNCHERS(48)
TRIM_DECLARE_LAUNCHERS(120)
TRIM_DECLARE_LAUNCHERS(0)

} // namespace trimgpu
