// trim_graph.cu — instantiates trim_graph_kernel (trim_graph.cuh) for the
// candidate-queue capacities 32*S, S in {1, 2, 4, 8, 16, 32} (ef <= 1024).
#define TRIM_M 1000 // trim_kernels.cuh's non-template kernels are compiled in trim_capi.cu
#include "trim_graph.cuh"
#include "trim_launch.h"

namespace trimgpu {

cudaError_t launch_graph(const GraphDev& g, const GraphParams& p, uint32_t S, size_t smem,
                         cudaStream_t st) {
    void (*kern)(GraphDev, GraphParams) = nullptr;
    switch (S) {
    case 1: kern = trim_graph_kernel<1>; break;
    case 2: kern = trim_graph_kernel<2>; break;
    case 4: kern = trim_graph_kernel<4>; break;
    case 8: kern = trim_graph_kernel<8>; break;
    case 16: kern = trim_graph_kernel<16>; break;
    case 32: kern = trim_graph_kernel<32>; break;
    default: return cudaErrorInvalidValue;
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess)
        return e;
    kern<<<static_cast<unsigned>(p.nq), kGraphThreads, smem, st>>>(g, p);
    return cudaGetLastError();
}

} // namespace trimgpu
