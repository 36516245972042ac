// trim_inst.cu — instantiates the filter kernels for one code length.
// Built once per TRIM_M in {16, 32, 48, 120, 0 (= runtime m and ksub)}.
#include "trim_baseline.cuh"
#include "trim_kernels.cuh"
#include "trim_launch.h"

#ifndef TRIM_M
#error "TRIM_M must be defined"
#endif
#if TRIM_M == 0
#define TRIM_KS 0
#else
#define TRIM_KS 256
#endif
#define TRIM_CAT2(a, b) a##b
#define TRIM_CAT(a, b) TRIM_CAT2(a, b)

namespace trimgpu {

namespace {
template <typename K, typename... A>
cudaError_t launch_t(K kern, dim3 grid, uint32_t threads, size_t smem, cudaStream_t st, A... args) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess)
        return e;
    kern<<<grid, threads, smem, st>>>(args...);
    return cudaGetLastError();
}
template <typename K, typename... A>
cudaError_t launch(K kern, dim3 grid, size_t smem, cudaStream_t st, A... args) {
    return launch_t(kern, grid, kThreads, smem, st, args...);
}
template <typename K, typename... A>
cudaError_t launch_knn_t(K kern, dim3 grid, size_t smem, cudaStream_t st, A... args) {
    return launch_t(kern, grid, knn_threads(TRIM_M), smem, st, args...);
}
} // namespace

cudaError_t TRIM_CAT(launch_knn_, TRIM_M)(const DevIndex& ix, const KnnParams& p, size_t smem,
                                          cudaStream_t st) {
    const uint32_t S = (p.k + 31) / 32;
    const dim3 grid(static_cast<unsigned>(p.nq));
#if TRIM_M == 0
    if (S > 8) { // k > 256: shared-memory top-k (the host routes every such call here)
        if (!p.plan)
            return launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 0, false>, grid, smem, st, ix, p);
        cudaError_t e = launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 0, true>, grid, smem, st, ix, p);
        if (e == cudaSuccess && p.probe)
            e = launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 0, true, false, true>, grid, smem, st, ix, p);
        return e;
    }
#endif
    if (p.plan) { // seeds + plan precomputed (trim_knn_setup_kernel)
        // IVF records flagged "near candidates only" go to the HARD flavour (no early-exit
        // stages); flat resume records (no probe lists) never carry the flag
        cudaError_t e = cudaSuccess;
        if (S <= 1) {
            e = launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 1, true>, grid, smem, st, ix, p);
            if (e == cudaSuccess && p.probe)
                e = launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 1, true, false, true>, grid, smem, st, ix, p);
        } else if (S <= 2) {
            e = launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 2, true>, grid, smem, st, ix, p);
            if (e == cudaSuccess && p.probe)
                e = launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 2, true, false, true>, grid, smem, st, ix, p);
        } else if (S <= 4) {
            e = launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 4, true>, grid, smem, st, ix, p);
            if (e == cudaSuccess && p.probe)
                e = launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 4, true, false, true>, grid, smem, st, ix, p);
        } else {
            e = launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 8, true>, grid, smem, st, ix, p);
            if (e == cudaSuccess && p.probe)
                e = launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 8, true, false, true>, grid, smem, st, ix, p);
        }
        return e;
    }
    if (S <= 1)
        return launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 1, false>, grid, smem, st, ix, p);
    if (S <= 2)
        return launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 2, false>, grid, smem, st, ix, p);
    if (S <= 4)
        return launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 4, false>, grid, smem, st, ix, p);
    return launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 8, false>, grid, smem, st, ix, p);
}

// segmented flat scans: the SEG instantiation (records of mode 1; the others exit at once)
cudaError_t TRIM_CAT(launch_knn_seg_, TRIM_M)(const DevIndex& ix, const KnnParams& p, size_t smem,
                                              cudaStream_t st) {
    const uint32_t S = (p.k + 31) / 32;
    const dim3 grid(static_cast<unsigned>(p.nq));
#if TRIM_M == 0
    if (S > 8)
        return launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 0, true, true>, grid, smem, st, ix, p);
#endif
    if (S <= 1)
        return launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 1, true, true>, grid, smem, st, ix, p);
    if (S <= 2)
        return launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 2, true, true>, grid, smem, st, ix, p);
    if (S <= 4)
        return launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 4, true, true>, grid, smem, st, ix, p);
    return launch_knn_t(trim_knn_kernel<TRIM_M, TRIM_KS, 8, true, true>, grid, smem, st, ix, p);
}

cudaError_t TRIM_CAT(launch_range_, TRIM_M)(const DevIndex& ix, const RangeParams& p, dim3 grid,
                                            size_t smem, cudaStream_t st) {
    return launch(trim_range_kernel<TRIM_M, TRIM_KS>, grid, smem, st, ix, p);
}

cudaError_t TRIM_CAT(launch_range_flat_, TRIM_M)(const DevIndex& ix, const RangeParams& p, dim3 grid,
                                                 size_t smem, uint32_t qt, cudaStream_t st) {
    return launch_t(trim_range_flat_kernel<TRIM_M, TRIM_KS>, grid, kFlatThreads, smem, st, ix, p, qt);
}

cudaError_t TRIM_CAT(launch_bl_est_, TRIM_M)(const DevIndex& ix, const BlParams& p, dim3 grid,
                                             size_t smem, cudaStream_t st) {
    return launch(trim_bl_est_kernel<TRIM_M, TRIM_KS>, grid, smem, st, ix, p);
}

} // namespace trimgpu
