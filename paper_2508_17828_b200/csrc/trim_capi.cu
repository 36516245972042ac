// trim_capi.cu — host implementation of include/trim_gpu.h.
//
// Owns the device copy of the index, per-call streams and stream-ordered
// workspaces, kernel dispatch, and the reference's error semantics
// (ivf/ivf.hpp:195-198, 246-249, 289-290, 311-314). There is no CPU path:
// every search runs the sm_100a kernels in trim_kernels.cuh.
#include <cub/device/device_segmented_sort.cuh>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/trim_gpu.h"
#include "trim_baseline.cuh"
#include "trim_graph.cuh"
#include "trim_kernels.cuh"
#include "trim_launch.h"

using namespace trimgpu;

#include "trim_host.h"

using namespace trimhost;

namespace trimhost {

int check_device_present() {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return set_err(TRIM_ECUDA, "no CUDA device available (%s); the TRIM GPU path has no CPU "
                                   "fallback",
                       cudaGetErrorString(e));
    return TRIM_OK;
}

// ---------------------------------------------------------------- dispatch
// Specialised instantiations for the configs' code lengths (m = 16, 32, 48,
// 120 with 256 centroids); anything else runs the runtime-(m, ksub) kernel.
#define TRIM_DISPATCH(NAME, ...)                                            \
    do {                                                                   \
        cudaError_t _r;                                                    \
        if (ix.ksub == 256 && ix.m == 16)                                  \
            _r = NAME##16(__VA_ARGS__);                                    \
        else if (ix.ksub == 256 && ix.m == 32)                             \
            _r = NAME##32(__VA_ARGS__);                                    \
        else if (ix.ksub == 256 && ix.m == 48)                             \
            _r = NAME##48(__VA_ARGS__);                                    \
        else if (ix.ksub == 256 && ix.m == 120)                            \
            _r = NAME##120(__VA_ARGS__);                                   \
        else                                                               \
            _r = NAME##0(__VA_ARGS__);                                     \
        CK(_r);                                                            \
    } while (0)

void launch_knn(const DevIndex& ix, const KnnParams& p, size_t smem, cudaStream_t st) {
    if (p.k > 256) { // the shared-memory top-k is instantiated in the runtime-(m, ksub) kernel only
        CK(launch_knn_0(ix, p, smem, st));
        return;
    }
    TRIM_DISPATCH(launch_knn_, ix, p, smem, st);
}

void launch_knn_seg(const DevIndex& ix, const KnnParams& p, size_t smem, cudaStream_t st) {
    if (p.k > 256) {
        CK(launch_knn_seg_0(ix, p, smem, st));
        return;
    }
    TRIM_DISPATCH(launch_knn_seg_, ix, p, smem, st);
}

void launch_range(const DevIndex& ix, const RangeParams& p, dim3 grid, size_t smem,
                  cudaStream_t st) {
    TRIM_DISPATCH(launch_range_, ix, p, grid, smem, st);
}

void launch_range_flat(const DevIndex& ix, const RangeParams& p, dim3 grid, size_t smem, uint32_t qt,
                       cudaStream_t st) {
    TRIM_DISPATCH(launch_range_flat_, ix, p, grid, smem, qt, st);
}

void launch_bl_est(const DevIndex& ix, const BlParams& p, dim3 grid, size_t smem,
                   cudaStream_t st) {
    TRIM_DISPATCH(launch_bl_est_, ix, p, grid, smem, st);
}

constexpr size_t kSmemLimit = 227 * 1024;

// 1 - gamma rounded up to a float (the stage check needs an upper bound on
// (1 - gamma) * glx).
float omg_round_up(float gamma) {
    const double exact = 1.0 - static_cast<double>(gamma);
    float f = static_cast<float>(exact);
    if (static_cast<double>(f) < exact)
        f = std::nextafter(f, 2.0f);
    return f;
}

// 1 - gamma rounded down.
float omg_round_down(float gamma) {
    const double exact = 1.0 - static_cast<double>(gamma);
    float f = static_cast<float>(exact);
    if (static_cast<double>(f) > exact)
        f = std::nextafter(f, -2.0f);
    return f;
}

// Test/measurement knobs, read per call (results and counters are identical
// for every setting):
//   TRIM_LIST_SKIP=0     disables the kNN list-level bound (A/B timing);
//   TRIM_EPS_SCALE=x>=1  widens the any-order ADC error interval x-fold, so the
//                        exact (reference-order) resolution paths run often.
//   TRIM_KNN_SETUP=0     seeds + plan inside trim_knn_kernel instead of trim_knn_setup_kernel.
bool knn_setup_enabled() {
    const char* e = std::getenv("TRIM_KNN_SETUP");
    return !(e && e[0] == '0');
}
bool list_skip_enabled() {
    const char* e = std::getenv("TRIM_LIST_SKIP");
    return !(e && e[0] == '0');
}
float filter_eps(uint32_t m) {
    float eps = adc_rel_eps(m);
    if (const char* e = std::getenv("TRIM_EPS_SCALE")) {
        const double x = std::atof(e);
        if (x > 1.0 && x * eps < 0.25)
            eps = static_cast<float>(x * eps);
    }
    return eps;
}

// The kernel specialisation (m template value) launch_* will pick.
int dispatch_m(const DevIndex& ix) {
    if (ix.ksub == 256 && (ix.m == 16 || ix.m == 32 || ix.m == 48 || ix.m == 120))
        return static_cast<int>(ix.m);
    return 0;
}

// Probe lists for a query batch (d_q rows padded to dim_stride). Returns
// the effective per-query probe count; d_probe is null when nlist == 1.
// probe_order for a batch into d_out (nq*np): the tiled kernel when np and the
// distance table fit its shared-memory plan, else the one-query bitonic kernel.
// TRIM_PROBE_MMA=0 forces the SIMT probe kernels (A/B and parity tests).
// TRIM_RANGE_TILED=0 forces the one-query range kernel for flat indexes.
bool probe_mma_enabled_range() {
    const char* e = std::getenv("TRIM_RANGE_TILED");
    return !(e && e[0] == '0');
}

bool probe_mma_enabled() {
    const char* e = std::getenv("TRIM_PROBE_MMA");
    return !(e && e[0] == '0');
}

bool probe_uses_mma(const trim_index* ix, uint32_t np) {
    const DevIndex& v = ix->dev;
    return ix->coarse_t && np <= kProbeMaxNp && v.nlist >= 256 &&
           probe_select_smem(v.nlist, v.dim_stride) <= kSmemLimit && probe_mma_enabled();
}

void launch_probe(const trim_index* ix, const float* d_q, uint64_t nq, uint32_t np, uint32_t* d_out,
                  cudaStream_t st) {
    const DevIndex& v = ix->dev;
    const size_t ssmem = probe_select_smem(v.nlist, v.dim_stride);
    if (probe_uses_mma(ix, np)) {
        const uint32_t K = mma_k(v.dim);
        const uint32_t ntiles = (v.nlist + kMmaN - 1) / kMmaN;
        const size_t ld = mma_ld(v.nlist);
        DevBuf approx(sizeof(float) * nq * ld, st);
        const size_t smem = probe_mma_smem(K);
        CK(cudaFuncSetAttribute(trim_probe_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
        const dim3 grid(static_cast<unsigned>((nq + kMmaM - 1) / kMmaM), (ntiles + kMmaTilesPerCta - 1) / kMmaTilesPerCta);
        trim_probe_mma_kernel<<<grid, kMmaThreads, smem, st>>>(d_q, nq, v.dim_stride, K, ix->coarse_t, ix->cn2,
                                                                v.nlist, approx.as<float>());
        CK(cudaGetLastError());
        CK(cudaFuncSetAttribute(trim_probe_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(ssmem)));
        trim_probe_select_kernel<<<static_cast<unsigned>(nq), kPSelThreads, ssmem, st>>>(
            v, d_q, nq, np, approx.as<float>(), ix->cn2, ix->cn, d_out);
        CK(cudaGetLastError());
        return;
    }
    if (np <= kProbeMaxNp) {
        for (uint32_t tile = 128; tile >= 32; tile >>= 1) {
            const size_t smem = probe_tiled_smem(v.nlist, v.dim_stride, tile);
            if (smem <= kSmemLimit) {
                CK(cudaFuncSetAttribute(trim_probe_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
                const unsigned grid = static_cast<unsigned>((nq + kProbeQ - 1) / kProbeQ);
                trim_probe_tiled_kernel<<<grid, kThreads, smem, st>>>(v, d_q, nq, np, tile, d_out);
                CK(cudaGetLastError());
                return;
            }
        }
    }
    const uint32_t nl2 = pow2_at_least(v.nlist);
    const size_t smem = sizeof(float) * v.dim_stride + sizeof(uint64_t) * nl2;
    CK(cudaFuncSetAttribute(trim_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(smem)));
    trim_probe_kernel<<<static_cast<unsigned>(nq), kThreads, smem, st>>>(v, d_q, nq, np, nl2, d_out);
    CK(cudaGetLastError());
}

uint32_t run_probe(const trim_index* ix, const float* d_q, uint64_t nq, uint32_t nprobe,
                   DevBuf& d_probe, cudaStream_t st) {
    const uint32_t np = std::min(nprobe, ix->dev.nlist);
    if (ix->dev.nlist == 1 || np == 0 || nq == 0)
        return np;
    d_probe = DevBuf(sizeof(uint32_t) * nq * np, st);
    launch_probe(ix, d_q, nq, np, d_probe.as<uint32_t>(), st);
    return np;
}

// Copy nq query rows (dim floats each, host or device) into a padded device
// buffer of dim_stride floats per row.
DevBuf upload_queries(const trim_index* ix, const float* q, uint64_t nq, cudaMemcpyKind kind,
                      cudaStream_t st) {
    const uint32_t dim = ix->dev.dim, ds = ix->dev.dim_stride;
    DevBuf d(sizeof(float) * nq * ds, st);
    if (nq == 0)
        return d;
    if (ds != dim) {
        CK(cudaMemsetAsync(d.p, 0, sizeof(float) * nq * ds, st));
        CK(cudaMemcpy2DAsync(d.p, sizeof(float) * ds, q, sizeof(float) * dim, sizeof(float) * dim,
                             nq, kind, st));
    } else {
        CK(cudaMemcpyAsync(d.p, q, sizeof(float) * nq * dim, kind, st));
    }
    return d;
}

// TRIM_FLAT_PARTITION=0 keeps flat range scans in row order (A/B; results and
// counters are identical either way).
bool flat_partition_enabled() {
    const char* e = std::getenv("TRIM_FLAT_PARTITION");
    return !(e && e[0] == '0');
}

// Block partition for flat range search: k-means centroids of a row sample,
// every row assigned to its (tf32-bound) nearest block, the entries regrouped
// by block (ascending ids inside a block), per-block R / lx range for the
// list-level bound, tcgen05 probe tiles of the block centroids. Any partition is
// valid (the bounds use the actual members); the range filter is order-free,
// so the members and counters are the reference's. Built once, on first use.
bool ensure_flat_partition(trim_index* ix) {
    std::lock_guard<std::mutex> lk(ix->part_mu);
    if (ix->part_tried)
        return ix->part_nb > 0;
    ix->part_tried = true;
    const DevIndex& v = ix->dev;
    const uint64_t n = ix->total;
    uint64_t min_rows = 1u << 16; // TRIM_FLAT_PARTITION_MIN_ROWS: tests partition small indexes
    if (const char* e = std::getenv("TRIM_FLAT_PARTITION_MIN_ROWS"))
        min_rows = std::strtoull(e, nullptr, 10);
    if (!flat_partition_enabled() || v.nlist != 1 || v.dim_stride != v.dim || mma_k(v.dim) > kMmaMaxK ||
        n < std::max<uint64_t>(min_rows, 1024) || n != v.n)
        return false;
    cudaStream_t st = nullptr;
    {
        DevBuf bad(sizeof(uint32_t), st);
        CK(cudaMemsetAsync(bad.p, 0, sizeof(uint32_t), st));
        trim_identity_check_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(v.list_ids, n, v.id_base,
                                                                                         bad.as<uint32_t>());
        uint32_t hb = 0;
        CK(cudaMemcpyAsync(&hb, bad.p, sizeof hb, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (hb)
            return false;
    }
    // blocks: ~4k rows each, up to 16,384 (several blocks per natural cluster of a large
    // index keep the per-block radius, and so the list-level bound, tight)
    uint32_t nb = 256;
    while (nb < 16384 && uint64_t(nb) * 2 * 2048 <= n)
        nb *= 2;
    if (const char* e = std::getenv("TRIM_FLAT_PARTITION_BLOCKS"))
        nb = std::max<uint32_t>(2, static_cast<uint32_t>(std::strtoul(e, nullptr, 10)));
    // k-means on a row sample (the reference's Fisher-Yates sampler)
    const uint64_t ns = std::min<uint64_t>(n, uint64_t(nb) * 40);
    std::vector<uint64_t> rows(ns);
    if (int rc = trim_sample_rows(n, ns, 0x5EED5EEDull, rows.data()))
        throw std::runtime_error(trim_last_error());
    DevBuf d_rows(sizeof(uint64_t) * ns, st), d_sample(sizeof(float) * ns * v.dim, st);
    CK(cudaMemcpyAsync(d_rows.p, rows.data(), sizeof(uint64_t) * ns, cudaMemcpyHostToDevice, st));
    trim_gather_rows_kernel<<<static_cast<unsigned>(ns), 128, 0, st>>>(v.vectors, v.dim_stride, d_rows.as<uint64_t>(),
                                                                       ns, v.dim, d_sample.as<float>());
    CK(cudaStreamSynchronize(st));
    float* cent = ix->alloc<float>(static_cast<size_t>(nb) * v.dim);
    if (nb <= 4096) {
        if (int rc = trim_kmeans_device(d_sample.as<float>(), ns, v.dim, nb, 6, 0x5EEDull, cent, ix->device))
            throw std::runtime_error(trim_last_error());
    } else {
        // two levels (k-means++ seeding scans the whole sample once per centroid): nb / 256
        // top clusters, then up to 256 blocks inside each from its own sample rows
        const uint32_t k1 = nb / 256;
        DevBuf c1(sizeof(float) * k1 * v.dim, st), a1(sizeof(uint32_t) * ns, st), d1(sizeof(float) * ns, st),
            order1(sizeof(uint32_t) * ns, st), offs1(sizeof(uint64_t) * (k1 + 1), st), sub(sizeof(float) * ns * v.dim, st);
        if (int rc = trim_kmeans_device(d_sample.as<float>(), ns, v.dim, k1, 6, 0x5EEDull, c1.as<float>(), ix->device))
            throw std::runtime_error(trim_last_error());
        if (int rc = trim_assign_device(d_sample.as<float>(), ns, v.dim, c1.as<float>(), k1, a1.as<uint32_t>(),
                                        d1.as<float>(), ix->device, st))
            throw std::runtime_error(trim_last_error());
        if (int rc = trim_ivf_lists_device(a1.as<uint32_t>(), ns, k1, offs1.as<uint64_t>(), order1.as<uint32_t>(),
                                           ix->device, st))
            throw std::runtime_error(trim_last_error());
        std::vector<uint64_t> ho(k1 + 1);
        CK(cudaMemcpyAsync(ho.data(), offs1.p, sizeof(uint64_t) * (k1 + 1), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        trim_gather_rows32_kernel<<<static_cast<unsigned>(ns), 128, 0, st>>>(d_sample.as<float>(), v.dim,
                                                                            order1.as<uint32_t>(), ns, v.dim, sub.as<float>());
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(st));
        uint32_t made = 0;
        for (uint32_t c = 0; c < k1; ++c) {
            const uint64_t cnt = ho[c + 1] - ho[c];
            const uint32_t k2 = static_cast<uint32_t>(std::min<uint64_t>(256, cnt / 8));
            if (k2 == 0)
                continue;
            if (int rc = trim_kmeans_device(sub.as<float>() + ho[c] * v.dim, cnt, v.dim, k2, 6, 0x5EEDull + c + 1,
                                            cent + static_cast<size_t>(made) * v.dim, ix->device))
                throw std::runtime_error(trim_last_error());
            made += k2;
        }
        if (made < 2)
            return false;
        nb = made;
    }
    DevIndex a = v;
    a.nlist = nb;
    a.coarse = cent; // dim_stride == dim
    const uint32_t K = mma_k(v.dim);
    const uint32_t ntiles = (nb + kMmaN - 1) / kMmaN;
    ix->part_tiles = ix->alloc<float4>(static_cast<size_t>(ntiles) * (K / 4) * kMmaN);
    ix->part_cn2 = ix->alloc<float>(nb);
    ix->part_cn = ix->alloc<float>(nb);
    trim_coarse_tile_kernel<<<ntiles, kThreads, 0, st>>>(a, K, ix->part_tiles);
    trim_coarse_norm_kernel<<<(nb + kThreads - 1) / kThreads, kThreads, 0, st>>>(a, ix->part_cn2, ix->part_cn);
    CK(cudaGetLastError());
    // assignment: argmin of the tf32 distance bounds, row chunks of 1M
    ix->part_assign = ix->alloc<uint32_t>(n); // kept: the segmented kNN layout regroups by it
    const uint64_t ld = mma_ld(nb); // D~ of a row chunk: at most 2 GB
    const uint64_t ch = std::max<uint64_t>(kMmaM, std::min<uint64_t>(1u << 20, (1ull << 29) / ld / kMmaM * kMmaM));
    DevBuf approx(sizeof(float) * ch * ld, st);
    CK(cudaFuncSetAttribute(trim_probe_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(probe_mma_smem(K))));
    for (uint64_t c0 = 0; c0 < n; c0 += ch) {
        const uint64_t nc = std::min<uint64_t>(ch, n - c0);
        const dim3 grid(static_cast<unsigned>((nc + kMmaM - 1) / kMmaM), (ntiles + kMmaTilesPerCta - 1) / kMmaTilesPerCta);
        trim_probe_mma_kernel<<<grid, kMmaThreads, probe_mma_smem(K), st>>>(
            v.vectors + c0 * v.dim_stride, nc, v.dim_stride, K, ix->part_tiles, ix->part_cn2, nb, approx.as<float>());
        trim_argmin_kernel<<<static_cast<unsigned>((nc + 7) / 8), 256, 0, st>>>(approx.as<float>(), nc, nb, ld,
                                                                                ix->part_assign + c0);
        CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(st));
    uint64_t* offs = ix->alloc<uint64_t>(nb + 1);
    DevBuf order(sizeof(uint32_t) * n, st);
    if (int rc = trim_ivf_lists_device(ix->part_assign, n, nb, offs, order.as<uint32_t>(), ix->device, st))
        throw std::runtime_error(trim_last_error());
    uint8_t* codes = ix->alloc<uint8_t>(n * v.code_stride);
    float* lx = ix->alloc<float>(n);
    uint32_t* ids = ix->alloc<uint32_t>(n);
    trim_partition_gather_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(
        order.as<uint32_t>(), n, v.codes, v.code_stride, v.lx, v.list_ids, codes, lx, ids);
    a.list_offsets = offs;
    a.list_ids = ids;
    a.codes = codes;
    a.lx = lx;
    float* R = ix->alloc<float>(nb);
    float* xmin = ix->alloc<float>(nb);
    float* xmax = ix->alloc<float>(nb);
    trim_list_meta_kernel<<<nb, kThreads, 0, st>>>(a, R, xmin, xmax);
    CK(cudaGetLastError());
    a.list_R = R;
    a.list_xmin = xmin;
    a.list_xmax = xmax;
    CK(cudaStreamSynchronize(st));
    ix->part = a;
    ix->part_nb = nb;
    return true;
}

// TRIM_FLAT_SEGMENTS=0 keeps flat kNN scans in row order (A/B; results and
// counters are identical either way).
bool flat_segments_enabled() {
    const char* e = std::getenv("TRIM_FLAT_SEGMENTS");
    return !(e && e[0] == '0');
}

// Segmented layout for flat kNN (trim_knn_seg_plan_kernel): on top of the block
// partition, rows n0.. regrouped by (segment of seg_len consecutive ids, block),
// ascending ids inside. n0 rows are scanned in order first (their top-k gives
// the threshold the blocks are pruned against); seg_len = rows-per-block-run x
// blocks, so a kept block contributes about one warp-chunk of rows per segment.
bool ensure_flat_segments(trim_index* ix) {
    if (!flat_segments_enabled() || !ensure_flat_partition(ix))
        return false;
    std::lock_guard<std::mutex> lk(ix->seg_mu);
    if (ix->seg_tried)
        return ix->seg_ok;
    ix->seg_tried = true;
    const DevIndex& v = ix->dev;
    const uint64_t n = ix->total;
    const uint32_t nb = ix->part_nb;
    // n0 rows stay in order; then segments that double in length (a query is planned as soon
    // as its threshold allows, knn_seg_batch) up to rows-per-block-run x blocks, then uniform
    uint64_t rpb = 256, n0 = std::max<uint64_t>(uint64_t(std::min<uint32_t>(nb, 4096)) * 16, 4096);
    if (const char* e = std::getenv("TRIM_SEG_ROWS_PER_BLOCK"))
        rpb = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10));
    if (const char* e = std::getenv("TRIM_SEG_N0"))
        n0 = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10));
    n0 = std::min<uint64_t>(n0, n / 4);
    if (n0 == 0 || n >= (1ull << 32))
        return false;
    const uint64_t seg_max = rpb * nb, rest = n - n0;
    std::vector<uint64_t> bounds{n0};
    for (uint64_t len = std::min(n0, seg_max); bounds.back() < n; len = std::min(len * 2, seg_max))
        bounds.push_back(std::min(n, bounds.back() + len));
    const uint64_t nseg = bounds.size() - 1;
    if (nseg == 0 || nseg * nb >= (1ull << 31))
        return false;
    cudaStream_t st = nullptr;
    DevBuf keys(sizeof(uint32_t) * rest, st), order(sizeof(uint32_t) * rest, st);
    DevBuf d_bounds(sizeof(uint64_t) * bounds.size(), st);
    CK(cudaMemcpyAsync(d_bounds.p, bounds.data(), sizeof(uint64_t) * bounds.size(), cudaMemcpyHostToDevice, st));
    trim_seg_key_kernel<<<static_cast<unsigned>((rest + 255) / 256), 256, 0, st>>>(
        ix->part_assign + n0, rest, d_bounds.as<uint64_t>(), static_cast<uint32_t>(nseg), nb, keys.as<uint32_t>());
    CK(cudaGetLastError());
    ix->seg_off = ix->alloc<uint64_t>(nseg * nb + 1);
    if (int rc = trim_ivf_lists_device(keys.as<uint32_t>(), rest, static_cast<uint32_t>(nseg * nb), ix->seg_off,
                                       order.as<uint32_t>(), ix->device, st))
        throw std::runtime_error(trim_last_error());
    uint8_t* codes = ix->alloc<uint8_t>(rest * v.code_stride);
    float* lx = ix->alloc<float>(rest);
    uint32_t* ids = ix->alloc<uint32_t>(rest);
    trim_partition_gather_kernel<<<static_cast<unsigned>((rest + 255) / 256), 256, 0, st>>>(
        order.as<uint32_t>(), rest, v.codes + n0 * v.code_stride, v.code_stride, v.lx + n0, v.list_ids + n0, codes, lx,
        ids);
    CK(cudaGetLastError());
    uint64_t* offs_a = ix->alloc<uint64_t>(2);
    const uint64_t ha[2] = {0, n0};
    CK(cudaMemcpyAsync(offs_a, ha, sizeof ha, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    ix->seg = v;
    ix->seg.codes = codes;
    ix->seg.lx = lx;
    ix->seg.list_ids = ids;
    ix->seg_head = v;
    ix->seg_head.list_offsets = offs_a;
    ix->seg_bounds = bounds;
    ix->seg_nseg = static_cast<uint32_t>(nseg);
    ix->seg_ok = true;
    return true;
}

// Query-tile size of the flat range kernel: as many LUTs as fit while two
// CTAs stay resident per SM (1 = no tiling).
// Code-major copy of the codebook (code c's sub-centroid j at c*dim +
// sub_off[j]): the read order of build_lut_blocked, one contiguous run per
// warp. `cent` is the device copy in the descriptor layout.
float* centroids_code_major(float* out, const float* cent, uint32_t ksub, uint32_t dim,
                            const std::vector<uint32_t>& sub, const std::vector<uint32_t>& off) {
    std::vector<float> h(static_cast<size_t>(ksub) * dim), t(h.size());
    CK(cudaMemcpy(h.data(), cent, sizeof(float) * h.size(), cudaMemcpyDeviceToHost));
    for (size_t j = 0; j < sub.size(); ++j)
        for (uint32_t c = 0; c < ksub; ++c)
            for (uint32_t e = 0; e < sub[j]; ++e)
                t[static_cast<size_t>(c) * dim + off[j] + e] = h[static_cast<size_t>(ksub) * off[j] + c * sub[j] + e];
    CK(cudaMemcpy(out, t.data(), sizeof(float) * t.size(), cudaMemcpyHostToDevice));
    return out;
}

uint32_t range_flat_qt(const DevIndex& v) {
    if (v.nlist != 1 || !probe_mma_enabled_range())
        return 1;
    const int mt = dispatch_m(v);
    uint32_t qt = kFlatMaxQ; // one 16-warp CTA per SM
    while (qt > 1 && range_flat_smem(mt, v.m, v.dim_stride, qt) > kSmemLimit)
        --qt;
    return qt;
}

// ivf::search_trim_ivf_range's filter for nb padded device queries: members
// as (d, id) keys into per-query pools of `cap`, counts, dc and evaluated.
void range_launch(const trim_index* ix, const float* d_q, uint64_t nq, const float* d_r2, uint32_t np,
                  const uint32_t* d_probe, float gamma, uint32_t cap, unsigned long long* d_keys,
                  unsigned int* d_cnt, unsigned long long* d_dc, unsigned long long* d_eval, cudaStream_t st) {
    const DevIndex& v = ix->dev;
    RangeParams p{};
    p.np = np;
    p.two_gamma = 2.0f * gamma;
    p.adc_eps = filter_eps(v.m);
    p.omg_hi = omg_round_up(gamma);
    p.cap = cap;
    if (!d_probe && ensure_flat_partition(const_cast<trim_index*>(ix)) &&
        range_smem_bytes(dispatch_m(ix->part), ix->part.m, ix->part.dim_stride, ix->part_nb) <= kSmemLimit) {
        // flat scan over the block partition: blocks whose bound proves est > r^2 are skipped
        const DevIndex& a = ix->part;
        const uint32_t nb = ix->part_nb, K = mma_k(v.dim);
        const uint32_t ntiles = (nb + kMmaN - 1) / kMmaN;
        DevBuf approx(sizeof(float) * nq * mma_ld(nb), st), kept(sizeof(uint32_t) * nq * nb, st),
            nkept(sizeof(uint32_t) * nq, st);
        CK(cudaFuncSetAttribute(trim_probe_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(probe_mma_smem(K))));
        trim_probe_mma_kernel<<<dim3(static_cast<unsigned>((nq + kMmaM - 1) / kMmaM),
                                     (ntiles + kMmaTilesPerCta - 1) / kMmaTilesPerCta),
                                kMmaThreads, probe_mma_smem(K), st>>>(d_q, nq, v.dim_stride, K, ix->part_tiles,
                                                                      ix->part_cn2, nb, approx.as<float>());
        const double u = std::ldexp(1.0, -24);
        const float kq1 = std::nextafter(static_cast<float>(1.0 - 2.0 * (v.dim + 16) * u), 0.0f);
        const float kq2 = std::nextafter(static_cast<float>(1.0 - 2.0 * (ix->max_sub_dim + v.m + 10) * u), 0.0f);
        const float kest = std::nextafter(static_cast<float>(1.0 - 16.0 * u), 0.0f);
        trim_block_select_kernel<<<static_cast<unsigned>(nq), kThreads, 0, st>>>(
            a, d_q, nq, d_r2, approx.as<float>(), ix->part_cn2, ix->part_cn, omg_round_down(gamma), p.omg_hi, kq1, kq2,
            kest, kept.as<uint32_t>(), nkept.as<uint32_t>(), ix->d_skipped);
        CK(cudaGetLastError());
        const size_t smem = range_smem_bytes(dispatch_m(a), a.m, a.dim_stride, nb);
        p.np = nb;
        p.np_q = nkept.as<uint32_t>();
        p.eval_override = ix->total;
        p.slice = 0;
        constexpr uint32_t kSlices = 4;
        for (uint64_t b = 0; b < nq; b += 65535) {
            RangeParams pb = p;
            const uint64_t nb2 = std::min<uint64_t>(65535, nq - b);
            pb.queries = d_q + b * v.dim_stride;
            pb.nq = nb2;
            pb.radius_sq = d_r2 + b;
            pb.probe = kept.as<uint32_t>() + b * nb;
            pb.np_q = nkept.as<uint32_t>() + b;
            pb.keys = d_keys + b * cap;
            pb.count = d_cnt + b;
            pb.dc = d_dc + b;
            pb.evaluated = d_eval + b;
            launch_range(a, pb, dim3(kSlices, static_cast<unsigned>(nb2)), smem, st);
        }
        return;
    }
    const uint64_t bound = ix->stream_bound(np);
    const uint32_t qt = d_probe ? 1u : range_flat_qt(v);
    if (qt > 1) { // flat scan, query-tiled; at most 65535 slices (grid.y)
        uint64_t slice = 512 * kFlatThreads; // 256k rows: the tile's LUT builds amortised over ~1.5M pairs
        if ((bound + slice - 1) / slice > 65535)
            slice = ((bound + 65534) / 65535 + kFlatThreads - 1) / kFlatThreads * kFlatThreads;
        const uint64_t nslices = std::max<uint64_t>(1, (bound + slice - 1) / slice);
        p.slice = static_cast<uint32_t>(slice);
        p.queries = d_q;
        p.nq = nq;
        p.radius_sq = d_r2;
        p.probe = nullptr;
        p.keys = d_keys;
        p.count = d_cnt;
        p.dc = d_dc;
        p.evaluated = d_eval;
        const uint64_t tiles = (nq + qt - 1) / qt;
        launch_range_flat(v, p, dim3(static_cast<unsigned>(tiles), static_cast<unsigned>(nslices)),
                          range_flat_smem(dispatch_m(v), v.m, v.dim_stride, qt), qt, st);
        return;
    }
    const size_t smem = range_smem_bytes(dispatch_m(v), v.m, v.dim_stride, np);
    const uint32_t slice = 32 * kRangeChunk;
    const uint64_t nslices = std::max<uint64_t>(1, (bound + slice - 1) / slice);
    p.slice = slice;
    for (uint64_t b = 0; b < nq; b += 65535) {
        const uint64_t nb = std::min<uint64_t>(65535, nq - b);
        p.queries = d_q + b * v.dim_stride;
        p.nq = nb;
        p.radius_sq = d_r2 + b;
        p.probe = d_probe ? d_probe + b * np : nullptr;
        p.keys = d_keys + b * cap;
        p.count = d_cnt + b;
        p.dc = d_dc + b;
        p.evaluated = d_eval + b;
        launch_range(v, p, dim3(static_cast<unsigned>(nslices), static_cast<unsigned>(nb)), smem, st);
    }
}

int validate_knn(uint32_t k, float gamma) {
    if (k == 0)
        return set_err(TRIM_EINVAL, "search_trim_ivf_knn: k must be positive");
    if (!(gamma >= 0.0f))
        return set_err(TRIM_EINVAL, "search_trim_ivf_knn: uncalibrated pruning profile");
    if (k > kSmemTopKMax)
        return set_err(TRIM_EINVAL, "search_trim_ivf_knn: k > %u is not supported by the GPU "
                                    "top-k (shared-memory slots)", kSmemTopKMax);
    return TRIM_OK;
}

// TRIM_FLAT_BOUNDS=0 disables the tensor-core distance bounds of flat kNN
// scans (A/B and parity tests; results are identical either way).
bool flat_bounds_enabled() {
    const char* e = std::getenv("TRIM_FLAT_BOUNDS");
    return !(e && e[0] == '0');
}

// Pre-tiled rows and row norms for trim_flat_dist_kernel, built once per index
// on first use (flat indexes only; ~ the size of the vectors).
bool ensure_flat_tiles(trim_index* ix) {
    std::lock_guard<std::mutex> lk(ix->flat_mu);
    if (ix->flat_tiles)
        return true;
    const DevIndex& v = ix->dev;
    const uint32_t K = flat_kpad(v.dim);
    const uint64_t nrt = (v.n + kMmaN - 1) / kMmaN;
    ix->flat_tiles = ix->alloc<float4>(nrt * (K / kFlatKB) * 8 * kMmaN);
    ix->xn = ix->alloc<float>(v.n);
    ix->xn2 = ix->alloc<float>(v.n);
    trim_flat_tile_kernel<<<static_cast<unsigned>(nrt), kThreads>>>(v.vectors, v.n, v.dim_stride, v.dim, K,
                                                                     ix->flat_tiles);
    CK(cudaGetLastError());
    trim_row_norm_kernel<<<static_cast<unsigned>((v.n + 255) / 256), 256>>>(v.vectors, v.n, v.dim_stride, v.dim,
                                                                           ix->xn2, ix->xn);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    return true;
}

// D~ for nq queries (tiled) x every row, row tiles in launches of <= 65535 (grid.y).
void launch_flat_dist(const float4* qtiles, const float* qn2, uint64_t nq, uint64_t nqt, const trim_index* ix,
                      uint32_t K, float* dap, uint64_t ld, uint64_t nrt, cudaStream_t st,
                      __nv_bfloat16* lb = nullptr) {
    for (uint64_t r0 = 0; r0 < nrt; r0 += 65535) {
        const uint64_t ny = std::min<uint64_t>(65535, nrt - r0);
        trim_flat_dist_kernel<<<dim3(static_cast<unsigned>(nqt), static_cast<unsigned>(ny)), kMmaThreads,
                                flat_mma_smem(), st>>>(qtiles, qn2, nq, ix->flat_tiles, ix->xn2, ix->dev.n, K, dap, ld,
                                                       r0, lb, ix->xn);
        CK(cudaGetLastError());
    }
}

// Shared memory of the kNN filter kernel for `np` stream runs (+ the SmemTopK keys for k > 256).
size_t knn_smem_for(const trim_index* ix, uint32_t k, uint32_t np, uint32_t& topk_off) {
    size_t smem = knn_smem_bytes(k > 256 ? 0 : dispatch_m(ix->dev), ix->dev.m, ix->dev.dim_stride, np);
    topk_off = 0;
    if (k > 256) { // SmemTopK keys after the kernel's own layout
        topk_off = static_cast<uint32_t>((smem + 15) & ~size_t(15));
        smem = topk_off + sizeof(unsigned long long) * smem_topk_slots(k);
    }
    return smem;
}

// Segmented flat kNN (ensure_flat_segments) for one batch: the first rows in
// order, the block bounds on tcgen05, the per-query plan (kept blocks merged by
// id into an entry table), then the table-driven kernel and — for the queries
// whose plan does not fit — the in-order kernel over the remaining rows.
// `pb` carries the batch's queries, outputs and dap.
constexpr uint32_t kSegTabCap = 32768; // table entries (kept rows) per query
constexpr uint32_t kSegRounds = 3;     // continue rounds before a query that cannot be planned resumes in order
// The first segment boundary the scan is planned at: rows [0, n_a) go in order. About 1.5 rows
// per block and neighbour wanted are needed before the k-th best comes from the query's own
// neighbourhood (queries that are not there yet continue in order, knn_seg_batch); false: no
// segment left.
bool seg_prefix(const trim_index* ix, uint32_t k, uint32_t& seg0, uint64_t& n_a) {
    const uint64_t want = std::min<uint64_t>(ix->total / 2, uint64_t(k) * std::min<uint32_t>(ix->part_nb, 4096) * 3 / 2);
    seg0 = 0;
    while (seg0 < ix->seg_nseg && ix->seg_bounds[seg0] < want)
        ++seg0;
    if (seg0 >= ix->seg_nseg)
        return false;
    n_a = ix->seg_bounds[seg0];
    return true;
}

void knn_seg_batch(const trim_index* ix, KnnParams pb, uint32_t seg0, uint64_t n_a, cudaStream_t st) {
    const DevIndex& v = ix->dev;
    const uint32_t k = pb.k, nb = ix->part_nb, K = mma_k(v.dim);
    const uint64_t nq = pb.nq;
    uint32_t off_a = 0;
    const size_t smem_a = knn_smem_for(ix, k, 1, off_a);
    // the first n_a rows, in order (pb.dap, if any, covers exactly these rows)
    DevBuf ids_a(sizeof(uint32_t) * nq * k, st), dist_a(sizeof(float) * nq * k, st),
        ct_a(sizeof(unsigned long long) * nq * 6, st), offs_a(sizeof(uint64_t) * 2, st);
    DevIndex head = ix->seg_head;
    if (seg0) { // (pageable copy of 16 bytes: staged by the runtime before the call returns)
        const uint64_t ha[2] = {0, n_a};
        CK(cudaMemcpyAsync(offs_a.p, ha, sizeof ha, cudaMemcpyHostToDevice, st));
        head.list_offsets = offs_a.as<uint64_t>();
    }
    KnnParams pa = pb;
    pa.np = 1;
    pa.probe = nullptr;
    pa.plan = nullptr;
    pa.ids_out = ids_a.as<uint32_t>();
    pa.dist_out = dist_a.as<float>();
    pa.counters = ct_a.as<unsigned long long>();
    pa.topk_off = off_a;
    pa.timeline = nullptr;
    launch_knn(head, pa, smem_a, st);
    // |q - c_b|^2 bounds to the block centroids
    const uint32_t ntiles = (nb + kMmaN - 1) / kMmaN;
    DevBuf approx(sizeof(float) * nq * mma_ld(nb), st);
    CK(cudaFuncSetAttribute(trim_probe_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(probe_mma_smem(K))));
    trim_probe_mma_kernel<<<dim3(static_cast<unsigned>((nq + kMmaM - 1) / kMmaM),
                                 (ntiles + kMmaTilesPerCta - 1) / kMmaTilesPerCta),
                            kMmaThreads, probe_mma_smem(K), st>>>(pb.queries, nq, v.dim_stride, K, ix->part_tiles,
                                                                  ix->part_cn2, nb, approx.as<float>());
    CK(cudaGetLastError());
    const KnnPlanLayout lo = KnnPlanLayout::of(1, k);
    DevBuf recs(sizeof(uint32_t) * lo.words * nq, st), tab(sizeof(uint32_t) * kSegTabCap * nq, st);
    SegPlanParams sp{};
    sp.queries = pb.queries;
    sp.nq = nq;
    sp.k = k;
    sp.np = 1;
    sp.tab_cap = kSegTabCap;
    sp.n = ix->total;
    sp.nseg = ix->seg_nseg;
    sp.seg_off = ix->seg_off;
    sp.ids = ix->seg.list_ids;
    sp.approx = approx.as<float>();
    sp.cn2 = ix->part_cn2;
    sp.cn = ix->part_cn;
    sp.ids_a = ids_a.as<uint32_t>();
    sp.dist_a = dist_a.as<float>();
    sp.ct_a = ct_a.as<unsigned long long>();
    sp.omg_lo = pb.omg_lo;
    sp.omg_hi = pb.omg_hi;
    sp.kq1 = pb.kq1;
    sp.kq2 = pb.kq2;
    sp.kest = pb.kest;
    sp.recs = recs.as<uint32_t>();
    sp.tab = tab.as<uint32_t>();
    sp.skipped = pb.skip_lists ? pb.skipped : nullptr;
    {
        const char* e = std::getenv("TRIM_SEG_FORCE_PLAIN"); // tests: every query takes the in-order resume
        sp.force_plain = (e && e[0] == '1') || !pb.skip_lists ? 1u : 0u;
    }
    DevBuf dbg;
    const bool debug = std::getenv("TRIM_SEG_DEBUG") != nullptr;
    if (debug) {
        dbg = DevBuf(sizeof(uint32_t) * 4 * nq, st);
        sp.dbg = dbg.as<uint32_t>();
    }
    // Plan; a query whose plan does not fit yet (its threshold still comes from other
    // neighbourhoods) scans the next segment in order and is planned again, up to
    // kSegRounds times; after the last round it resumes in order for good.
    uint32_t rounds = kSegRounds;
    if (const char* e = std::getenv("TRIM_SEG_ROUNDS"))
        rounds = static_cast<uint32_t>(std::strtoul(e, nullptr, 10));
    KnnParams pc = pa; // continue rounds: in order over the original arrays, state in place
    pc.dap = nullptr;
    pc.dap_ld = 0;
    pc.plan = recs.as<uint32_t>();
    pc.mode_sel = 2;
    for (uint32_t r = 0;; ++r) {
        const uint32_t g = seg0 + r;
        const bool last = r >= rounds || g + 1 >= ix->seg_nseg;
        sp.round = r;
        sp.seg0 = g;
        sp.n0 = ix->seg_bounds[g];
        sp.n_next = last ? 0 : ix->seg_bounds[g + 1];
        trim_knn_seg_plan_kernel<<<static_cast<unsigned>(nq), kThreads, 0, st>>>(ix->part, sp);
        CK(cudaGetLastError());
        if (debug) { // plan statistics of the batch (synchronises)
            std::vector<uint32_t> h(4 * nq), hm(lo.words * nq);
            CK(cudaMemcpyAsync(h.data(), dbg.p, sizeof(uint32_t) * 4 * nq, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(hm.data(), recs.p, sizeof(uint32_t) * lo.words * nq, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            uint64_t mode[3] = {0, 0, 0}, kept = 0, rows = 0, kmax = 0;
            for (uint64_t i = 0; i < nq; ++i) {
                const uint32_t md = hm[i * lo.words + 7] & 0xffu;
                ++mode[md < 3 ? md : 0];
                if (md == 1) {
                    kept += h[4 * i];
                    kmax = std::max<uint64_t>(kmax, h[4 * i]);
                    rows += hm[i * lo.words + 3];
                }
            }
            std::fprintf(stderr,
                         "[trim seg] round %u: nq=%llu nb=%u rows_in_order=%llu segments=%u..%u: planned=%llu "
                         "(kept/q=%.1f max %llu, table rows/q=%.1f) continue=%llu in-order=%llu\n",
                         r, (unsigned long long)nq, nb, (unsigned long long)sp.n0, g, ix->seg_nseg,
                         (unsigned long long)mode[1], mode[1] ? double(kept) / mode[1] : 0.0, (unsigned long long)kmax,
                         mode[1] ? double(rows) / mode[1] : 0.0, (unsigned long long)mode[2],
                         (unsigned long long)mode[0]);
        }
        if (last)
            break;
        launch_knn(v, pc, smem_a, st); // records of mode 2: [bounds[g], bounds[g + 1]) in order
    }
    pb.plan = recs.as<uint32_t>();
    pb.np = 1;
    pb.probe = nullptr;
    pb.dap = nullptr; // the distance bounds cover the in-order prefix only
    pb.dap_ld = 0;
    pb.tab = tab.as<uint32_t>();
    pb.tab_cap = kSegTabCap;
    pb.mode_sel = 0;
    pb.topk_off = off_a;
    launch_knn(v, pb, smem_a, st);           // records of mode 0: in order over the original arrays (the long ones first)
    launch_knn_seg(ix->seg, pb, smem_a, st); // records of mode 1: the entry tables
}

// kNN filter launch over padded device queries and precomputed probe lists
// (d_probe null => nlist == 1, the single list 0).
int knn_launch(const trim_index* ix, const float* d_q, uint64_t nq, uint32_t k, uint32_t np,
               const uint32_t* d_probe, float gamma, uint32_t* d_ids, float* d_dist,
               unsigned long long* d_ct, uint32_t* d_status, cudaStream_t st) {
    if (nq == 0)
        return TRIM_OK;
    if (ix->dev.nlist == 1 && np == 1)
        d_probe = nullptr; // a flat index: the one list, whatever the caller's probe array says
    size_t smem = knn_smem_bytes(k > 256 ? 0 : dispatch_m(ix->dev), ix->dev.m, ix->dev.dim_stride, np);
    uint32_t topk_off = 0;
    if (k > 256) { // SmemTopK keys after the kernel's own layout
        topk_off = static_cast<uint32_t>((smem + 15) & ~size_t(15));
        smem = topk_off + sizeof(unsigned long long) * smem_topk_slots(k);
    }
    if (smem > kSmemLimit)
        return set_err(TRIM_EINVAL,
                       "search_trim_ivf_knn: per-query state (%zu B for m=%u, ksub=%u, "
                       "nprobe=%u) exceeds 227 KB of shared memory",
                       smem, ix->dev.m, ix->dev.ksub, np);
    KnnParams p{};
    p.queries = d_q;
    p.nq = nq;
    p.k = k;
    p.np = np;
    p.probe = d_probe;
    p.two_gamma = 2.0f * gamma;
    p.adc_eps = filter_eps(ix->dev.m);
    p.omg_hi = omg_round_up(gamma);
    p.ids_out = d_ids;
    p.dist_out = d_dist;
    p.counters = d_ct;
    p.status = d_status;
    p.topk_off = topk_off;
    // list-level bound slack (list_lower_bound): relative error bounds of the
    // fp32 coarse distance (dim terms), of sqrt of the reference ADC (LUT entries of
    // <= max_sd terms summed over m), and of relaxed_lb's evaluation; u = 2^-24
    {
        const double u = std::ldexp(1.0, -24);
        const double kq1 = 1.0 - 2.0 * (ix->dev.dim + 16) * u;
        const double kq2 = 1.0 - 2.0 * (ix->max_sub_dim + ix->dev.m + 10) * u;
        const double kest = 1.0 - 16.0 * u;
        p.kq1 = std::nextafter(static_cast<float>(kq1), 0.0f);
        p.kq2 = std::nextafter(static_cast<float>(kq2), 0.0f);
        p.kest = std::nextafter(static_cast<float>(kest), 0.0f);
        p.omg_lo = omg_round_down(gamma);
        { // StageCut constants, rounded to the safe side
            const double ol = p.omg_lo, oh = p.omg_hi, c1 = 1.0 - std::max(ol * ol, oh * oh);
            float f = static_cast<float>(c1);
            if (static_cast<double>(f) > c1)
                f = std::nextafter(f, -INFINITY);
            p.stage_c1 = f;
            const double e = p.adc_eps, um = 1.0 - std::ldexp(1.0, -24);
            if (e < 1.0) {
                const double ka = (1.0 + std::ldexp(1.0, -20)) / ((1.0 - e) * um * um);
                float g = static_cast<float>(ka);
                if (static_cast<double>(g) < ka)
                    g = std::nextafter(g, INFINITY);
                p.stage_ka = g;
            } else {
                p.stage_ka = INFINITY;
            }
        }
        p.skip_lists = list_skip_enabled() ? 1u : 0u;
        p.skipped = ix->d_skipped;
        p.timeline = g_timeline;
    }
    // flat scans: tensor-core distance bounds for every (query, row), so only
    // members that can enter the top-k get the exact distance
    // (up to 16M rows: D~ holds nq x rows floats and the pre-tiled rows another copy of the vectors)
    // flat scans of partitioned indexes: segmented block stream (knn_seg_batch); the distance
    // bounds then cover only the rows scanned in order
    uint32_t seg0 = 0;
    uint64_t n_a = 0;
    const bool seg = ix->dev.nlist == 1 && !d_probe && np == 1 && ensure_flat_segments(const_cast<trim_index*>(ix)) &&
                     uint64_t(k) * 4 <= ix->seg_bounds[0] && seg_prefix(ix, k, seg0, n_a) &&
                     knn_smem_bytes(k > 256 ? 0 : dispatch_m(ix->dev), ix->dev.m, ix->dev.dim_stride, 1) <= kSmemLimit;
    const uint64_t bound_rows = seg ? n_a : ix->dev.n;
    const bool flat_bounds = ix->dev.nlist == 1 && np == 1 && ix->dev.n > 0 && ix->dev.n <= (16ull << 20) &&
                             flat_bounds_enabled() && ensure_flat_tiles(const_cast<trim_index*>(ix));
    const uint64_t ld = flat_bounds ? (bound_rows + kMmaN - 1) / kMmaN * kMmaN : 0;
    // slices: grid.x <= 2^31-1; with bounds, D~ of a slice (nq x ld floats) within ~8 GB
    uint64_t slice = 1u << 30;
    if (flat_bounds)
        slice = std::max<uint64_t>(kMmaM, (8ull << 30) / (ld * 2) / kMmaM * kMmaM);
    if (seg)
        slice = std::min<uint64_t>(slice, 2048); // the entry tables: 128 KB per query
    for (uint64_t b = 0; b < nq; b += slice) {
        KnnParams pb = p;
        pb.nq = std::min<uint64_t>(slice, nq - b);
        DevBuf dap;
        if (flat_bounds) {
            const DevIndex& v = ix->dev;
            const uint32_t K = flat_kpad(v.dim);
            const uint64_t nqt = (pb.nq + kMmaM - 1) / kMmaM, nrt = ld / kMmaN;
            const float* qb = d_q + b * v.dim_stride;
            DevBuf qtiles(sizeof(float4) * nqt * (K / kFlatKB) * 8 * kMmaM, st), qn2(sizeof(float) * pb.nq, st);
            trim_flat_tile_kernel<<<static_cast<unsigned>(nqt), kThreads, 0, st>>>(qb, pb.nq, v.dim_stride, v.dim, K,
                                                                                   qtiles.as<float4>());
            CK(cudaGetLastError());
            trim_query_norm_kernel<<<static_cast<unsigned>((pb.nq + 255) / 256), 256, 0, st>>>(qb, pb.nq, v.dim_stride,
                                                                                               v.dim, qn2.as<float>());
            CK(cudaGetLastError());
            dap = DevBuf(sizeof(__nv_bfloat16) * pb.nq * ld, st); // bf16 lower bounds D~ - E
            CK(cudaFuncSetAttribute(trim_flat_dist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(flat_mma_smem())));
            launch_flat_dist(qtiles.as<float4>(), qn2.as<float>(), pb.nq, nqt, ix, K, nullptr, ld, nrt, st,
                             dap.as<__nv_bfloat16>());
            pb.dap = dap.as<__nv_bfloat16>();
            pb.dap_ld = ld;
        }
        pb.queries = d_q + b * ix->dev.dim_stride;
        pb.probe = p.probe ? p.probe + b * np : nullptr;
        pb.ids_out = d_ids + b * k;
        pb.dist_out = d_dist + b * k;
        pb.counters = d_ct ? d_ct + b * 6 : nullptr;
        pb.timeline = p.timeline ? p.timeline + b * kTimeline : nullptr;
        DevBuf recs;
        if (pb.probe && knn_setup_enabled()) { // seeds + plan ahead of the filter kernel
            const KnnPlanLayout lo = KnnPlanLayout::of(np, k);
            recs = DevBuf(sizeof(uint32_t) * lo.words * pb.nq, st);
            const size_t ssm = sizeof(uint64_t) * np + sizeof(uint32_t) * (np + 1);
            if (ssm > 48 * 1024)
                CK(cudaFuncSetAttribute(trim_knn_setup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(ssm)));
            trim_knn_setup_kernel<<<static_cast<unsigned>(pb.nq), kWarp, ssm, st>>>(ix->dev, pb, recs.as<uint32_t>());
            CK(cudaGetLastError());
            pb.plan = recs.as<uint32_t>();
        }
        if (seg) {
            knn_seg_batch(ix, pb, seg0, n_a, st);
            continue;
        }
        launch_knn(ix->dev, pb, smem, st);
    }
    return TRIM_OK;
}

// Probe + filter over padded device queries.
int knn_device(const trim_index* ix, const float* d_q, uint64_t nq, uint32_t k, uint32_t nprobe,
               float gamma, uint32_t* d_ids, float* d_dist, unsigned long long* d_ct,
               uint32_t* d_status, cudaStream_t st) {
    if (nq == 0)
        return TRIM_OK;
    DevBuf d_probe;
    const uint32_t np = run_probe(ix, d_q, nq, nprobe, d_probe, st);
    return knn_launch(ix, d_q, nq, k, np, d_probe.as<uint32_t>(), gamma, d_ids, d_dist, d_ct, d_status,
                      st);
}

// ivf::search_baseline_ivfpq over padded device queries; host outputs.
int baseline_device(const trim_index* ix, const float* d_q, uint64_t nq, uint32_t k, uint32_t np,
                    const uint32_t* d_probe, uint32_t kp, uint32_t* ids_out, float* dist_out,
                    trim_counters* counters_out, cudaStream_t st) {
    if (kp > kSelSmemKeys)
        return set_err(TRIM_EINVAL, "search_baseline_ivfpq: k_prime > %u is not supported",
                       kSelSmemKeys);
    const uint64_t bound = std::max<uint64_t>(1, ix->stream_bound(np));
    const uint32_t slice = 32 * kBaselineSlice;
    const uint64_t nslices = (bound + slice - 1) / slice;
    const uint64_t qb = std::max<uint64_t>(1, std::min<uint64_t>({nq, 65535, (1ull << 31) / (bound * 8)}));
    size_t est_smem = lut_bytes(dispatch_m(ix->dev), ix->dev.m) + sizeof(float) * ix->dev.dim_stride;
    est_smem += sizeof(uint64_t) * np + sizeof(uint32_t) * (np + 1);
    if (est_smem > kSmemLimit)
        return set_err(TRIM_EINVAL, "search_baseline_ivfpq: per-query state exceeds 227 KB");
    uint32_t kp2 = pow2_at_least(kp);
    const size_t ref_smem = sizeof(float) * ix->dev.dim_stride + sizeof(unsigned long long) * kp2;
    const size_t sel_smem = sizeof(unsigned long long) * kSelSmemKeys;
    DevBuf d_keys(sizeof(unsigned long long) * qb * bound, st), d_tot(sizeof(unsigned long long) * nq, st),
        d_sel(sizeof(unsigned long long) * qb * kp, st), d_ids(sizeof(uint32_t) * nq * k, st),
        d_dist(sizeof(float) * nq * k, st);
    CK(cudaFuncSetAttribute(trim_bl_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(sel_smem)));
    CK(cudaFuncSetAttribute(trim_bl_refine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(ref_smem)));
    for (uint64_t b = 0; b < nq; b += qb) {
        const uint64_t nb = std::min<uint64_t>(qb, nq - b);
        BlParams p{};
        p.queries = d_q + b * ix->dev.dim_stride;
        p.nq = nb;
        p.np = np;
        p.probe = d_probe ? d_probe + b * np : nullptr;
        p.slice = slice;
        p.stride = bound;
        p.keys = d_keys.as<unsigned long long>();
        p.total = d_tot.as<unsigned long long>() + b;
        launch_bl_est(ix->dev, p, dim3(static_cast<unsigned>(nslices), static_cast<unsigned>(nb)),
                      est_smem, st);
        trim_bl_select_kernel<<<static_cast<unsigned>(nb), kSelThreads, sel_smem, st>>>(
            d_keys.as<unsigned long long>(), bound, p.total, kp, d_sel.as<unsigned long long>());
        CK(cudaGetLastError());
        trim_bl_refine_kernel<<<static_cast<unsigned>(nb), kThreads, ref_smem, st>>>(
            ix->dev, p.queries, d_sel.as<unsigned long long>(), p.total, kp, kp2, k,
            d_ids.as<uint32_t>() + b * k, d_dist.as<float>() + b * k);
        CK(cudaGetLastError());
    }
    std::vector<unsigned long long> tot(nq);
    CK(cudaMemcpyAsync(ids_out, d_ids.p, sizeof(uint32_t) * nq * k, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(dist_out, d_dist.p, sizeof(float) * nq * k, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(tot.data(), d_tot.p, sizeof(unsigned long long) * nq, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (uint64_t i = 0; i < nq; ++i)
        if (tot[i] < k)
            return set_err(TRIM_EINVAL, "search_baseline_ivfpq: k exceeds probed vectors");
    if (counters_out) {
        for (uint64_t i = 0; i < nq; ++i) {
            trim_counters& c = counters_out[i];
            c.evaluated = tot[i];
            c.edc = tot[i];
            c.dc = std::min<uint64_t>(kp, tot[i]);
            c.pruned = c.evaluated - c.dc;
            c.hops = 0;
            c.coarse_dc = ix->dev.nlist;
        }
    }
    return TRIM_OK;
}

// ------------------------------------------------------------ graph search
} // namespace

struct trim_graph {
    int device = 0;
    GraphDev dev{};
    std::vector<void*> allocs;
    ~trim_graph() {
        if (!allocs.empty()) {
            int prev = 0;
            cudaGetDevice(&prev);
            cudaSetDevice(device);
            for (void* p : allocs)
                cudaFree(p);
            cudaSetDevice(prev);
        }
    }
    template <typename T>
    T* alloc(size_t count) {
        void* p = nullptr;
        CK(cudaMalloc(&p, std::max<size_t>(sizeof(T) * count, 16)));
        allocs.push_back(p);
        return static_cast<T*>(p);
    }
};

namespace {

// Candidate-queue register sets: 32*S >= max(ef, k) slots.
uint32_t graph_slots(uint32_t need) {
    uint32_t S = 1;
    while (32u * S < need)
        S <<= 1;
    return S;
}

// One graph search over nq device-resident queries (rows padded to
// dim_stride). Workspace: a visited bitmap and a search-queue heap per query;
// queries run in groups that fit `budget` bytes, and a query whose search
// queue outgrew the first capacity is re-run with capacity n + 1 (exact).
// kNN writes d_ids/d_dist (nq x k); range writes the pool (nq x cap keys) and
// counts. d_ct: nq x 6 counters.
void graph_run(trim_graph* gr, const float* d_q, uint64_t nq, uint32_t k, uint32_t ef, float gamma,
               bool range, const float* d_r2, uint32_t* d_ids, float* d_dist, unsigned long long* d_pool,
               uint64_t cap, unsigned long long* d_counts, unsigned long long* d_ct, cudaStream_t st) {
    const GraphDev& g = gr->dev;
    const uint64_t n = g.ix.n, vwords = (n + 31) / 32;
    const uint32_t S = graph_slots(std::max(ef, range ? 1u : k));
    // first run: the search queue in shared memory (TRIM_GRAPH_HEAP_CAP entries,
    // default 1024; tests force overflows with a tiny one); overflowed queries
    // are re-run with a global-memory queue of capacity n + 1 (exact)
    uint64_t hs = 1024;
    if (const char* e = std::getenv("TRIM_GRAPH_HEAP_CAP"))
        hs = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10));
    hs = std::min<uint64_t>(hs, n + 1);
    const size_t budget = size_t(1) << 30;
    GraphParams p{};
    p.k = k;
    p.ef = ef;
    p.two_gamma = 2.0f * gamma;
    p.range = range ? 1u : 0u;
    p.cap = cap;
    p.vwords = vwords;
    // run queries [q0, q0 + nb), or the nb queries listed in d_map
    auto run = [&](uint64_t q0, uint64_t nb, bool global_heap, const uint32_t* d_map, uint32_t* d_status) {
        const uint64_t heap_cap = global_heap ? n + 1 : hs;
        const size_t smem = graph_smem_bytes(g.ix.m, g.ix.ksub, g.ix.dim_stride, global_heap ? 0 : hs);
        if (smem > kSmemLimit) {
            set_err(TRIM_EINVAL, "graph search: per-query shared memory (%zu B) exceeds 227 KB", smem);
            throw CudaError{TRIM_EINVAL};
        }
        const size_t per_q = vwords * 4 + (global_heap ? heap_cap * 8 : 0);
        const uint64_t group = std::max<uint64_t>(1, std::min<uint64_t>(nb, budget / per_q));
        DevBuf vis(vwords * 4 * group, st), heap(global_heap ? heap_cap * 8 * group : 8, st);
        for (uint64_t g0 = 0; g0 < nb; g0 += group) {
            const uint64_t gn = std::min(group, nb - g0), qi = d_map ? 0 : q0 + g0;
            CK(cudaMemsetAsync(vis.p, 0, vwords * 4 * gn, st));
            GraphParams pp = p;
            pp.nq = gn;
            pp.qmap = d_map ? d_map + g0 : nullptr;
            pp.queries = d_q + qi * g.ix.dim_stride;
            pp.r2 = range ? d_r2 + qi : nullptr;
            pp.ids_out = range ? nullptr : d_ids + qi * k;
            pp.dist_out = range ? nullptr : d_dist + qi * k;
            pp.pool = range ? d_pool + qi * cap : nullptr;
            pp.counts = range ? d_counts + qi : nullptr;
            pp.counters = d_ct + qi * 6;
            pp.visited = vis.as<uint32_t>();
            pp.heap = global_heap ? heap.as<unsigned long long>() : nullptr;
            pp.heap_cap = heap_cap;
            pp.status = d_status + qi;
            CK(launch_graph(g, pp, S, smem, st));
        }
    };
    DevBuf d_status(sizeof(uint32_t) * std::max<uint64_t>(nq, 1), st);
    CK(cudaMemsetAsync(d_status.p, 0, sizeof(uint32_t) * nq, st));
    run(0, nq, false, nullptr, d_status.as<uint32_t>());
    if (hs >= n + 1)
        return;
    std::vector<uint32_t> status(nq);
    CK(cudaMemcpyAsync(status.data(), d_status.p, sizeof(uint32_t) * nq, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::vector<uint32_t> redo;
    for (uint64_t i = 0; i < nq; ++i)
        if (status[i] & 1u)
            redo.push_back(static_cast<uint32_t>(i));
    if (redo.empty())
        return;
    DevBuf d_map(sizeof(uint32_t) * redo.size(), st);
    CK(cudaMemcpyAsync(d_map.p, redo.data(), sizeof(uint32_t) * redo.size(), cudaMemcpyHostToDevice, st));
    run(0, redo.size(), true, d_map.as<uint32_t>(), d_status.as<uint32_t>());
    CK(cudaStreamSynchronize(st)); // d_map / redo stay alive until the re-run is done
}

DevBuf graph_upload_queries(const trim_graph* gr, const float* q, uint64_t nq, cudaStream_t st) {
    const uint32_t dim = gr->dev.ix.dim, ds = gr->dev.ix.dim_stride;
    DevBuf d(sizeof(float) * std::max<uint64_t>(nq, 1) * ds, st);
    if (nq == 0)
        return d;
    CK(cudaMemsetAsync(d.p, 0, sizeof(float) * nq * ds, st));
    CK(cudaMemcpy2DAsync(d.p, sizeof(float) * ds, q, sizeof(float) * dim, sizeof(float) * dim, nq,
                         cudaMemcpyHostToDevice, st));
    return d;
}

void put_counters_host(trim_counters* out, const std::vector<unsigned long long>& ct, uint64_t nq) {
    for (uint64_t i = 0; i < nq; ++i) {
        out[i].dc = ct[i * 6 + 0];
        out[i].edc = ct[i * 6 + 1];
        out[i].pruned = ct[i * 6 + 2];
        out[i].evaluated = ct[i * 6 + 3];
        out[i].hops = ct[i * 6 + 4];
        out[i].coarse_dc = ct[i * 6 + 5];
    }
}

} // namespace

extern "C" {

const char* trim_last_error(void) { return g_err.c_str(); }

void trim__set_last_error(const char* msg) { g_err = msg; }

void trim__set_knn_timeline(void* d_buf) { g_timeline = static_cast<unsigned long long*>(d_buf); }

int trim_abi_version(void) { return TRIM_ABI_VERSION; }

void trim_free(void* p) { std::free(p); }

int trim_index_create(const trim_index_desc* d, trim_index_t* out) {
    if (!d || !out)
        return set_err(TRIM_EINVAL, "trim_index_create: null argument");
    *out = nullptr;
    if (d->dim == 0)
        return set_err(TRIM_EDATA, "dataset dimension must be >= 1");
    if (d->m == 0 || d->m > d->dim)
        return set_err(TRIM_EINVAL, "PqParams: need 1 <= m <= dim");
    if (d->ksub == 0 || d->ksub > 256)
        return set_err(TRIM_EINVAL, "PqParams: need 1 <= c <= 256 for byte codes");
    if (d->m > 128)
        return set_err(TRIM_EINVAL, "trim_index_create: m > 128 subspaces is not supported");
    if (d->nlist == 0)
        return set_err(TRIM_EINVAL, "build_ivf: need 1 <= nlist <= n");
    if (d->nlist > 16384)
        return set_err(TRIM_EINVAL, "trim_index_create: nlist > 16384 is not supported by the "
                                    "shared-memory probe sort");
    if (d->code_stride < d->m)
        return set_err(TRIM_EINVAL, "trim_index_create: code_stride < m");
    if (!d->sub_dims || !d->centroids || !d->coarse || !d->list_offsets)
        return set_err(TRIM_EINVAL, "trim_index_create: null array in descriptor");
    if (int rc = check_device_present())
        return rc;
    if (d->ndevices > 0 && d->shard_mode != TRIM_SHARD_SINGLE) {
        if (!d->devices)
            return set_err(TRIM_EINVAL, "trim_index_create: ndevices > 0 needs devices[]");
        if (d->shard_mode != TRIM_SHARD_ID && d->shard_mode != TRIM_SHARD_REPLICAS)
            return set_err(TRIM_EINVAL, "trim_index_create: unknown shard_mode %d", (int)d->shard_mode);
        return guarded([&]() -> int { return group_create(d, out); });
    }
    return create_single(d, out);
}

} // extern "C"

int trimhost::create_single(const trim_index_desc* d, trim_index** out) {
    *out = nullptr;
    return guarded([&]() -> int {
        const bool host = d->memory == TRIM_MEM_HOST;
        const cudaMemcpyKind kind = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        DeviceGuard g(d->device);
        { // keep the per-call stream-ordered workspaces (queries, probe scratch,
          // results, flat-scan entry tables: up to ~0.5 GB per batch in flight) cached
          // in the device's pool, but return anything beyond 4 GiB (e.g. a flat-bound
          // slice) to the device at the next synchronisation, so it never starves other
          // allocators
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, d->device) == cudaSuccess) {
                uint64_t thr = 0;
                cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
                if (thr < (4ull << 30)) {
                    thr = 4ull << 30;
                    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
                }
            }
        }
        auto* ix = new trim_index;
        ix->device = d->device;
        // host copies of the small arrays (sub_dims, offsets)
        std::vector<uint32_t> sub(d->m);
        std::vector<uint64_t> offs(d->nlist + 1);
        if (host) {
            std::memcpy(sub.data(), d->sub_dims, sizeof(uint32_t) * d->m);
            std::memcpy(offs.data(), d->list_offsets, sizeof(uint64_t) * (d->nlist + 1));
        } else {
            CK(cudaMemcpy(sub.data(), d->sub_dims, sizeof(uint32_t) * d->m, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(offs.data(), d->list_offsets, sizeof(uint64_t) * (d->nlist + 1),
                          cudaMemcpyDeviceToHost));
        }
        uint64_t sdsum = 0;
        std::vector<uint32_t> suboff(d->m);
        for (uint32_t j = 0; j < d->m; ++j) {
            suboff[j] = static_cast<uint32_t>(sdsum);
            sdsum += sub[j];
        }
        for (uint32_t j = 0; j < d->m; ++j)
            ix->max_sub_dim = std::max(ix->max_sub_dim, sub[j]);
        if (sdsum != d->dim) {
            delete ix;
            return set_err(TRIM_EDATA, "codebook sub_dims do not sum to dim");
        }
        if (offs[0] != 0) {
            delete ix;
            return set_err(TRIM_EDATA, "ivf offsets must start at 0");
        }
        for (uint32_t l = 0; l < d->nlist; ++l)
            if (offs[l + 1] < offs[l]) {
                delete ix;
                return set_err(TRIM_EDATA, "ivf offsets are not monotone");
            }
        const uint64_t total = offs[d->nlist];
        if (total > 0xFFFFFFFFull) {
            delete ix;
            return set_err(TRIM_EINVAL, "trim_index_create: more than 2^32-1 entries per device");
        }
        if (total && (!d->list_ids || !d->list_codes || !d->list_lx || !d->vectors)) {
            delete ix;
            return set_err(TRIM_EINVAL, "trim_index_create: null list array in descriptor");
        }
        if (host) {
            for (uint64_t e = 0; e < total; ++e) {
                const uint64_t id = d->list_ids[e];
                if (id < d->id_base || id - d->id_base >= d->n) {
                    delete ix;
                    return set_err(TRIM_EDATA,
                                   "ivf entry id %llu outside the vector rows [%llu, %llu)",
                                   (unsigned long long)id, (unsigned long long)d->id_base,
                                   (unsigned long long)(d->id_base + d->n));
                }
            }
        }
        ix->total = total;
        ix->list_offsets = offs;
        std::vector<uint64_t> sizes(d->nlist);
        for (uint32_t l = 0; l < d->nlist; ++l)
            sizes[l] = offs[l + 1] - offs[l];
        std::sort(sizes.begin(), sizes.end(), std::greater<uint64_t>());
        ix->top_prefix.assign(d->nlist + 1, 0);
        for (uint32_t l = 0; l < d->nlist; ++l)
            ix->top_prefix[l + 1] = ix->top_prefix[l] + sizes[l];
        ix->max_list = d->nlist ? sizes[0] : 0;

        DevIndex& v = ix->dev;
        v.dim = d->dim;
        v.dim_stride = round_up(d->dim, 4);
        v.m = d->m;
        v.ksub = d->ksub;
        v.code_stride = round_up(d->m, 16);
        v.nlist = d->nlist;
        v.sd_uniform = sub.empty() ? 0u : sub[0];
        for (uint32_t j = 1; j < d->m; ++j)
            if (sub[j] != sub[0])
                v.sd_uniform = 0;
        v.n = d->n;
        v.id_base = d->id_base;
        ix->code_stride_host = d->code_stride;
        try {
            uint32_t* dsub = ix->alloc<uint32_t>(d->m);
            uint32_t* doff = ix->alloc<uint32_t>(d->m);
            CK(cudaMemcpy(dsub, sub.data(), sizeof(uint32_t) * d->m, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(doff, suboff.data(), sizeof(uint32_t) * d->m, cudaMemcpyHostToDevice));
            v.sub_dims = dsub;
            v.sub_offsets = doff;
            float* cent = ix->alloc<float>(static_cast<size_t>(d->ksub) * d->dim);
            CK(cudaMemcpy(cent, d->centroids, sizeof(float) * d->ksub * d->dim, kind));
            v.centroids = cent;
            v.centroids_t = centroids_code_major(ix->alloc<float>(static_cast<size_t>(d->ksub) * d->dim), cent,
                                                 d->ksub, d->dim, sub, suboff);
            float* coarse = ix->alloc<float>(static_cast<size_t>(d->nlist) * v.dim_stride);
            CK(cudaMemset(coarse, 0, sizeof(float) * d->nlist * v.dim_stride));
            CK(cudaMemcpy2D(coarse, sizeof(float) * v.dim_stride, d->coarse, sizeof(float) * d->dim,
                            sizeof(float) * d->dim, d->nlist, kind));
            v.coarse = coarse;
            uint64_t* loff = ix->alloc<uint64_t>(d->nlist + 1);
            CK(cudaMemcpy(loff, offs.data(), sizeof(uint64_t) * (d->nlist + 1),
                          cudaMemcpyHostToDevice));
            v.list_offsets = loff;
            uint32_t* ids = ix->alloc<uint32_t>(total);
            uint8_t* codes = ix->alloc<uint8_t>(total * v.code_stride);
            float* lx = ix->alloc<float>(total);
            float* vec = ix->alloc<float>(d->n * v.dim_stride);
            if (total) {
                CK(cudaMemcpy(ids, d->list_ids, sizeof(uint32_t) * total, kind));
                CK(cudaMemset(codes, 0, total * v.code_stride));
                CK(cudaMemcpy2D(codes, v.code_stride, d->list_codes, d->code_stride, d->m, total,
                                kind));
                CK(cudaMemcpy(lx, d->list_lx, sizeof(float) * total, kind));
            }
            if (d->n) {
                if (v.dim_stride != d->dim) {
                    CK(cudaMemset(vec, 0, sizeof(float) * d->n * v.dim_stride));
                    CK(cudaMemcpy2D(vec, sizeof(float) * v.dim_stride, d->vectors,
                                    sizeof(float) * d->dim, sizeof(float) * d->dim, d->n, kind));
                } else {
                    CK(cudaMemcpy(vec, d->vectors, sizeof(float) * d->n * d->dim, kind));
                }
            }
            v.list_ids = ids;
            v.codes = codes;
            v.lx = lx;
            v.vectors = vec;
            float* lr = ix->alloc<float>(d->nlist);
            float* lxmin = ix->alloc<float>(d->nlist);
            float* lxmax = ix->alloc<float>(d->nlist);
            v.list_R = lr;
            v.list_xmin = lxmin;
            v.list_xmax = lxmax;
            ix->d_skipped = ix->alloc<unsigned long long>(1);
            CK(cudaMemset(ix->d_skipped, 0, sizeof(unsigned long long)));
            trim_list_meta_kernel<<<d->nlist, kThreads>>>(v, lr, lxmin, lxmax);
            CK(cudaGetLastError());
            if (mma_k(v.dim) <= kMmaMaxK) {
                const uint32_t K = mma_k(v.dim), ntiles = (d->nlist + kMmaN - 1) / kMmaN;
                ix->coarse_t = ix->alloc<float4>(static_cast<size_t>(ntiles) * (K / 4) * kMmaN);
                ix->cn2 = ix->alloc<float>(d->nlist);
                ix->cn = ix->alloc<float>(d->nlist);
                trim_coarse_tile_kernel<<<ntiles, kThreads>>>(v, K, ix->coarse_t);
                CK(cudaGetLastError());
                trim_coarse_norm_kernel<<<(d->nlist + kThreads - 1) / kThreads, kThreads>>>(v, ix->cn2, ix->cn);
            }
            CK(cudaGetLastError());
            CK(cudaDeviceSynchronize());
        } catch (...) {
            delete ix;
            throw;
        }
        *out = ix;
        return TRIM_OK;
    });
}

extern "C" {

int trim_index_destroy(trim_index_t index) {
    delete index;
    return TRIM_OK;
}

int trim_index_get_info(trim_index_t ix, trim_index_info* info) {
    if (!ix || !info)
        return set_err(TRIM_EINVAL, "trim_index_get_info: null argument");
    info->dim = ix->dev.dim;
    info->m = ix->dev.m;
    info->ksub = ix->dev.ksub;
    info->nlist = ix->dev.nlist;
    info->n = ix->dev.n;
    info->total_entries = ix->total;
    info->id_base = ix->dev.id_base;
    info->max_list_size = ix->max_list;
    info->device_bytes = ix->bytes;
    info->device = ix->device;
    info->range_query_tile = ix->is_group() ? range_flat_qt(ix->parts[0]->dev) : range_flat_qt(ix->dev);
    info->ndevices = ix->is_group() ? static_cast<uint32_t>(ix->parts.size()) : 1u;
    info->shard_mode = ix->shard_mode;
    info->nccl = ix->nccl ? 1u : 0u;
    if (ix->is_group()) {
        info->device_bytes = 0;
        info->max_list_size = 0;
        for (const trim_index* pt : ix->parts) {
            info->device_bytes += pt->bytes;
            info->max_list_size = std::max(info->max_list_size, pt->max_list);
        }
    }
    return TRIM_OK;
}

int trim_index_skip_stats(trim_index_t ix, uint64_t* skipped, int reset) {
    if (!ix || !skipped)
        return set_err(TRIM_EINVAL, "trim_index_skip_stats: null argument");
    if (ix->is_group()) { // summed over the parts
        uint64_t tot = 0;
        for (trim_index* pt : ix->parts) {
            uint64_t v = 0;
            if (int rc = trim_index_skip_stats(pt, &v, reset))
                return rc;
            tot += v;
        }
        *skipped = tot;
        return TRIM_OK;
    }
    return guarded([&]() -> int {
        DeviceGuard g(ix->device);
        CK(cudaDeviceSynchronize());
        unsigned long long v = 0;
        CK(cudaMemcpy(&v, ix->d_skipped, sizeof v, cudaMemcpyDeviceToHost));
        if (reset)
            CK(cudaMemset(ix->d_skipped, 0, sizeof v));
        *skipped = v;
        return TRIM_OK;
    });
}

int trim_probe_launches(trim_index_t ix, uint32_t nprobe, uint32_t* launches) {
    if (!ix || !launches)
        return set_err(TRIM_EINVAL, "trim_probe_launches: null argument");
    if (ix->is_group())
        ix = ix->parts[0];
    const uint32_t np = std::min(nprobe, ix->dev.nlist);
    *launches = (ix->dev.nlist == 1 || np == 0) ? 0u : (probe_uses_mma(ix, np) ? 2u : 1u);
    return TRIM_OK;
}

int trim_search_knn(trim_index_t ix, const float* queries, uint64_t nq, uint32_t k,
                    uint32_t nprobe, float gamma, uint32_t* ids_out, float* dist_out,
                    trim_counters* counters_out) {
    if (!ix)
        return set_err(TRIM_EINVAL, "search_trim_ivf_knn: null index");
    if (int rc = validate_knn(k, gamma))
        return rc;
    if (nq == 0)
        return TRIM_OK;
    if (ix->is_group())
        return guarded([&]() -> int {
            return group_search_knn(ix, queries, nq, k, nprobe, gamma, ids_out, dist_out, counters_out);
        });
    return guarded([&]() -> int {
        DeviceGuard g(ix->device);
        cudaStream_t st = thread_stream(ix->device);
        DevBuf d_q = upload_queries(ix, queries, nq, cudaMemcpyHostToDevice, st);
        DevBuf d_ids(sizeof(uint32_t) * nq * k, st), d_dist(sizeof(float) * nq * k, st);
        DevBuf d_ct(sizeof(unsigned long long) * nq * 6, st), d_status(sizeof(uint32_t), st);
        CK(cudaMemsetAsync(d_status.p, 0, sizeof(uint32_t), st));
        if (int rc = knn_device(ix, d_q.as<float>(), nq, k, nprobe, gamma, d_ids.as<uint32_t>(),
                                d_dist.as<float>(), d_ct.as<unsigned long long>(),
                                d_status.as<uint32_t>(), st))
            return rc;
        uint32_t* status_h = pinned_word(); // pinned: the readback stays an async copy
        CK(cudaMemcpyAsync(ids_out, d_ids.p, sizeof(uint32_t) * nq * k, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(dist_out, d_dist.p, sizeof(float) * nq * k, cudaMemcpyDeviceToHost, st));
        if (counters_out)
            CK(cudaMemcpyAsync(counters_out, d_ct.p, sizeof(trim_counters) * nq,
                               cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(status_h, d_status.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (*status_h & 1u)
            return set_err(TRIM_EINVAL, "search_trim_ivf_knn: k exceeds probed vectors");
        return TRIM_OK;
    });
}

int trim_search_knn_device(trim_index_t ix, const float* d_queries, uint64_t nq, uint32_t k,
                           uint32_t nprobe, float gamma, uint32_t* d_ids, float* d_dist,
                           trim_counters* d_counters, uint32_t* d_status, void* stream) {
    if (!ix)
        return set_err(TRIM_EINVAL, "search_trim_ivf_knn: null index");
    if (int rc = validate_knn(k, gamma))
        return rc;
    if (nq == 0)
        return TRIM_OK;
    if (ix->is_group())
        return guarded([&]() -> int {
            return group_search_knn_device(ix, d_queries, nq, k, nprobe, gamma, d_ids, d_dist, d_counters, d_status,
                                           stream);
        });
    return guarded([&]() -> int {
        DeviceGuard g(ix->device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (ix->dev.dim_stride != ix->dev.dim) {
            DevBuf d_q = upload_queries(ix, d_queries, nq, cudaMemcpyDeviceToDevice, st);
            return knn_device(ix, d_q.as<float>(), nq, k, nprobe, gamma, d_ids, d_dist,
                              reinterpret_cast<unsigned long long*>(d_counters), d_status, st);
        }
        return knn_device(ix, d_queries, nq, k, nprobe, gamma, d_ids, d_dist,
                          reinterpret_cast<unsigned long long*>(d_counters), d_status, st);
    });
}

int trim_probe_device(trim_index_t ix, const float* d_queries, uint64_t nq, uint32_t nprobe,
                      uint32_t* d_lists, void* stream) {
    if (!ix)
        return set_err(TRIM_EINVAL, "probe_order: null index");
    if (nq == 0 || nprobe == 0)
        return TRIM_OK;
    if (ix->is_group()) // the coarse quantizer is replicated: the home part's probe order
        ix = ix->parts[0];
    if (ix->dev.dim_stride != ix->dev.dim)
        return set_err(TRIM_EINVAL, "trim_probe_device: dim must be a multiple of 4 (use trim_probe)");
    return guarded([&]() -> int {
        DeviceGuard g(ix->device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const uint32_t np = std::min(nprobe, ix->dev.nlist);
        if (ix->dev.nlist == 1) {
            CK(cudaMemsetAsync(d_lists, 0, sizeof(uint32_t) * nq * np, st));
            return TRIM_OK;
        }
        launch_probe(ix, d_queries, nq, np, d_lists, st);
        return TRIM_OK;
    });
}

int trim_search_knn_preassigned_device(trim_index_t ix, const float* d_queries, uint64_t nq,
                                       uint32_t k, const uint32_t* d_lists, uint32_t np, float gamma,
                                       uint32_t* d_ids, float* d_dist, trim_counters* d_counters,
                                       uint32_t* d_status, void* stream) {
    if (!ix)
        return set_err(TRIM_EINVAL, "search_trim_ivf_knn: null index");
    if (int rc = validate_knn(k, gamma))
        return rc;
    if (ix->is_group())
        return set_err(TRIM_EINVAL, "trim_search_knn_preassigned_device: takes a single-device index "
                                    "(a multi-device index: trim_search_knn_device)");
    if (np > ix->dev.nlist)
        return set_err(TRIM_EINVAL, "search_trim_ivf_knn: np > nlist");
    if (ix->dev.dim_stride != ix->dev.dim)
        return set_err(TRIM_EINVAL,
                       "trim_search_knn_preassigned_device: dim must be a multiple of 4");
    return guarded([&]() -> int {
        DeviceGuard g(ix->device);
        return knn_launch(ix, d_queries, nq, k, np, np ? d_lists : nullptr, gamma, d_ids, d_dist,
                          reinterpret_cast<unsigned long long*>(d_counters), d_status,
                          static_cast<cudaStream_t>(stream));
    });
}

int trim_search_range(trim_index_t ix, const float* queries, uint64_t nq, const float* radius,
                      uint32_t nprobe, float gamma, uint64_t* offsets_out, uint32_t** ids_out,
                      float** dist_out, trim_counters* counters_out) {
    if (!ix || !offsets_out || !ids_out || !dist_out)
        return set_err(TRIM_EINVAL, "search_trim_ivf_range: null argument");
    *ids_out = nullptr;
    *dist_out = nullptr;
    for (uint64_t i = 0; i < nq; ++i)
        if (radius[i] < 0.0f)
            return set_err(TRIM_EINVAL, "search_trim_ivf_range: negative radius");
    if (!(gamma >= 0.0f))
        return set_err(TRIM_EINVAL, "search_trim_ivf_range: uncalibrated pruning profile");
    offsets_out[0] = 0;
    if (nq == 0) {
        *ids_out = static_cast<uint32_t*>(std::malloc(4));
        *dist_out = static_cast<float*>(std::malloc(4));
        return TRIM_OK;
    }
    if (ix->is_group())
        return guarded([&]() -> int {
            return group_search_range(ix, queries, nq, radius, nprobe, gamma, offsets_out, ids_out, dist_out,
                                      counters_out);
        });
    return guarded([&]() -> int {
        DeviceGuard g(ix->device);
        cudaStream_t st = thread_stream(ix->device);
        DevBuf d_q = upload_queries(ix, queries, nq, cudaMemcpyHostToDevice, st);
        // ivf.hpp:315: radius_sq = radius * radius in fp32
        std::vector<float> r2(nq);
        for (uint64_t i = 0; i < nq; ++i)
            r2[i] = radius[i] * radius[i];
        DevBuf d_r2(sizeof(float) * nq, st);
        CK(cudaMemcpyAsync(d_r2.p, r2.data(), sizeof(float) * nq, cudaMemcpyHostToDevice, st));
        DevBuf d_probe;
        const uint32_t np = run_probe(ix, d_q.as<float>(), nq, nprobe, d_probe, st);
        const size_t smem = range_smem_bytes(dispatch_m(ix->dev), ix->dev.m, ix->dev.dim_stride, np);
        if (smem > kSmemLimit)
            return set_err(TRIM_EINVAL,
                           "search_trim_ivf_range: per-query state (%zu B) exceeds 227 KB", smem);
        DevBuf d_cnt(sizeof(unsigned int) * nq, st), d_dc(sizeof(unsigned long long) * nq, st),
            d_eval(sizeof(unsigned long long) * nq, st);
        uint32_t cap = 1024;
        std::vector<unsigned int> cnt(nq);
        DevBuf d_keys;
        for (int attempt = 0; attempt < 2; ++attempt) {
            d_keys = DevBuf(sizeof(unsigned long long) * nq * cap, st);
            CK(cudaMemsetAsync(d_cnt.p, 0, sizeof(unsigned int) * nq, st));
            CK(cudaMemsetAsync(d_dc.p, 0, sizeof(unsigned long long) * nq, st));
            CK(cudaMemsetAsync(d_eval.p, 0, sizeof(unsigned long long) * nq, st));
            range_launch(ix, d_q.as<float>(), nq, d_r2.as<float>(), np, d_probe.p ? d_probe.as<uint32_t>() : nullptr,
                         gamma, cap, d_keys.as<unsigned long long>(), d_cnt.as<unsigned int>(),
                         d_dc.as<unsigned long long>(), d_eval.as<unsigned long long>(), st);
            CK(cudaMemcpyAsync(cnt.data(), d_cnt.p, sizeof(unsigned int) * nq,
                               cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            const unsigned int mx = *std::max_element(cnt.begin(), cnt.end());
            if (mx <= cap)
                break;
            cap = mx;
        }
        // per-query sort by (dist, id) — ivf.hpp:341
        std::vector<uint64_t> beg(nq), endv(nq);
        uint64_t tot = 0;
        for (uint64_t i = 0; i < nq; ++i) {
            beg[i] = i * cap;
            endv[i] = i * cap + cnt[i];
            offsets_out[i] = tot;
            tot += cnt[i];
        }
        offsets_out[nq] = tot;
        DevBuf d_beg(sizeof(uint64_t) * nq, st), d_end(sizeof(uint64_t) * nq, st),
            d_sorted(sizeof(unsigned long long) * nq * cap, st);
        CK(cudaMemcpyAsync(d_beg.p, beg.data(), sizeof(uint64_t) * nq, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(d_end.p, endv.data(), sizeof(uint64_t) * nq, cudaMemcpyHostToDevice, st));
        size_t tmp_bytes = 0;
        CK(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp_bytes, d_keys.as<unsigned long long>(),
                                              d_sorted.as<unsigned long long>(),
                                              static_cast<int64_t>(nq * cap), static_cast<int64_t>(nq),
                                              d_beg.as<uint64_t>(), d_end.as<uint64_t>(), st));
        DevBuf d_tmp(tmp_bytes, st);
        CK(cub::DeviceSegmentedSort::SortKeys(d_tmp.p, tmp_bytes, d_keys.as<unsigned long long>(),
                                              d_sorted.as<unsigned long long>(),
                                              static_cast<int64_t>(nq * cap), static_cast<int64_t>(nq),
                                              d_beg.as<uint64_t>(), d_end.as<uint64_t>(), st));
        DevBuf d_offs(sizeof(uint64_t) * (nq + 1), st);
        CK(cudaMemcpyAsync(d_offs.p, offsets_out, sizeof(uint64_t) * (nq + 1), cudaMemcpyHostToDevice,
                           st));
        DevBuf d_ids(sizeof(uint32_t) * std::max<uint64_t>(tot, 1), st),
            d_dist(sizeof(float) * std::max<uint64_t>(tot, 1), st);
        trim_unpack_keys_kernel<<<static_cast<unsigned>(nq), 128, 0, st>>>(
            d_sorted.as<unsigned long long>(), cap, d_offs.as<uint64_t>(), nq, d_ids.as<uint32_t>(),
            d_dist.as<float>());
        CK(cudaGetLastError());
        auto* hid = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * std::max<uint64_t>(tot, 1)));
        auto* hd = static_cast<float*>(std::malloc(sizeof(float) * std::max<uint64_t>(tot, 1)));
        if (!hid || !hd) {
            std::free(hid);
            std::free(hd);
            return set_err(TRIM_ENOMEM, "search_trim_ivf_range: result allocation failed");
        }
        std::vector<unsigned long long> dc(nq), ev(nq);
        CK(cudaMemcpyAsync(hid, d_ids.p, sizeof(uint32_t) * tot, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hd, d_dist.p, sizeof(float) * tot, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(dc.data(), d_dc.p, sizeof(unsigned long long) * nq, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(ev.data(), d_eval.p, sizeof(unsigned long long) * nq, cudaMemcpyDeviceToHost,
                           st));
        cudaError_t se = cudaStreamSynchronize(st);
        if (se != cudaSuccess) {
            std::free(hid);
            std::free(hd);
            CK(se);
        }
        if (counters_out) {
            for (uint64_t i = 0; i < nq; ++i) {
                trim_counters& c = counters_out[i];
                c.evaluated = ev[i];
                c.edc = ev[i];
                c.dc = dc[i];
                c.pruned = ev[i] - dc[i];
                c.hops = 0;
                c.coarse_dc = ix->dev.nlist;
            }
        }
        *ids_out = hid;
        *dist_out = hd;
        return TRIM_OK;
    });
}

int trim_search_range_device(trim_index_t ix, const float* d_queries, uint64_t nq, const float* d_radius,
                             uint32_t nprobe, float gamma, uint32_t cap, uint32_t* d_counts, uint32_t* d_ids,
                             float* d_dist, trim_counters* d_counters, uint32_t* d_status, void* stream) {
    if (!ix || (nq && (!d_queries || !d_radius || !d_counts || !d_ids || !d_dist)))
        return set_err(TRIM_EINVAL, "search_trim_ivf_range: null argument");
    if (!(gamma >= 0.0f))
        return set_err(TRIM_EINVAL, "search_trim_ivf_range: uncalibrated pruning profile");
    if (cap == 0)
        return set_err(TRIM_EINVAL, "trim_search_range_device: cap must be positive");
    if (ix->is_group())
        return set_err(TRIM_EINVAL, "trim_search_range_device: takes a single-device index "
                                    "(a multi-device index: trim_search_range)");
    if (ix->dev.dim_stride != ix->dev.dim)
        return set_err(TRIM_EINVAL, "trim_search_range_device: dim must be a multiple of 4");
    if (nq == 0)
        return TRIM_OK;
    return guarded([&]() -> int {
        DeviceGuard g(ix->device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const unsigned g1 = static_cast<unsigned>((nq + 255) / 256);
        DevBuf d_r2(sizeof(float) * nq, st);
        trim_range_r2_kernel<<<g1, 256, 0, st>>>(d_radius, nq, d_r2.as<float>(), d_status);
        CK(cudaGetLastError());
        DevBuf d_probe;
        const uint32_t np = run_probe(ix, d_queries, nq, nprobe, d_probe, st);
        if (np == 0)
            return set_err(TRIM_EINVAL, "search_trim_ivf_range: nprobe must be positive");
        DevBuf d_cnt(sizeof(unsigned int) * nq, st), d_dc(sizeof(unsigned long long) * nq, st),
            d_eval(sizeof(unsigned long long) * nq, st), d_keys(sizeof(unsigned long long) * nq * cap, st);
        CK(cudaMemsetAsync(d_cnt.p, 0, sizeof(unsigned int) * nq, st));
        CK(cudaMemsetAsync(d_dc.p, 0, sizeof(unsigned long long) * nq, st));
        CK(cudaMemsetAsync(d_eval.p, 0, sizeof(unsigned long long) * nq, st));
        range_launch(ix, d_queries, nq, d_r2.as<float>(), np, d_probe.p ? d_probe.as<uint32_t>() : nullptr, gamma,
                     cap, d_keys.as<unsigned long long>(), d_cnt.as<unsigned int>(), d_dc.as<unsigned long long>(),
                     d_eval.as<unsigned long long>(), st);
        DevBuf d_beg(sizeof(uint64_t) * nq, st), d_end(sizeof(uint64_t) * nq, st),
            d_sorted(sizeof(unsigned long long) * nq * cap, st);
        trim_range_seg_kernel<<<g1, 256, 0, st>>>(d_cnt.as<unsigned int>(), nq, cap, d_beg.as<uint64_t>(),
                                                  d_end.as<uint64_t>(), d_status);
        CK(cudaGetLastError());
        size_t tmp_bytes = 0;
        CK(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp_bytes, d_keys.as<unsigned long long>(),
                                              d_sorted.as<unsigned long long>(),
                                              static_cast<int64_t>(nq * cap), static_cast<int64_t>(nq),
                                              d_beg.as<uint64_t>(), d_end.as<uint64_t>(), st));
        DevBuf d_tmp(tmp_bytes, st);
        CK(cub::DeviceSegmentedSort::SortKeys(d_tmp.p, tmp_bytes, d_keys.as<unsigned long long>(),
                                              d_sorted.as<unsigned long long>(),
                                              static_cast<int64_t>(nq * cap), static_cast<int64_t>(nq),
                                              d_beg.as<uint64_t>(), d_end.as<uint64_t>(), st));
        trim_range_finish_kernel<<<static_cast<unsigned>(nq), 128, 0, st>>>(
            d_sorted.as<unsigned long long>(), d_cnt.as<unsigned int>(), d_dc.as<unsigned long long>(),
            d_eval.as<unsigned long long>(), nq, cap, ix->dev.nlist, d_counts, d_ids, d_dist,
            reinterpret_cast<unsigned long long*>(d_counters));
        CK(cudaGetLastError());
        return TRIM_OK;
    });
}

int trim_ground_truth_knn(trim_index_t ix, const float* queries, uint64_t nq, uint32_t k, uint32_t* ids_out,
                          float* dist_out) {
    if (!ix || (nq && (!queries || !ids_out || !dist_out)))
        return set_err(TRIM_EINVAL, "ground_truth_knn: null argument");
    if (k == 0 || k > ix->dev.n)
        return set_err(TRIM_EINVAL, "brute_force_knn: k out of range");
    if (k > kGtCap)
        return set_err(TRIM_EINVAL, "ground_truth_knn: k > 4096 is not supported by the GPU selection");
    if (ix->is_group()) {
        if (ix->shard_mode != TRIM_SHARD_REPLICAS)
            return set_err(TRIM_EINVAL, "ground_truth_knn: needs every row on one device (single or replicas index)");
        ix = ix->parts[0];
    }
    if (nq == 0)
        return TRIM_OK;
    return guarded([&]() -> int {
        DeviceGuard g(ix->device);
        cudaStream_t st = thread_stream(ix->device);
        ensure_flat_tiles(ix);
        const DevIndex& v = ix->dev;
        DevBuf d_q = upload_queries(ix, queries, nq, cudaMemcpyHostToDevice, st);
        const uint32_t K = flat_kpad(v.dim);
        const uint64_t ld = (v.n + kMmaN - 1) / kMmaN * kMmaN, nrt = ld / kMmaN;
        const uint64_t slice = std::max<uint64_t>(kMmaM, (4ull << 30) / (ld * 4) / kMmaM * kMmaM);
        DevBuf d_ids(sizeof(uint32_t) * nq * k, st), d_dist(sizeof(float) * nq * k, st);
        CK(cudaFuncSetAttribute(trim_flat_dist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(flat_mma_smem())));
        CK(cudaFuncSetAttribute(trim_gt_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(gt_smem(v.dim_stride))));
        for (uint64_t b = 0; b < nq; b += slice) {
            const uint64_t nb = std::min<uint64_t>(slice, nq - b);
            const uint64_t nqt = (nb + kMmaM - 1) / kMmaM;
            const float* qb = d_q.as<float>() + b * v.dim_stride;
            DevBuf qtiles(sizeof(float4) * nqt * (K / kFlatKB) * 8 * kMmaM, st), qn2(sizeof(float) * nb, st);
            trim_flat_tile_kernel<<<static_cast<unsigned>(nqt), kThreads, 0, st>>>(qb, nb, v.dim_stride, v.dim, K,
                                                                                   qtiles.as<float4>());
            trim_query_norm_kernel<<<static_cast<unsigned>((nb + 255) / 256), 256, 0, st>>>(qb, nb, v.dim_stride,
                                                                                            v.dim, qn2.as<float>());
            DevBuf dap(sizeof(float) * nb * ld, st), scratch(sizeof(float) * nb * ld, st);
            launch_flat_dist(qtiles.as<float4>(), qn2.as<float>(), nb, nqt, ix, K, dap.as<float>(), ld, nrt, st);
            trim_gt_select_kernel<<<static_cast<unsigned>(nb), kGtThreads, gt_smem(v.dim_stride), st>>>(
                v, qb, nb, k, dap.as<float>(), ld, ix->xn, ix->xn2, scratch.as<float>(), d_ids.as<uint32_t>() + b * k,
                d_dist.as<float>() + b * k);
            CK(cudaGetLastError());
        }
        CK(cudaMemcpyAsync(ids_out, d_ids.p, sizeof(uint32_t) * nq * k, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(dist_out, d_dist.p, sizeof(float) * nq * k, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return TRIM_OK;
    });
}

int trim_search_baseline_ivfpq(trim_index_t ix, const float* queries, uint64_t nq, uint32_t k,
                               uint32_t nprobe, uint32_t k_prime, uint32_t* ids_out,
                               float* dist_out, trim_counters* counters_out) {
    if (!ix)
        return set_err(TRIM_EINVAL, "search_baseline_ivfpq: null index");
    if (k == 0 || k > k_prime)
        return set_err(TRIM_EINVAL, "search_baseline_ivfpq: need 1 <= k <= k_prime");
    if (nprobe == 0)
        return set_err(TRIM_EINVAL, "search_baseline_ivfpq: nprobe must be positive");
    if (nq == 0)
        return TRIM_OK;
    if (ix->is_group())
        return guarded([&]() -> int {
            return group_search_baseline(ix, queries, nq, k, nprobe, k_prime, ids_out, dist_out, counters_out);
        });
    return guarded([&]() -> int {
        DeviceGuard g(ix->device);
        cudaStream_t st = thread_stream(ix->device);
        DevBuf d_q = upload_queries(ix, queries, nq, cudaMemcpyHostToDevice, st);
        DevBuf d_probe;
        const uint32_t np = run_probe(ix, d_q.as<float>(), nq, nprobe, d_probe, st);
        return baseline_device(ix, d_q.as<float>(), nq, k, np, d_probe.as<uint32_t>(), k_prime,
                               ids_out, dist_out, counters_out, st);
    });
}

int trim_build_lut(trim_index_t ix, const float* queries, uint64_t nq, float* lut_out) {
    if (!ix)
        return set_err(TRIM_EINVAL, "build_distance_table: null index");
    if (nq == 0)
        return TRIM_OK;
    if (ix->is_group()) // the codebook is replicated
        ix = ix->parts[0];
    return guarded([&]() -> int {
        DeviceGuard g(ix->device);
        cudaStream_t st = thread_stream(ix->device);
        DevBuf d_q = upload_queries(ix, queries, nq, cudaMemcpyHostToDevice, st);
        DevBuf d_lut(sizeof(float) * nq * ix->dev.m * ix->dev.ksub, st);
        trim_lut_kernel<<<static_cast<unsigned>(nq), kThreads, sizeof(float) * ix->dev.dim_stride, st>>>(
            ix->dev, d_q.as<float>(), d_lut.as<float>());
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(lut_out, d_lut.p, sizeof(float) * nq * ix->dev.m * ix->dev.ksub,
                           cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return TRIM_OK;
    });
}

int trim_probe(trim_index_t ix, const float* queries, uint64_t nq, uint32_t nprobe,
               uint32_t* lists_out) {
    if (!ix)
        return set_err(TRIM_EINVAL, "probe_order: null index");
    if (nq == 0)
        return TRIM_OK;
    if (ix->is_group()) // the coarse quantizer is replicated
        ix = ix->parts[0];
    return guarded([&]() -> int {
        DeviceGuard g(ix->device);
        cudaStream_t st = thread_stream(ix->device);
        DevBuf d_q = upload_queries(ix, queries, nq, cudaMemcpyHostToDevice, st);
        DevBuf d_probe;
        const uint32_t np = run_probe(ix, d_q.as<float>(), nq, nprobe, d_probe, st);
        if (np == 0)
            return TRIM_OK;
        if (!d_probe.p) { // nlist == 1
            for (uint64_t i = 0; i < nq; ++i)
                lists_out[i] = 0;
            CK(cudaStreamSynchronize(st));
            return TRIM_OK;
        }
        CK(cudaMemcpyAsync(lists_out, d_probe.p, sizeof(uint32_t) * nq * np, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return TRIM_OK;
    });
}

int trim_merge_topk_device(const float* d_dist, const uint32_t* d_ids, uint32_t nshards,
                           uint64_t nq, uint32_t k, float* d_dist_out, uint32_t* d_ids_out,
                           int device, void* stream) {
    if (nshards == 0 || k == 0)
        return set_err(TRIM_EINVAL, "trim_merge_topk_device: need nshards >= 1 and k >= 1");
    if (static_cast<uint64_t>(nshards) * k > 16384)
        return set_err(TRIM_EINVAL, "trim_merge_topk_device: nshards*k > 16384");
    if (nq == 0)
        return TRIM_OK;
    return guarded([&]() -> int {
        DeviceGuard g(device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const uint32_t n2 = pow2_at_least(nshards * k);
        const size_t smem = sizeof(uint64_t) * n2;
        CK(cudaFuncSetAttribute(trim_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
        trim_merge_kernel<<<static_cast<unsigned>(nq), kThreads, smem, st>>>(
            d_dist, d_ids, nshards, nq, k, n2, d_dist_out, d_ids_out);
        CK(cudaGetLastError());
        return TRIM_OK;
    });
}

// ------------------------------------------------------------ graph search
// (include/trim_gpu.h: trim_graph_*; graph/search.hpp:188-347)
int trim_graph_create(const trim_graph_desc* d, trim_graph_t* out) {
    if (!d || !out)
        return set_err(TRIM_EINVAL, "trim_graph_create: null argument");
    *out = nullptr;
    if (d->n == 0)
        return set_err(TRIM_EINVAL, "trim_graph_create: empty graph");
    if (d->n >= 0xFFFFFFFFull)
        return set_err(TRIM_EINVAL, "trim_graph_create: more than 2^32-2 nodes");
    if (d->dim == 0 || d->m == 0 || d->ksub == 0 || d->ksub > 256 || d->levels == 0)
        return set_err(TRIM_EINVAL, "trim_graph_create: need dim, m, levels >= 1 and 1 <= ksub <= 256");
    if (!d->sub_dims || !d->centroids || !d->codes || !d->lx || !d->vectors || !d->offsets ||
        !d->nbr_base || (d->total_nbrs && !d->nbrs))
        return set_err(TRIM_EINVAL, "trim_graph_create: null array in descriptor");
    if (d->code_stride < d->m)
        return set_err(TRIM_EINVAL, "trim_graph_create: code_stride < m");
    if (d->entry >= d->n)
        return set_err(TRIM_EDATA, "graph entry %u outside [0, %llu)", d->entry, (unsigned long long)d->n);
    if (int rc = check_device_present())
        return rc;
    const bool host = d->memory == TRIM_MEM_HOST;
    const cudaMemcpyKind kind = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    return guarded([&]() -> int {
        DeviceGuard dg(d->device);
        const uint64_t n = d->n, L = d->levels;
        std::vector<uint32_t> sub(d->m);
        CK(cudaMemcpy(sub.data(), d->sub_dims, sizeof(uint32_t) * d->m,
                      host ? cudaMemcpyHostToHost : cudaMemcpyDeviceToHost));
        std::vector<uint32_t> suboff(d->m);
        uint64_t sdsum = 0;
        for (uint32_t j = 0; j < d->m; ++j) {
            suboff[j] = static_cast<uint32_t>(sdsum);
            sdsum += sub[j];
        }
        if (sdsum != d->dim)
            return set_err(TRIM_EDATA, "codebook sub_dims do not sum to dim");
        if (host) { // graph/hnsw.hpp:58-83 invariants: monotone CSR, ids < count
            for (uint64_t l = 0; l < L; ++l) {
                const uint64_t* o = d->offsets + l * (n + 1);
                if (o[0] != 0)
                    return set_err(TRIM_EDATA, "graph level %llu offsets must start at 0", (unsigned long long)l);
                for (uint64_t i = 0; i < n; ++i)
                    if (o[i + 1] < o[i])
                        return set_err(TRIM_EDATA, "graph level %llu offsets are not monotone", (unsigned long long)l);
                if (d->nbr_base[l] + o[n] > d->total_nbrs)
                    return set_err(TRIM_EDATA, "graph level %llu adjacency exceeds total_nbrs", (unsigned long long)l);
                for (uint64_t e = 0; e < o[n]; ++e)
                    if (d->nbrs[d->nbr_base[l] + e] >= n)
                        return set_err(TRIM_EDATA, "graph neighbour id %u outside [0, %llu)",
                                       d->nbrs[d->nbr_base[l] + e], (unsigned long long)n);
            }
        }
        auto* gr = new trim_graph;
        gr->device = d->device;
        try {
            DevIndex& v = gr->dev.ix;
            v.dim = d->dim;
            v.dim_stride = round_up(d->dim, 4);
            v.m = d->m;
            v.ksub = d->ksub;
            v.code_stride = round_up(d->m, 16);
            v.nlist = 0;
            v.sd_uniform = sub[0];
            for (uint32_t j = 1; j < d->m; ++j)
                if (sub[j] != sub[0])
                    v.sd_uniform = 0;
            v.n = n;
            v.id_base = 0;
            uint32_t* dsub = gr->alloc<uint32_t>(d->m);
            uint32_t* doff = gr->alloc<uint32_t>(d->m);
            CK(cudaMemcpy(dsub, sub.data(), sizeof(uint32_t) * d->m, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(doff, suboff.data(), sizeof(uint32_t) * d->m, cudaMemcpyHostToDevice));
            v.sub_dims = dsub;
            v.sub_offsets = doff;
            float* cent = gr->alloc<float>(static_cast<size_t>(d->ksub) * d->dim);
            CK(cudaMemcpy(cent, d->centroids, sizeof(float) * d->ksub * d->dim, kind));
            v.centroids = cent;
            v.centroids_t = centroids_code_major(gr->alloc<float>(static_cast<size_t>(d->ksub) * d->dim), cent,
                                                 d->ksub, d->dim, sub, suboff);
            uint8_t* codes = gr->alloc<uint8_t>(n * v.code_stride);
            CK(cudaMemset(codes, 0, n * v.code_stride));
            CK(cudaMemcpy2D(codes, v.code_stride, d->codes, d->code_stride, d->m, n, kind));
            v.codes = codes;
            float* lx = gr->alloc<float>(n);
            CK(cudaMemcpy(lx, d->lx, sizeof(float) * n, kind));
            v.lx = lx;
            float* vec = gr->alloc<float>(n * v.dim_stride);
            CK(cudaMemset(vec, 0, sizeof(float) * n * v.dim_stride));
            CK(cudaMemcpy2D(vec, sizeof(float) * v.dim_stride, d->vectors, sizeof(float) * d->dim,
                            sizeof(float) * d->dim, n, kind));
            v.vectors = vec;
            uint64_t* offs = gr->alloc<uint64_t>(L * (n + 1));
            CK(cudaMemcpy(offs, d->offsets, sizeof(uint64_t) * L * (n + 1), kind));
            uint64_t* base = gr->alloc<uint64_t>(L);
            CK(cudaMemcpy(base, d->nbr_base, sizeof(uint64_t) * L, kind));
            uint32_t* nb = gr->alloc<uint32_t>(std::max<uint64_t>(d->total_nbrs, 1));
            if (d->total_nbrs)
                CK(cudaMemcpy(nb, d->nbrs, sizeof(uint32_t) * d->total_nbrs, kind));
            gr->dev.levels = d->levels;
            gr->dev.entry = d->entry;
            gr->dev.offsets = offs;
            gr->dev.nbr_base = base;
            gr->dev.nbrs = nb;
            CK(cudaDeviceSynchronize());
        } catch (...) {
            delete gr;
            throw;
        }
        *out = gr;
        return TRIM_OK;
    });
}

int trim_graph_destroy(trim_graph_t graph) {
    delete graph;
    return TRIM_OK;
}

int trim_graph_search_knn(trim_graph_t gr, const float* queries, uint64_t nq, uint32_t k, uint32_t ef,
                          float gamma, uint32_t* ids_out, float* dist_out, trim_counters* counters_out) {
    if (!gr || (nq && (!queries || !ids_out || !dist_out)))
        return set_err(TRIM_EINVAL, "search_trim_knn: null argument");
    if (k == 0 || k > ef)
        return set_err(TRIM_EINVAL, "search_trim_knn: need 1 <= k <= ef");
    if (!(gamma >= 0.0f))
        return set_err(TRIM_EINVAL, "search_trim_knn: uncalibrated pruning profile");
    if (ef > 1024)
        return set_err(TRIM_EINVAL, "search_trim_knn: ef > 1024 is not supported on the GPU path");
    if (nq == 0)
        return TRIM_OK;
    return guarded([&]() -> int {
        DeviceGuard g(gr->device);
        cudaStream_t st = thread_stream(gr->device);
        DevBuf d_q = graph_upload_queries(gr, queries, nq, st);
        DevBuf d_ids(sizeof(uint32_t) * nq * k, st), d_dist(sizeof(float) * nq * k, st),
            d_ct(sizeof(unsigned long long) * nq * 6, st);
        graph_run(gr, d_q.as<float>(), nq, k, ef, gamma, false, nullptr, d_ids.as<uint32_t>(),
                  d_dist.as<float>(), nullptr, 0, nullptr, d_ct.as<unsigned long long>(), st);
        std::vector<unsigned long long> ct(nq * 6);
        CK(cudaMemcpyAsync(ids_out, d_ids.p, sizeof(uint32_t) * nq * k, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(dist_out, d_dist.p, sizeof(float) * nq * k, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(ct.data(), d_ct.p, sizeof(unsigned long long) * nq * 6, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (counters_out)
            put_counters_host(counters_out, ct, nq);
        return TRIM_OK;
    });
}

int trim_graph_search_knn_device(trim_graph_t gr, const float* d_queries, uint64_t nq, uint32_t k,
                                 uint32_t ef, float gamma, uint32_t* d_ids, float* d_dist,
                                 unsigned long long* d_counters, void* stream) {
    if (!gr || (nq && (!d_queries || !d_ids || !d_dist || !d_counters)))
        return set_err(TRIM_EINVAL, "search_trim_knn: null argument");
    if (k == 0 || k > ef)
        return set_err(TRIM_EINVAL, "search_trim_knn: need 1 <= k <= ef");
    if (!(gamma >= 0.0f))
        return set_err(TRIM_EINVAL, "search_trim_knn: uncalibrated pruning profile");
    if (ef > 1024)
        return set_err(TRIM_EINVAL, "search_trim_knn: ef > 1024 is not supported on the GPU path");
    if (nq == 0)
        return TRIM_OK;
    return guarded([&]() -> int {
        DeviceGuard g(gr->device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const uint32_t dim = gr->dev.ix.dim, ds = gr->dev.ix.dim_stride;
        DevBuf d_pad;
        const float* q = d_queries;
        if (ds != dim) {
            d_pad = DevBuf(sizeof(float) * nq * ds, st);
            CK(cudaMemsetAsync(d_pad.p, 0, sizeof(float) * nq * ds, st));
            CK(cudaMemcpy2DAsync(d_pad.p, sizeof(float) * ds, d_queries, sizeof(float) * dim, sizeof(float) * dim,
                                 nq, cudaMemcpyDeviceToDevice, st));
            q = d_pad.as<float>();
        }
        graph_run(gr, q, nq, k, ef, gamma, false, nullptr, d_ids, d_dist, nullptr, 0, nullptr, d_counters, st);
        return TRIM_OK;
    });
}

int trim_graph_search_range(trim_graph_t gr, const float* queries, uint64_t nq, const float* radius,
                            uint32_t ef, float gamma, uint64_t* offsets_out, uint32_t** ids_out,
                            float** dist_out, trim_counters* counters_out) {
    if (!gr || !offsets_out || !ids_out || !dist_out || (nq && (!queries || !radius)))
        return set_err(TRIM_EINVAL, "search_trim_range: null argument");
    *ids_out = nullptr;
    *dist_out = nullptr;
    for (uint64_t i = 0; i < nq; ++i)
        if (radius[i] < 0.0f)
            return set_err(TRIM_EINVAL, "search_trim_range: negative radius");
    if (!(gamma >= 0.0f))
        return set_err(TRIM_EINVAL, "search_trim_range: uncalibrated pruning profile");
    if (ef == 0 || ef > 1024)
        return set_err(TRIM_EINVAL, "search_trim_range: the GPU path needs 1 <= ef <= 1024");
    offsets_out[0] = 0;
    if (nq == 0) {
        *ids_out = static_cast<uint32_t*>(std::malloc(4));
        *dist_out = static_cast<float*>(std::malloc(4));
        return TRIM_OK;
    }
    return guarded([&]() -> int {
        DeviceGuard g(gr->device);
        cudaStream_t st = thread_stream(gr->device);
        DevBuf d_q = graph_upload_queries(gr, queries, nq, st);
        std::vector<float> r2(nq); // search.hpp:278: radius * radius in fp32
        for (uint64_t i = 0; i < nq; ++i)
            r2[i] = radius[i] * radius[i];
        DevBuf d_r2(sizeof(float) * nq, st), d_counts(sizeof(unsigned long long) * nq, st),
            d_ct(sizeof(unsigned long long) * nq * 6, st);
        CK(cudaMemcpyAsync(d_r2.p, r2.data(), sizeof(float) * nq, cudaMemcpyHostToDevice, st));
        uint64_t cap = std::min<uint64_t>(gr->dev.ix.n, 1024);
        std::vector<unsigned long long> cnt(nq);
        DevBuf d_pool;
        for (int attempt = 0; attempt < 2; ++attempt) {
            d_pool = DevBuf(sizeof(unsigned long long) * nq * cap, st);
            graph_run(gr, d_q.as<float>(), nq, 0, ef, gamma, true, d_r2.as<float>(), nullptr, nullptr,
                      d_pool.as<unsigned long long>(), cap, d_counts.as<unsigned long long>(),
                      d_ct.as<unsigned long long>(), st);
            CK(cudaMemcpyAsync(cnt.data(), d_counts.p, sizeof(unsigned long long) * nq, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            const unsigned long long mx = *std::max_element(cnt.begin(), cnt.end());
            if (mx <= cap)
                break;
            cap = mx; // the exact size: the second run cannot overflow
        }
        // per-query sort by (dist, id) — search.hpp:336
        std::vector<uint64_t> beg(nq), endv(nq);
        uint64_t tot = 0;
        for (uint64_t i = 0; i < nq; ++i) {
            beg[i] = i * cap;
            endv[i] = i * cap + cnt[i];
            offsets_out[i] = tot;
            tot += cnt[i];
        }
        offsets_out[nq] = tot;
        DevBuf d_beg(sizeof(uint64_t) * nq, st), d_end(sizeof(uint64_t) * nq, st),
            d_sorted(sizeof(unsigned long long) * std::max<uint64_t>(nq * cap, 1), st);
        CK(cudaMemcpyAsync(d_beg.p, beg.data(), sizeof(uint64_t) * nq, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(d_end.p, endv.data(), sizeof(uint64_t) * nq, cudaMemcpyHostToDevice, st));
        size_t tmp_bytes = 0;
        CK(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp_bytes, d_pool.as<unsigned long long>(),
                                              d_sorted.as<unsigned long long>(), static_cast<int64_t>(nq * cap),
                                              static_cast<int64_t>(nq), d_beg.as<uint64_t>(), d_end.as<uint64_t>(), st));
        DevBuf d_tmp(tmp_bytes, st);
        CK(cub::DeviceSegmentedSort::SortKeys(d_tmp.p, tmp_bytes, d_pool.as<unsigned long long>(),
                                              d_sorted.as<unsigned long long>(), static_cast<int64_t>(nq * cap),
                                              static_cast<int64_t>(nq), d_beg.as<uint64_t>(), d_end.as<uint64_t>(), st));
        DevBuf d_offs(sizeof(uint64_t) * (nq + 1), st);
        CK(cudaMemcpyAsync(d_offs.p, offsets_out, sizeof(uint64_t) * (nq + 1), cudaMemcpyHostToDevice, st));
        DevBuf d_ids(sizeof(uint32_t) * std::max<uint64_t>(tot, 1), st),
            d_dist(sizeof(float) * std::max<uint64_t>(tot, 1), st);
        trim_unpack_keys_kernel<<<static_cast<unsigned>(nq), 128, 0, st>>>(
            d_sorted.as<unsigned long long>(), static_cast<uint32_t>(cap), d_offs.as<uint64_t>(), nq,
            d_ids.as<uint32_t>(), d_dist.as<float>());
        CK(cudaGetLastError());
        auto* hid = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * std::max<uint64_t>(tot, 1)));
        auto* hd = static_cast<float*>(std::malloc(sizeof(float) * std::max<uint64_t>(tot, 1)));
        if (!hid || !hd) {
            std::free(hid);
            std::free(hd);
            return set_err(TRIM_ENOMEM, "search_trim_range: result allocation failed");
        }
        std::vector<unsigned long long> ct(nq * 6);
        CK(cudaMemcpyAsync(hid, d_ids.p, sizeof(uint32_t) * tot, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hd, d_dist.p, sizeof(float) * tot, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(ct.data(), d_ct.p, sizeof(unsigned long long) * nq * 6, cudaMemcpyDeviceToHost, st));
        cudaError_t se = cudaStreamSynchronize(st);
        if (se != cudaSuccess) {
            std::free(hid);
            std::free(hd);
            CK(se);
        }
        if (counters_out)
            put_counters_host(counters_out, ct, nq);
        *ids_out = hid;
        *dist_out = hd;
        return TRIM_OK;
    });
}

} // extern "C"
