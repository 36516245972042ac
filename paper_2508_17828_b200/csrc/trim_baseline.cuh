// trim_baseline.cuh — ivf::search_baseline_ivfpq (ivf/ivf.hpp:193-237) on
// sm_100a: the two-phase IVFPQ the paper compares TRIM against.
//
//   1. trim_bl_est_kernel   ADC estimate (no sqrt, ivf.hpp:207) for every probed
//                           entry, stored as a sortable (est, id) key — the
//                           ScoredId order partial_sort uses (ivf.hpp:218-220);
//   2. trim_bl_select_kernel exact k'-th smallest key per query by 8-bit radix
//                           select in shared memory, then the k' keys <= it;
//   3. trim_bl_refine_kernel exact L2 of the k' (ivf.hpp:224-228), bitonic sort
//                           by (d, id), first k (ivf.hpp:230-235).
#pragma once

#include "trim_kernels.cuh"

namespace trimgpu {

struct BlParams {
    const float* queries;
    uint64_t nq;
    uint32_t np;
    const uint32_t* probe;
    uint32_t slice;
    uint64_t stride;              // scratch keys per query
    unsigned long long* keys;     // nq*stride
    unsigned long long* total;    // nq stream lengths
};

template <int M, int KS>
__global__ void __launch_bounds__(kThreads)
trim_bl_est_kernel(DevIndex ix, BlParams p) {
    unsigned char* smem = trim_dyn_smem;
    const uint32_t q = blockIdx.y, tid = threadIdx.x;
    const uint32_t m = M > 0 ? static_cast<uint32_t>(M) : ix.m;
    float* lut = reinterpret_cast<float*>(smem);
    float* qv = lut + lut_bytes(M, m) / sizeof(float);
    size_t off = lut_bytes(M, m) + sizeof(float) * ix.dim_stride;
    StreamSmem st;
    st.base = reinterpret_cast<uint64_t*>(smem + off);
    off += sizeof(uint64_t) * p.np;
    st.cum = reinterpret_cast<uint32_t*>(smem + off);
    const float* qg = p.queries + static_cast<size_t>(q) * ix.dim_stride;
    for (uint32_t i = tid; i < ix.dim_stride; i += kThreads)
        qv[i] = qg[i];
    const uint32_t total = load_stream(ix, p.probe ? p.probe + static_cast<size_t>(q) * p.np : nullptr,
                                       p.np, st);
    if (blockIdx.x == 0 && tid == 0)
        p.total[q] = total;
    const uint32_t begin = blockIdx.x * p.slice;
    if (begin >= total)
        return;
    const uint32_t end = min(total, begin + p.slice);
    build_lut_blocked<M>(ix, qv, lut);
    __syncthreads();
    uint32_t lo = 0, hi = p.np;
    while (lo + 1 < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (st.cum[mid] <= begin)
            lo = mid;
        else
            hi = mid;
    }
    uint32_t li = lo;
    unsigned long long* out = p.keys + static_cast<size_t>(q) * p.stride;
    for (uint32_t pp = begin + tid; pp < end; pp += kThreads) {
        while (st.cum[li + 1] <= pp)
            ++li;
        const uint32_t e = static_cast<uint32_t>(st.base[li] + (pp - st.cum[li]));
        // exact reference-order ADC, conflict-free (lane-rotated schedule)
        const float est = adc_exact<M>(ix.codes + static_cast<size_t>(e) * ix.code_stride, m,
                                       tid & 31u);
        out[pp] = scored_key(est, __ldg(ix.list_ids + e));
    }
}

constexpr int kSelThreads = 1024;
constexpr uint32_t kSelSmemKeys = 16384; // finish in shared memory below this

#ifndef TRIM_M // non-template kernels: compiled once, in trim_capi.cu
// One CTA per query: the k'-th smallest key (keys are unique: ids are),
// then every key <= it, into sel[q*kp ...]. n <= kp selects everything.
__global__ void __launch_bounds__(kSelThreads)
trim_bl_select_kernel(const unsigned long long* keys, uint64_t stride,
                      const unsigned long long* totals, uint32_t kp, unsigned long long* sel) {
    unsigned char* smem = trim_dyn_smem;
    unsigned long long* sk = reinterpret_cast<unsigned long long*>(smem);
    __shared__ uint32_t hist[256];
    __shared__ uint32_t s_bucket, s_rank, s_count, s_n;
    const uint32_t q = blockIdx.x, tid = threadIdx.x;
    const unsigned long long* kq = keys + static_cast<size_t>(q) * stride;
    unsigned long long* out = sel + static_cast<size_t>(q) * kp;
    const uint32_t n = static_cast<uint32_t>(totals[q]);
    if (n <= kp) {
        for (uint32_t i = tid; i < n; i += kSelThreads)
            out[i] = kq[i];
        return;
    }
    unsigned long long prefix = 0, pmask = 0;
    uint32_t rank = kp; // 1-based rank of the threshold key among the matching set
    uint32_t cnt = n;
    int shift = 56;
    for (; shift >= 0 && cnt > kSelSmemKeys; shift -= 8) {
        for (uint32_t i = tid; i < 256; i += kSelThreads)
            hist[i] = 0;
        __syncthreads();
        for (uint32_t i = tid; i < n; i += kSelThreads) {
            const unsigned long long key = kq[i];
            if ((key & pmask) == prefix)
                atomicAdd(&hist[(key >> shift) & 0xFFu], 1u);
        }
        __syncthreads();
        if (tid == 0) {
            uint32_t c = 0, b = 0;
            for (; b < 256; ++b) {
                if (c + hist[b] >= rank)
                    break;
                c += hist[b];
            }
            s_bucket = b;
            s_rank = rank - c;
            s_count = hist[b];
        }
        __syncthreads();
        prefix |= static_cast<unsigned long long>(s_bucket) << shift;
        pmask |= 0xFFull << shift;
        rank = s_rank;
        cnt = s_count;
        __syncthreads();
    }
    // gather the matching keys into shared memory and sort them
    if (tid == 0)
        s_n = 0;
    __syncthreads();
    for (uint32_t i = tid; i < n; i += kSelThreads) {
        const unsigned long long key = kq[i];
        if ((key & pmask) == prefix) {
            const uint32_t s = atomicAdd(&s_n, 1u);
            sk[s] = key;
        }
    }
    __syncthreads();
    uint32_t n2 = 1;
    while (n2 < cnt)
        n2 <<= 1;
    for (uint32_t i = cnt + tid; i < n2; i += kSelThreads)
        sk[i] = ~0ull;
    __syncthreads();
    for (uint32_t size = 2; size <= n2; size <<= 1)
        for (uint32_t stride2 = size >> 1; stride2 > 0; stride2 >>= 1) {
            for (uint32_t i = tid; i < n2 / 2; i += kSelThreads) {
                const uint32_t lo = 2 * i - (i & (stride2 - 1));
                const uint32_t hi = lo + stride2;
                const bool up = (lo & size) == 0;
                const unsigned long long a = sk[lo], b = sk[hi];
                if ((a > b) == up) {
                    sk[lo] = b;
                    sk[hi] = a;
                }
            }
            __syncthreads();
        }
    const unsigned long long thr = sk[rank - 1];
    __syncthreads();
    if (tid == 0)
        s_n = 0;
    __syncthreads();
    for (uint32_t i = tid; i < n; i += kSelThreads) {
        const unsigned long long key = kq[i];
        if (key <= thr) {
            const uint32_t s = atomicAdd(&s_n, 1u);
            out[s] = key;
        }
    }
}

// One CTA per query: exact distances of the refine pool, sort by (d,id),
// first k. pool size = min(kp, total).
__global__ void __launch_bounds__(kThreads)
trim_bl_refine_kernel(DevIndex ix, const float* queries, const unsigned long long* sel,
                      const unsigned long long* totals, uint32_t kp, uint32_t kp_pow2, uint32_t k,
                      uint32_t* ids_out, float* dist_out) {
    unsigned char* smem = trim_dyn_smem;
    float* qv = reinterpret_cast<float*>(smem);
    unsigned long long* sk = reinterpret_cast<unsigned long long*>(smem + sizeof(float) * ix.dim_stride);
    const uint32_t q = blockIdx.x, tid = threadIdx.x;
    for (uint32_t i = tid; i < ix.dim_stride; i += kThreads)
        qv[i] = queries[static_cast<size_t>(q) * ix.dim_stride + i];
    __syncthreads();
    const uint32_t n = static_cast<uint32_t>(min(static_cast<unsigned long long>(kp), totals[q]));
    for (uint32_t i = tid; i < kp_pow2; i += kThreads) {
        unsigned long long key = ~0ull;
        if (i < n) {
            const uint32_t id = static_cast<uint32_t>(sel[static_cast<size_t>(q) * kp + i]);
            const float* row = ix.vectors + static_cast<size_t>(id - ix.id_base) * ix.dim_stride;
            key = scored_key(euclid_sq_vec4(qv, row, ix.dim), id);
        }
        sk[i] = key;
    }
    __syncthreads();
    for (uint32_t size = 2; size <= kp_pow2; size <<= 1)
        for (uint32_t stride2 = size >> 1; stride2 > 0; stride2 >>= 1) {
            for (uint32_t i = tid; i < kp_pow2 / 2; i += kThreads) {
                const uint32_t lo = 2 * i - (i & (stride2 - 1));
                const uint32_t hi = lo + stride2;
                const bool up = (lo & size) == 0;
                const unsigned long long a = sk[lo], b = sk[hi];
                if ((a > b) == up) {
                    sk[lo] = b;
                    sk[hi] = a;
                }
            }
            __syncthreads();
        }
    for (uint32_t i = tid; i < k; i += kThreads) {
        const unsigned long long key = i < n ? sk[i] : ~0ull;
        ids_out[static_cast<size_t>(q) * k + i] = key == ~0ull ? kInvalidId : static_cast<uint32_t>(key);
        dist_out[static_cast<size_t>(q) * k + i] =
            key == ~0ull ? __int_as_float(0x7f800000) : __uint_as_float(static_cast<uint32_t>(key >> 32));
    }
}

#endif // TRIM_M

} // namespace trimgpu
