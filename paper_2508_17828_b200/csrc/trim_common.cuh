// trim_common.cuh — device arithmetic shared by the TRIM kernels.
//
// Every fp32 operation that feeds a comparison is written with an explicit
// round-to-nearest intrinsic (__fadd_rn/__fsub_rn/__fmul_rn/__fsqrt_rn), in
// the exact order of the reference, so the compiler cannot contract or
// reassociate it. The library is additionally built with -fmad=false. The
// reference binary has no FMA, so results are bit-identical.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdio>

namespace trimgpu {

constexpr int kWarp = 32;
constexpr uint32_t kInvalidId = 0xFFFFFFFFu;

struct DevIndex {
    uint32_t dim;
    uint32_t dim_stride; // floats per vector row (dim rounded up to 4)
    uint32_t m;
    uint32_t ksub;
    uint32_t code_stride; // bytes per code row (m rounded up to 16)
    uint32_t nlist;
    uint32_t sd_uniform; // common sub-dimension when every subspace has it, else 0
    uint64_t n;
    uint64_t id_base;
    const uint32_t* sub_dims;    // m
    const uint32_t* sub_offsets; // m
    const float* centroids;      // ksub*dim; subspace j at ksub*sub_offsets[j]
    const float* centroids_t;    // ksub*dim code-major: code c's sub-centroid j at c*dim + sub_offsets[j]
    const float* coarse;         // nlist*dim_stride
    const uint64_t* list_offsets;
    const uint32_t* list_ids;
    const uint8_t* codes; // total*code_stride
    const float* lx;      // total
    const float* vectors; // n*dim_stride
    // per-list metadata for the list-level bound (trim_list_meta_kernel)
    const float* list_R;    // nlist: >= max over the list of |c_l - landmark(x)|
    const float* list_xmin; // nlist: min stored lx of the list
    const float* list_xmax; // nlist: max stored lx of the list
};

// core/distance.hpp:11-29: four interleaved accumulators, remainder into
// acc0, (acc0+acc1)+(acc2+acc3). `a` is the query side (a[i] - b[i]).
__device__ __forceinline__ float euclid_sq_generic(const float* a, const float* b, uint32_t dim) {
    float acc0 = 0.0f, acc1 = 0.0f, acc2 = 0.0f, acc3 = 0.0f;
    uint32_t i = 0;
    for (; i + 4 <= dim; i += 4) {
        const float d0 = __fsub_rn(a[i], b[i]);
        const float d1 = __fsub_rn(a[i + 1], b[i + 1]);
        const float d2 = __fsub_rn(a[i + 2], b[i + 2]);
        const float d3 = __fsub_rn(a[i + 3], b[i + 3]);
        acc0 = __fadd_rn(acc0, __fmul_rn(d0, d0));
        acc1 = __fadd_rn(acc1, __fmul_rn(d1, d1));
        acc2 = __fadd_rn(acc2, __fmul_rn(d2, d2));
        acc3 = __fadd_rn(acc3, __fmul_rn(d3, d3));
    }
    for (; i < dim; ++i) {
        const float d = __fsub_rn(a[i], b[i]);
        acc0 = __fadd_rn(acc0, __fmul_rn(d, d));
    }
    return __fadd_rn(__fadd_rn(acc0, acc1), __fadd_rn(acc2, acc3));
}

// Same arithmetic, both operands 16-byte aligned rows: one float4 feeds
// acc0..acc3 in exactly the CPU order. `q` lives in shared memory (all lanes
// read the same address: broadcast), `x` in global memory.
__device__ __forceinline__ float euclid_sq_vec4(const float* __restrict__ q,
                                                const float* __restrict__ x, uint32_t dim,
                                                bool prefetch = false) {
    float acc0 = 0.0f, acc1 = 0.0f, acc2 = 0.0f, acc3 = 0.0f;
    const uint32_t nv = dim >> 2;
    const float4* q4 = reinterpret_cast<const float4*>(q);
    const float4* x4 = reinterpret_cast<const float4*>(x);
    // long rows (>= 1 KB): the whole row in flight at once (one DRAM round trip);
    // the loop below, which keeps only a few loads in flight, then hits L1
    if (prefetch || dim >= 256)
        for (uint32_t o = 0; o < dim * 4u; o += 128u)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const char*>(x) + o));
#pragma unroll 4
    for (uint32_t v = 0; v < nv; ++v) {
        const float4 a = q4[v];
        const float4 b = __ldg(x4 + v);
        const float d0 = __fsub_rn(a.x, b.x);
        const float d1 = __fsub_rn(a.y, b.y);
        const float d2 = __fsub_rn(a.z, b.z);
        const float d3 = __fsub_rn(a.w, b.w);
        acc0 = __fadd_rn(acc0, __fmul_rn(d0, d0));
        acc1 = __fadd_rn(acc1, __fmul_rn(d1, d1));
        acc2 = __fadd_rn(acc2, __fmul_rn(d2, d2));
        acc3 = __fadd_rn(acc3, __fmul_rn(d3, d3));
    }
    for (uint32_t i = nv << 2; i < dim; ++i) {
        const float d = __fsub_rn(q[i], __ldg(x + i));
        acc0 = __fadd_rn(acc0, __fmul_rn(d, d));
    }
    return __fadd_rn(__fadd_rn(acc0, acc1), __fadd_rn(acc2, acc3));
}

// trim/lower_bound.hpp:18-22: strict_lb + ((2*gamma)*gl_q)*gl_x.
// `two_gamma` is 2.0f*gamma (exact: scaling by 2).
__device__ __forceinline__ float relaxed_lb(float glq, float glx, float two_gamma) {
    const float d = __fsub_rn(glq, glx);
    return __fadd_rn(__fmul_rn(d, d), __fmul_rn(__fmul_rn(two_gamma, glq), glx));
}

// ScoredId ordering (core/ground_truth.hpp:39-50): dist, then id.
__device__ __forceinline__ bool scored_less(float da, uint32_t ia, float db, uint32_t ib) {
    return da < db || (da == db && ia < ib);
}

// Sortable 64-bit key for (dist >= 0, id): float bits are monotone for
// non-negative floats, so key order == ScoredId order.
__device__ __forceinline__ uint64_t scored_key(float d, uint32_t id) {
    return (static_cast<uint64_t>(__float_as_uint(d)) << 32) | id;
}

// pq/pq.hpp:158-172 into shared memory: lut[j*ksub + c] for all (j, c),
// thread-strided over c. Centroid reads come from L2 (the codebook is tiny).
__device__ __forceinline__ void build_lut_smem(const DevIndex& ix, const float* q_smem,
                                               float* lut) {
    for (uint32_t j = 0; j < ix.m; ++j) {
        const uint32_t sd = ix.sub_dims[j];
        const uint32_t off = ix.sub_offsets[j];
        const float* cb = ix.centroids + static_cast<size_t>(ix.ksub) * off;
        for (uint32_t c = threadIdx.x; c < ix.ksub; c += blockDim.x)
            lut[j * ix.ksub + c] = euclid_sq_generic(q_smem + off, cb + c * sd, sd);
    }
}

// euclidean_sq (core/distance.hpp:11-29) of one row by a QUAD of lanes:
// lane `sub` (0..3) of the quad owns accumulator acc_sub and adds
// (q[4t+sub] - x[4t+sub])^2 for t = 0, 1, ... — exactly the reference's
// chain for that accumulator (the tail, dim % 4, goes to acc0 = sub 0); then
// (acc0 + acc1) + (acc2 + acc3) by two xor-shuffles (fp addition is
// commutative, so every lane of the quad ends with the same bits). A third
// of the instructions of one lane walking the whole row, and 8 rows per warp
// pass. Warp-collective: all 32 lanes call it (`row` may be null on idle
// quads); q in shared memory, rows 16-byte aligned.
__device__ __forceinline__ float euclid_sq_quad(const float* __restrict__ q, const float* __restrict__ row,
                                                uint32_t dim, uint32_t sub) {
    float acc = 0.0f;
    if (row) {
        const uint32_t nv = dim >> 2;
        // the row's 128-byte lines in flight at once (one DRAM round trip)
        for (uint32_t o = sub * 128u; o < dim * 4u; o += 512u)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const char*>(row) + o));
        const float* x = row + sub;
        const float* qq = q + sub;
#pragma unroll 8
        for (uint32_t t = 0; t < nv; ++t) {
            const float d = __fsub_rn(qq[4 * t], __ldg(x + 4 * t));
            acc = __fadd_rn(acc, __fmul_rn(d, d));
        }
        if (sub == 0)
            for (uint32_t i = nv << 2; i < dim; ++i) {
                const float d = __fsub_rn(q[i], __ldg(row + i));
                acc = __fadd_rn(acc, __fmul_rn(d, d));
            }
    }
    const float t = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 1));
    return __fadd_rn(t, __shfl_xor_sync(0xffffffffu, t, 2));
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

} // namespace trimgpu
