// trim_flat_mma.cuh — distance bounds for flat kNN scans on the tensor cores.
//
// A flat scan (nlist = 1, ivf.hpp:318-320 with one list) evaluates candidates
// in row order; for every evaluated candidate the reference computes the exact
// euclidean_sq (distance.hpp:11-29) and replaces the top-k iff (d, id) < top
// (ivf.hpp:276-282). At low γ nearly every row is evaluated (config 4: 1M rows
// of 960 floats per query), but only rows that can enter the top-k need d
// exactly: any d_lb > T_pub (>= the live threshold) loses the comparison.
//
// trim_flat_dist_kernel computes D~[q][r] = |q|^2 + |x_r|^2 - 2 q.x_r for a
// tile of 128 queries x 128 rows per CTA with tcgen05.mma kind::tf32: the K
// dimension streams in blocks of 32 floats through a 3-stage shared-memory
// ring filled by cp.async.bulk from pre-tiled copies (the queries tiled per
// call, the rows once per index), fp32 accumulators in TMEM, tcgen05.ld
// epilogue. tf32 keeps 10 mantissa bits, so |D~ - d| <= E = 2^-7|q||x| +
// 2^-14(|q|^2 + |x|^2) (dot error <= (2^-9 + 2^-20)|q||x| by Cauchy-Schwarz,
// doubled; accumulation and the fp32 epilogue inside the second term and the
// margin). trim_knn_kernel uses d_lb = D~ - E to skip the exact distance of
// members that provably cannot enter the top-k.
#pragma once

#include <cuda_bf16.h>

#include "trim_probe_mma.cuh"

namespace trimgpu {

constexpr uint32_t kFlatKB = 32;      // floats of K per stage
#ifndef TRIM_FLAT_STAGES
#define TRIM_FLAT_STAGES 3
#endif
constexpr uint32_t kFlatStages = TRIM_FLAT_STAGES;
constexpr uint32_t kFlatBlockBytes = kMmaM * kFlatKB * 4; // 16 KB per operand per stage

__host__ __device__ inline uint32_t flat_kpad(uint32_t dim) { return (dim + kFlatKB - 1) / kFlatKB * kFlatKB; }
__host__ __device__ inline size_t flat_mma_smem() { return size_t(kFlatStages) * 2 * kFlatBlockBytes + 256; }

// rows [nrows x stride] -> tiles [ceil(nrows/128)][kpad/32][8 chunks][128 rows][4 floats]
// (zero padded), the image of the K-major no-swizzle shared-memory operand.
__global__ void trim_flat_tile_kernel(const float* __restrict__ rows, uint64_t nrows, uint32_t stride, uint32_t dim,
                                      uint32_t kpad, float4* __restrict__ out) {
    const uint64_t tile = blockIdx.x;
    const uint32_t nkb = kpad / kFlatKB;
    const uint32_t per = nkb * 8 * kMmaM; // float4 per tile
    for (uint32_t i = threadIdx.x; i < per; i += blockDim.x) {
        const uint32_t r = i % kMmaM, ch = (i / kMmaM) % 8, kb = i / (kMmaM * 8);
        const uint64_t row = tile * kMmaM + r;
        const uint32_t k0 = kb * kFlatKB + ch * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < nrows) {
            const float* src = rows + row * stride;
            if (k0 + 3 < dim) {
                v = *reinterpret_cast<const float4*>(src + k0);
            } else {
                float t[4] = {0.f, 0.f, 0.f, 0.f};
                for (uint32_t j = 0; j < 4; ++j)
                    if (k0 + j < dim)
                        t[j] = src[k0 + j];
                v = make_float4(t[0], t[1], t[2], t[3]);
            }
        }
        out[tile * per + i] = v;
    }
}

// |x|^2 (fp32 from fp64) and |x| rounded up, per row.
__global__ void trim_row_norm_kernel(const float* __restrict__ rows, uint64_t nrows, uint32_t stride, uint32_t dim,
                                     float* __restrict__ n2, float* __restrict__ n) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= nrows)
        return;
    const float* x = rows + r * stride;
    double s = 0.0;
    for (uint32_t i = 0; i < dim; ++i)
        s += static_cast<double>(x[i]) * x[i];
    n2[r] = static_cast<float>(s);
    n[r] = __double2float_ru(sqrt(s) * (1.0 + 1e-12));
}

// Bound on |D~ - |q - x|^2| of the tf32 distance (2x margin); norms rounded up.
__device__ __forceinline__ float gt_err(float qn, float qn2, float xn, float xn2) {
    return __fadd_ru(__fmul_ru(__fmul_ru(qn, xn), 1.0f / 128.0f), __fmul_ru(__fadd_ru(qn2, xn2), 1.0f / 16384.0f));
}

// grid (query tiles, row tiles) — query tiles fastest, so the CTAs sharing a
// row tile run together and read it from HBM once. kMmaThreads threads.
// Two outputs: dap (fp32 D~, the exact ground-truth kernel takes D~ +- E), or,
// when lb is set (the kNN filter), the rigorous lower bound D~ - E (E =
// 2^-7|q||x| + 2^-14(|q|^2 + |x|^2) from rounded-up norms, gt_err) rounded
// down to bf16: half the bytes of the nq x rows matrix, and the filter loads
// no norms.
__global__ void __launch_bounds__(kMmaThreads, 2)
trim_flat_dist_kernel(const float4* __restrict__ qtiles, const float* __restrict__ qn2, uint64_t nq,
                      const float4* __restrict__ rtiles, const float* __restrict__ xn2, uint64_t nrows, uint32_t kpad,
                      float* __restrict__ dap, uint64_t ld, uint64_t rt0, __nv_bfloat16* __restrict__ lb,
                      const float* __restrict__ xn) {
    extern __shared__ __align__(128) unsigned char fm_smem[];
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
    const uint64_t qt = blockIdx.x, rt = rt0 + blockIdx.y; // row tiles launched in groups of <= 65535
    const uint32_t nkb = kpad / kFlatKB;
    const size_t tile_f4 = static_cast<size_t>(nkb) * 8 * kMmaM;
    unsigned char* sA = fm_smem;                                   // [stages][16 KB]
    unsigned char* sB = fm_smem + kFlatStages * kFlatBlockBytes;   // [stages][16 KB]
    uint64_t* bars = reinterpret_cast<uint64_t*>(fm_smem + 2 * kFlatStages * kFlatBlockBytes);
    __shared__ uint32_t s_tmem;
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kFlatStages),
                   done = smem_u32(bars + 2 * kFlatStages);
    if (tid == 0) {
        for (uint32_t s = 0; s < kFlatStages; ++s) {
            mbar_init_u(full0 + 8 * s, 1);
            mbar_init_u(empty0 + 8 * s, 1);
        }
        mbar_init_u(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    if (warp == 0) {
        if (lane == 0) {
            const float4* a = qtiles + qt * tile_f4;
            const float4* b = rtiles + rt * tile_f4;
            for (uint32_t kb = 0; kb < nkb; ++kb) {
                const uint32_t s = kb % kFlatStages;
                if (kb >= kFlatStages)
                    mbar_wait_u(empty0 + 8 * s, ((kb / kFlatStages) - 1) & 1u);
                mbar_expect_tx(full0 + 8 * s, 2 * kFlatBlockBytes);
                bulk_g2s(smem_u32(sA + s * kFlatBlockBytes), a + static_cast<size_t>(kb) * 8 * kMmaM,
                         kFlatBlockBytes, full0 + 8 * s);
                bulk_g2s(smem_u32(sB + s * kFlatBlockBytes), b + static_cast<size_t>(kb) * 8 * kMmaM,
                         kFlatBlockBytes, full0 + 8 * s);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            for (uint32_t kb = 0; kb < nkb; ++kb) {
                const uint32_t s = kb % kFlatStages;
                mbar_wait_u(full0 + 8 * s, (kb / kFlatStages) & 1u);
                tc_fence_after();
                const uint32_t a0 = smem_u32(sA + s * kFlatBlockBytes), b0 = smem_u32(sB + s * kFlatBlockBytes);
#pragma unroll
                for (uint32_t ks = 0; ks < kFlatKB / 8; ++ks) {
                    const uint64_t ad = umma_desc(a0 + ks * 2 * (kMmaM * 16), kMmaM * 16, 128);
                    const uint64_t bd = umma_desc(b0 + ks * 2 * (kMmaN * 16), kMmaN * 16, 128);
                    tc_mma_tf32(tmem, ad, bd, (kb | ks) ? 1u : 0u);
                }
                tc_commit(empty0 + 8 * s);
            }
            tc_commit(done);
        }
        __syncwarp();
    } else {
        const uint32_t quarter = warp & 3u;
        const uint64_t q = qt * kMmaM + quarter * 32 + lane;
        const float qq = q < nq ? qn2[q] : 0.0f;
        const float qq_up = __fmul_ru(qq, 1.0f + 1.0f / 1048576.0f), qn_up = __fsqrt_ru(qq_up);
        mbar_wait_u(done, 0);
        tc_fence_after();
        const uint64_t r0 = rt * kMmaN;
#pragma unroll 1
        for (uint32_t j0 = 0; j0 < kMmaN; j0 += 32) {
            float v[32];
            tc_ld32(tmem + ((quarter * 32u) << 16) + j0, v);
            if (q < nq && lb) {
                uint4* dst = reinterpret_cast<uint4*>(lb + q * ld + r0 + j0);
#pragma unroll
                for (int j = 0; j < 32; j += 8) {
                    uint32_t w[4];
#pragma unroll
                    for (int h = 0; h < 8; h += 2) {
                        float l2[2];
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const uint64_t r = min(r0 + j0 + j + h + e, nrows - 1);
                            const float x2 = __ldg(xn2 + r);
                            const float dt = __fsub_rn(__fadd_rn(qq, x2), __fmul_rn(2.0f, v[j + h + e]));
                            l2[e] = __fsub_rd(dt, gt_err(qn_up, qq_up, __ldg(xn + r), x2));
                        }
                        const __nv_bfloat162 b = __halves2bfloat162(__float2bfloat16_rd(l2[0]), __float2bfloat16_rd(l2[1]));
                        w[h / 2] = *reinterpret_cast<const uint32_t*>(&b);
                    }
                    dst[j / 8] = make_uint4(w[0], w[1], w[2], w[3]);
                }
            } else if (q < nq) {
                float4* dst = reinterpret_cast<float4*>(dap + q * ld + r0 + j0);
#pragma unroll
                for (int j = 0; j < 32; j += 4) {
                    float4 o;
                    const uint64_t r = r0 + j0 + j;
                    o.x = __fsub_rn(__fadd_rn(qq, __ldg(xn2 + min(r + 0, nrows - 1))), __fmul_rn(2.0f, v[j + 0]));
                    o.y = __fsub_rn(__fadd_rn(qq, __ldg(xn2 + min(r + 1, nrows - 1))), __fmul_rn(2.0f, v[j + 1]));
                    o.z = __fsub_rn(__fadd_rn(qq, __ldg(xn2 + min(r + 2, nrows - 1))), __fmul_rn(2.0f, v[j + 2]));
                    o.w = __fsub_rn(__fadd_rn(qq, __ldg(xn2 + min(r + 3, nrows - 1))), __fmul_rn(2.0f, v[j + 3]));
                    dst[j / 4] = o;
                }
            }
        }
        tc_fence_before();
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
    }
}

// |q|^2 per query row (fp64 sum, rounded to fp32) for the epilogue.
__global__ void trim_query_norm_kernel(const float* __restrict__ q, uint64_t nq, uint32_t stride, uint32_t dim,
                                       float* __restrict__ n2) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nq)
        return;
    double s = 0.0;
    for (uint32_t j = 0; j < dim; ++j)
        s += static_cast<double>(q[i * stride + j]) * q[i * stride + j];
    n2[i] = static_cast<float>(s);
}

} // namespace trimgpu

namespace trimgpu {

// --------------------------------------------------------------------------
// Exact brute-force ground truth (core/ground_truth.hpp:53-74, 97-113): the k
// smallest (euclidean_sq, id) over every row, in the reference's fp32
// 4-accumulator arithmetic, from the tensor-core bounds D~ +- E: one CTA per
// query takes tau >= the k-th smallest upper bound (two 11-bit radix passes
// over the row keys in global memory), keeps the rows whose lower bound is <=
// tau (the true k nearest are among them), computes their exact distances and
// sorts by (d, id). More than kGtCap survivors (massive ties) fall back to
// exact distances for every row.
// --------------------------------------------------------------------------
constexpr uint32_t kGtCap = 4096;
constexpr uint32_t kGtThreads = 256;

__host__ __device__ inline size_t gt_smem(uint32_t dim_stride) {
    return sizeof(uint64_t) * kGtCap + sizeof(uint32_t) * 2048 + sizeof(float) * dim_stride + 64;
}


// Radix select over keys produced by key_of(row) for rows [0, n): the prefix
// after `passes` 11/11/10-bit passes of the rank-th smallest key.
template <typename KeyFn>
__device__ uint32_t gt_radix(uint64_t n, uint32_t rank, uint32_t* hist, uint32_t* sc, int passes, KeyFn key_of) {
    const uint32_t tid = threadIdx.x;
    uint32_t prefix = 0, pmask = 0;
    for (int p = 0; p < passes; ++p) {
        const uint32_t shift = p == 0 ? 21u : (p == 1 ? 10u : 0u);
        const uint32_t nb = p < 2 ? 2048u : 1024u;
        for (uint32_t i = tid; i < nb; i += kGtThreads)
            hist[i] = 0;
        __syncthreads();
        for (uint64_t r = tid; r < n; r += kGtThreads) {
            const uint32_t kk = key_of(r);
            if ((kk & pmask) == prefix)
                atomicAdd(&hist[(kk >> shift) & (nb - 1)], 1u);
        }
        __syncthreads();
        const uint32_t per = nb / kGtThreads;
        uint32_t s = 0;
        for (uint32_t i = 0; i < per; ++i)
            s += hist[tid * per + i];
        uint32_t tot;
        const uint32_t excl = block_excl_scan(s, sc + 8, &tot);
        if (excl < rank && rank <= excl + s) {
            uint32_t cum = excl;
            for (uint32_t i = 0; i < per; ++i) {
                const uint32_t h = hist[tid * per + i];
                if (cum + h >= rank) {
                    sc[0] = tid * per + i;
                    sc[1] = cum;
                    break;
                }
                cum += h;
            }
        }
        __syncthreads();
        prefix |= sc[0] << shift;
        pmask |= (nb - 1) << shift;
        rank -= sc[1];
        __syncthreads();
    }
    return prefix;
}

__global__ void __launch_bounds__(kGtThreads)
trim_gt_select_kernel(DevIndex ix, const float* __restrict__ queries, uint64_t nq, uint32_t k,
                      const float* __restrict__ dap, uint64_t ld, const float* __restrict__ xn,
                      const float* __restrict__ xn2, float* __restrict__ scratch, uint32_t* __restrict__ ids_out,
                      float* __restrict__ dist_out) {
    extern __shared__ __align__(16) unsigned char gs_smem[];
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint64_t q = blockIdx.x;
    if (q >= nq)
        return;
    const uint64_t n = ix.n;
    uint64_t* sq = reinterpret_cast<uint64_t*>(gs_smem);          // [kGtCap]
    uint32_t* hist = reinterpret_cast<uint32_t*>(sq + kGtCap);     // [2048]
    float* qv = reinterpret_cast<float*>(hist + 2048);             // [dim_stride]
    uint32_t* sc = reinterpret_cast<uint32_t*>(qv + ix.dim_stride); // [16]
    const float* qrow = queries + q * ix.dim_stride;
    const float* arow = dap + q * ld;
    float qp = 0.0f;
    for (uint32_t i = tid; i < ix.dim_stride; i += kGtThreads) {
        const float x = qrow[i];
        qv[i] = x;
        qp = __fadd_ru(qp, __fmul_ru(x, x));
    }
    for (int o = 16; o > 0; o >>= 1)
        qp = __fadd_ru(qp, __shfl_xor_sync(0xffffffffu, qp, o));
    if (lane == 0)
        hist[warp] = __float_as_uint(qp);
    __syncthreads();
    float qn2 = 0.0f;
    for (uint32_t w = 0; w < kGtThreads / 32; ++w)
        qn2 = __fadd_ru(qn2, __uint_as_float(hist[w]));
    qn2 = __fmul_ru(qn2, 1.0f + 1.0f / 65536.0f);
    const float qn = __fsqrt_ru(qn2);
    __syncthreads();
    auto ukey = [&](uint64_t r) { return f2key(__fadd_ru(arow[r], gt_err(qn, qn2, __ldg(xn + r), __ldg(xn2 + r)))); };
    const float tau = key2f(gt_radix(n, k, hist, sc, 2, ukey) | 0x3FFu);
    if (tid == 0)
        sc[2] = 0;
    __syncthreads();
    for (uint64_t r = tid; r < n; r += kGtThreads)
        if (__fsub_rd(arow[r], gt_err(qn, qn2, __ldg(xn + r), __ldg(xn2 + r))) <= tau) {
            const uint32_t slot = atomicAdd(&sc[2], 1u);
            if (slot < kGtCap)
                sq[slot] = r;
        }
    __syncthreads();
    const uint32_t ncand = sc[2];
    uint32_t* io = ids_out + q * k;
    float* dout = dist_out + q * k;
    if (ncand <= kGtCap) {
        uint32_t n2 = 1;
        while (n2 < ncand)
            n2 <<= 1;
        for (uint32_t i = tid; i < n2; i += kGtThreads) {
            uint64_t kk = ~0ull;
            if (i < ncand) {
                const uint64_t r = sq[i];
                const float d = euclid_sq_vec4(qv, ix.vectors + r * ix.dim_stride, ix.dim);
                kk = (static_cast<uint64_t>(__float_as_uint(d)) << 32) | static_cast<uint32_t>(ix.id_base + r);
            }
            sq[i] = kk;
        }
        __syncthreads();
        for (uint32_t size = 2; size <= n2; size <<= 1)
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                for (uint32_t i = tid; i < n2 / 2; i += kGtThreads) {
                    const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                    const bool up = (lo & size) == 0;
                    const uint64_t a = sq[lo], b = sq[hi];
                    if ((a > b) == up) {
                        sq[lo] = b;
                        sq[hi] = a;
                    }
                }
                __syncthreads();
            }
        for (uint32_t i = tid; i < k; i += kGtThreads) {
            io[i] = static_cast<uint32_t>(sq[i] & 0xffffffffu);
            dout[i] = __uint_as_float(static_cast<uint32_t>(sq[i] >> 32));
        }
        return;
    }
    // massive ties: exact distances of every row (into scratch), exact selection
    float* ex = scratch + q * ld;
    for (uint64_t r = tid; r < n; r += kGtThreads)
        ex[r] = euclid_sq_vec4(qv, ix.vectors + r * ix.dim_stride, ix.dim);
    __syncthreads();
    auto ekey = [&](uint64_t r) { return __float_as_uint(ex[r]); };
    const uint32_t kth = gt_radix(n, k, hist, sc, 3, ekey);
    if (tid == 0)
        sc[2] = 0;
    __syncthreads();
    for (uint64_t r = tid; r < n; r += kGtThreads) // rows below the k-th distance: fewer than k
        if (__float_as_uint(ex[r]) < kth)
            sq[atomicAdd(&sc[2], 1u)] = (static_cast<uint64_t>(__float_as_uint(ex[r])) << 32) |
                                        static_cast<uint32_t>(ix.id_base + r);
    __syncthreads();
    const uint32_t n_lt = sc[2];
    if (warp == 0) { // ties at the k-th distance: the lowest ids, in order
        uint32_t n_eq = 0;
        const uint32_t need = k - n_lt;
        for (uint64_t r0 = 0; r0 < n && n_eq < need; r0 += 32) {
            const uint64_t r = r0 + lane;
            const bool eq = r < n && __float_as_uint(ex[r]) == kth;
            const uint32_t beq = __ballot_sync(0xffffffffu, eq);
            const uint32_t rr = n_eq + __popc(beq & ((1u << lane) - 1u));
            if (eq && rr < need)
                sq[n_lt + rr] = (static_cast<uint64_t>(kth) << 32) | static_cast<uint32_t>(ix.id_base + r);
            n_eq += __popc(beq);
        }
    }
    uint32_t n2 = 1;
    while (n2 < k)
        n2 <<= 1;
    for (uint32_t i = k + tid; i < n2; i += kGtThreads)
        sq[i] = ~0ull;
    __syncthreads();
    for (uint32_t size = 2; size <= n2; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = tid; i < n2 / 2; i += kGtThreads) {
                const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t a = sq[lo], b = sq[hi];
                if ((a > b) == up) {
                    sq[lo] = b;
                    sq[hi] = a;
                }
            }
            __syncthreads();
        }
    for (uint32_t i = tid; i < k; i += kGtThreads) {
        io[i] = static_cast<uint32_t>(sq[i] & 0xffffffffu);
        dout[i] = __uint_as_float(static_cast<uint32_t>(sq[i] >> 32));
    }
}

} // namespace trimgpu
