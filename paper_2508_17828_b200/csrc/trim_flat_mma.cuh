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

#include "trim_probe_mma.cuh"

namespace trimgpu {

constexpr uint32_t kFlatKB = 32;      // floats of K per stage
constexpr uint32_t kFlatStages = 3;
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

// grid (query tiles, row tiles) — query tiles fastest, so the CTAs sharing a
// row tile run together and read it from HBM once. kMmaThreads threads.
__global__ void __launch_bounds__(kMmaThreads, 2)
trim_flat_dist_kernel(const float4* __restrict__ qtiles, const float* __restrict__ qn2, uint64_t nq,
                      const float4* __restrict__ rtiles, const float* __restrict__ xn2, uint64_t nrows, uint32_t kpad,
                      float* __restrict__ dap, uint64_t ld) {
    extern __shared__ __align__(128) unsigned char fm_smem[];
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
    const uint64_t qt = blockIdx.x, rt = blockIdx.y;
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
        mbar_wait_u(done, 0);
        tc_fence_after();
        const uint64_t r0 = rt * kMmaN;
#pragma unroll 1
        for (uint32_t j0 = 0; j0 < kMmaN; j0 += 32) {
            float v[32];
            tc_ld32(tmem + ((quarter * 32u) << 16) + j0, v);
            if (q < nq) {
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
