// trim_probe_mma.cuh — detail_ivf::probe_order (ivf/ivf.hpp:173-187) for large
// nlist, with the coarse-distance GEMM on the 5th-generation tensor cores.
//
// The probe order is defined by exact fp32 distances (distance.hpp:11-29,
// four interleaved accumulators) with ties broken by list id. Computing all
// nq x nlist of them in that order is pure SIMT work (~37M warp-FP
// instructions per 1024 queries at nlist 4096, d 96). Instead:
//
//  1. trim_probe_mma_kernel: D~[q][c] = |q|^2 + |c|^2 - 2 q.c with q.c from
//     tcgen05.mma kind::tf32 (operands staged in shared memory — the query
//     tile by the CTA, centroid tiles by cp.async.bulk from a pre-tiled copy
//     — accumulators in TMEM, read back with tcgen05.ld). |D~ - d| <= E(q,c)
//     = 2^-6 |q||c| + 2^-14 (|q|^2 + |c|^2): tf32 keeps 10 mantissa bits
//     (relative input error <= 2^-10, so |dot error| <= 2^-8.9 |q||c| by
//     Cauchy-Schwarz, accumulation included), the fp32 epilogue and norms
//     are far inside the second term; both terms carry a 2x margin.
//  2. trim_probe_select_kernel (one CTA per query): tau >= the np-th
//     smallest upper bound U_c = D~_c + E_c (two 11-bit radix passes, bucket
//     upper edge); every list the exact order can place in the first np has
//     L_c = D~_c - E_c <= tau (np lists have d <= tau, a list with L_c > tau
//     has d > tau: strictly worse than all of them). Those
//     candidates get the exact reference-order distance and are sorted by
//     (d, id); the first np are the reference's probe order. If more than
//     kSelCap lists survive (degenerate data), the CTA computes every exact
//     distance and selects among them directly — same result, slower.
#pragma once

#include "trim_common.cuh"

namespace trimgpu {

constexpr uint32_t kMmaM = 128;        // queries per CTA (MMA M, TMEM lanes)
constexpr uint32_t kMmaN = 128;        // centroids per tile (MMA N)
constexpr uint32_t kMmaTilesPerCta = 2;
constexpr uint32_t kMmaThreads = 192;  // warp 0: loads, warp 1: MMA, warps 2-5: epilogue
constexpr uint32_t kMmaMaxK = 128;     // K = dim rounded up to 8
constexpr uint32_t kSelCap = 512;      // exact-distance candidates per query

__host__ __device__ inline uint32_t mma_k(uint32_t dim) { return (dim + 7u) & ~7u; }
__host__ __device__ inline size_t mma_tile_bytes(uint32_t K) { return size_t(kMmaN) * K * 4u; }
__host__ __device__ inline size_t probe_mma_smem(uint32_t K) {
    return size_t(kMmaM) * K * 4u + 2 * mma_tile_bytes(K) + 128;
}
__host__ __device__ inline uint32_t mma_ld(uint32_t nlist) { return (nlist + kMmaN - 1) / kMmaN * kMmaN; }

// Shared-memory matrix descriptor, K-major, no swizzle ("interleaved" core
// matrices of 8 rows x 16 bytes): element (row r, k) of a tile lives at
// (k/4)*LBO + (r/8)*SBO + (r%8)*16 + (k%4)*4. Our tiles store each 16-byte
// K-chunk for all rows contiguously: LBO = rows*16, SBO = 128.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (saddr >> 4) & 0x3FFFu;
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46; // descriptor version (sm_100)
    return d;        // base offset 0, layout type 0 (SWIZZLE_NONE)
}

// Instruction descriptor: D f32, A/B tf32, both K-major, N = kMmaN, M = kMmaM.
constexpr uint32_t kMmaIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((kMmaN >> 3) << 17) | ((kMmaM >> 4) << 24);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init_u(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_u(uint32_t bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(bar),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_u(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done)
                     : "r"(bar), "r"(parity)
                     : "memory");
    }
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
                 "l"(adesc), "l"(bdesc), "r"(kMmaIdesc), "r"(accum)
                 : "memory");
}
// 32 consecutive fp32 columns of this thread's TMEM lane.
__device__ __forceinline__ void tc_ld32(uint32_t taddr, float v[32]) {
    uint32_t r[32];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                   "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
                   "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
                   "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i)
        v[i] = __uint_as_float(r[i]);
}

// Pre-tiled coarse centroids (built once per index): tile t holds centroids
// [t*128, t*128+128) as K/4 chunks of 128 rows x 16 bytes (zero padded), the
// exact image of the shared-memory B operand.
__global__ void trim_coarse_tile_kernel(DevIndex ix, uint32_t K, float4* out) {
    const uint32_t t = blockIdx.x;
    const uint32_t nk = K / 4;
    for (uint32_t i = threadIdx.x; i < nk * kMmaN; i += blockDim.x) {
        const uint32_t kc = i / kMmaN, r = i % kMmaN, c = t * kMmaN + r;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (c < ix.nlist) {
            const float* row = ix.coarse + static_cast<size_t>(c) * ix.dim_stride;
            const uint32_t k0 = kc * 4;
            if (k0 < ix.dim_stride)
                v = *reinterpret_cast<const float4*>(row + k0);
        }
        out[static_cast<size_t>(t) * nk * kMmaN + i] = v;
    }
}

// |c|^2 (fp32, from fp64) and |c| rounded up, per centroid.
__global__ void trim_coarse_norm_kernel(DevIndex ix, float* cn2, float* cn) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ix.nlist)
        return;
    const float* row = ix.coarse + static_cast<size_t>(c) * ix.dim_stride;
    double s = 0.0;
    for (uint32_t i = 0; i < ix.dim; ++i)
        s += static_cast<double>(row[i]) * row[i];
    cn2[c] = static_cast<float>(s);
    cn[c] = __double2float_ru(sqrt(s) * (1.0 + 1e-12));
}

// grid (ceil(nq/128), ceil(ntiles/kMmaTilesPerCta)), kMmaThreads threads.
__global__ void __launch_bounds__(kMmaThreads, 1)
trim_probe_mma_kernel(const float* __restrict__ queries, uint64_t nq, uint32_t dim_stride, uint32_t K,
                      const float4* __restrict__ coarse_t, const float* __restrict__ cn2, uint32_t nlist,
                      float* __restrict__ approx) {
    extern __shared__ __align__(128) unsigned char pm_smem[];
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
    const uint64_t q0 = static_cast<uint64_t>(blockIdx.x) * kMmaM;
    const uint32_t ntiles = (nlist + kMmaN - 1) / kMmaN;
    const uint32_t t0 = blockIdx.y * kMmaTilesPerCta;
    const uint32_t t1 = min(ntiles, t0 + kMmaTilesPerCta);
    const uint32_t nt = t1 - t0;
    const uint32_t nk = K / 4;
    const size_t tb = mma_tile_bytes(K);

    float4* sA = reinterpret_cast<float4*>(pm_smem);                        // [nk][128]
    unsigned char* sB = pm_smem + static_cast<size_t>(kMmaM) * K * 4;        // 2 x [nk][128]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + 2 * tb);
    __shared__ uint32_t s_tmem;
    const uint32_t full0 = smem_u32(bars + 0), empty0 = smem_u32(bars + 2);
    const uint32_t tfull0 = smem_u32(bars + 4), tempty0 = smem_u32(bars + 6);

    // query tile -> core-matrix layout (chunk kc of row r at kc*2048 + r*16)
    for (uint32_t i = tid; i < nk * kMmaM; i += kMmaThreads) {
        const uint32_t kc = i / kMmaM, r = i % kMmaM;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (q0 + r < nq && kc * 4 < dim_stride)
            v = *reinterpret_cast<const float4*>(queries + (q0 + r) * dim_stride + kc * 4);
        sA[i] = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); // generic writes -> tensor-core reads
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init_u(full0 + 8 * b, 1);
            mbar_init_u(empty0 + 8 * b, 1);
            mbar_init_u(tfull0 + 8 * b, 1);
            mbar_init_u(tempty0 + 8 * b, 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) { // TMEM: two 128-column fp32 accumulators
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    if (warp == 0) {
        if (lane == 0) {
            for (uint32_t i = 0; i < nt; ++i) {
                const uint32_t b = i & 1u;
                if (i >= 2)
                    mbar_wait_u(empty0 + 8 * b, ((i >> 1) - 1) & 1u);
                mbar_expect_tx(full0 + 8 * b, static_cast<uint32_t>(tb));
                bulk_g2s(smem_u32(sB + b * tb), coarse_t + static_cast<size_t>(t0 + i) * nk * kMmaN,
                         static_cast<uint32_t>(tb), full0 + 8 * b);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t a0 = smem_u32(sA);
            for (uint32_t i = 0; i < nt; ++i) {
                const uint32_t b = i & 1u;
                mbar_wait_u(full0 + 8 * b, (i >> 1) & 1u);
                if (i >= 2)
                    mbar_wait_u(tempty0 + 8 * b, ((i >> 1) - 1) & 1u);
                tc_fence_after();
                const uint32_t b0 = smem_u32(sB + b * tb);
                for (uint32_t ks = 0; ks < K / 8; ++ks) {
                    const uint64_t ad = umma_desc(a0 + ks * 2 * (kMmaM * 16), kMmaM * 16, 128);
                    const uint64_t bd = umma_desc(b0 + ks * 2 * (kMmaN * 16), kMmaN * 16, 128);
                    tc_mma_tf32(tmem + b * kMmaN, ad, bd, ks > 0 ? 1u : 0u);
                }
                tc_commit(empty0 + 8 * b); // smem tile free once these MMAs complete
                tc_commit(tfull0 + 8 * b); // accumulator ready
            }
        }
        __syncwarp();
    } else {
        // epilogue: thread <-> query row 32*(warp%4) + lane (its TMEM lane)
        const uint32_t quarter = warp & 3u;
        const uint32_t r = quarter * 32 + lane;
        const uint64_t q = q0 + r;
        float qn2 = 0.0f;
        for (uint32_t kc = 0; kc < nk; ++kc) {
            const float4 v = sA[kc * kMmaM + r];
            qn2 = __fadd_rn(qn2, __fadd_rn(__fadd_rn(__fmul_rn(v.x, v.x), __fmul_rn(v.y, v.y)),
                                           __fadd_rn(__fmul_rn(v.z, v.z), __fmul_rn(v.w, v.w))));
        }
        const size_t ld = mma_ld(nlist);
        for (uint32_t i = 0; i < nt; ++i) {
            const uint32_t b = i & 1u;
            mbar_wait_u(tfull0 + 8 * b, (i >> 1) & 1u);
            tc_fence_after();
            const uint32_t c0 = (t0 + i) * kMmaN;
#pragma unroll 1
            for (uint32_t j0 = 0; j0 < kMmaN; j0 += 32) {
                float v[32];
                tc_ld32(tmem + ((quarter * 32u) << 16) + b * kMmaN + j0, v);
                if (q < nq) {
                    float4* dst = reinterpret_cast<float4*>(approx + q * ld + c0 + j0);
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        float4 o;
                        o.x = __fsub_rn(__fadd_rn(qn2, __ldg(cn2 + min(c0 + j0 + j + 0, nlist - 1))), __fmul_rn(2.0f, v[j + 0]));
                        o.y = __fsub_rn(__fadd_rn(qn2, __ldg(cn2 + min(c0 + j0 + j + 1, nlist - 1))), __fmul_rn(2.0f, v[j + 1]));
                        o.z = __fsub_rn(__fadd_rn(qn2, __ldg(cn2 + min(c0 + j0 + j + 2, nlist - 1))), __fmul_rn(2.0f, v[j + 2]));
                        o.w = __fsub_rn(__fadd_rn(qn2, __ldg(cn2 + min(c0 + j0 + j + 3, nlist - 1))), __fmul_rn(2.0f, v[j + 3]));
                        dst[j / 4] = o;
                    }
                }
            }
            tc_fence_before();
            mbar_arrive_u(tempty0 + 8 * b);
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    }
}

// Orderable key of a float (ascending float order = ascending unsigned order).
__device__ __forceinline__ uint32_t f2key(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

// Warp radix select: the value of the rank-th smallest (1-based) key among
// keys[0..n) (shared memory), 8 bits per pass. h: 256-entry warp histogram.
__device__ __forceinline__ uint32_t warp_radix_select(const uint32_t* keys, uint32_t n, uint32_t rank, uint32_t* h,
                                                      uint32_t lane) {
    uint32_t prefix = 0, pmask = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (uint32_t i = lane; i < 256; i += 32)
            h[i] = 0;
        __syncwarp();
        for (uint32_t c = lane; c < n; c += 32) {
            const uint32_t kk = keys[c];
            if ((kk & pmask) == prefix)
                atomicAdd(&h[(kk >> shift) & 0xFFu], 1u);
        }
        __syncwarp();
        uint32_t loc[8], s = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            loc[i] = h[8 * lane + i];
            s += loc[i];
        }
        uint32_t incl = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= static_cast<uint32_t>(o))
                incl += t;
        }
        const uint32_t excl = incl - s;
        const bool mine = excl < rank && rank <= incl;
        uint32_t bucket = 0, before = 0;
        if (mine) {
            uint32_t cum = excl;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (cum + loc[i] >= rank) {
                    bucket = 8 * lane + i;
                    before = cum;
                    break;
                }
                cum += loc[i];
            }
        }
        const uint32_t src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
        bucket = __shfl_sync(0xffffffffu, bucket, src);
        before = __shfl_sync(0xffffffffu, before, src);
        prefix |= bucket << shift;
        pmask |= 0xFFu << shift;
        rank -= before;
        __syncwarp();
    }
    return prefix;
}

// Warp bitonic sort of n2 (power of two) u64 keys in shared memory, ascending.
__device__ __forceinline__ void warp_bitonic(uint64_t* sq, uint32_t n2, uint32_t lane) {
    for (uint32_t size = 2; size <= n2; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = lane; i < n2 / 2; i += 32) {
                const uint32_t lo = 2 * i - (i & (stride - 1));
                const uint32_t hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t a = sq[lo], b = sq[hi];
                if ((a > b) == up) {
                    sq[lo] = b;
                    sq[hi] = a;
                }
            }
            __syncwarp();
        }
}

constexpr uint32_t kPSelThreads = 256;

__host__ __device__ inline size_t probe_select_smem(uint32_t nlist, uint32_t dim_stride) {
    return sizeof(uint64_t) * kSelCap + sizeof(uint32_t) * nlist + sizeof(uint32_t) * 2048 +
           sizeof(float) * dim_stride + 64;
}

// Block-wide exclusive scan of one value per thread (kPSelThreads threads);
// returns the exclusive prefix, *total the sum. ws: 8 words of scratch.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* ws, uint32_t* total) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= static_cast<uint32_t>(o))
            incl += t;
    }
    if (lane == 31)
        ws[warp] = incl;
    __syncthreads();
    uint32_t before = 0, tot = 0;
#pragma unroll
    for (uint32_t w = 0; w < kPSelThreads / 32; ++w) {
        const uint32_t x = ws[w];
        before += w < warp ? x : 0u;
        tot += x;
    }
    __syncthreads();
    *total = tot;
    return before + incl - v;
}

// Block radix select over keys[0..n) (shared memory): digits of 11, 11 and 10
// bits from the top. Returns the key prefix after `passes` passes; with 3
// passes that is the rank-th smallest key (1-based) itself.
__device__ __forceinline__ uint32_t block_radix_select(const uint32_t* keys, uint32_t n, uint32_t rank,
                                                       uint32_t* hist, uint32_t* sc, int passes) {
    const uint32_t tid = threadIdx.x;
    uint32_t prefix = 0, pmask = 0;
    for (int p = 0; p < passes; ++p) {
        const uint32_t shift = p == 0 ? 21u : (p == 1 ? 10u : 0u);
        const uint32_t nb = p < 2 ? 2048u : 1024u;
        for (uint32_t i = tid; i < nb; i += kPSelThreads)
            hist[i] = 0;
        __syncthreads();
        for (uint32_t c = tid; c < n; c += kPSelThreads) {
            const uint32_t kk = keys[c];
            if ((kk & pmask) == prefix)
                atomicAdd(&hist[(kk >> shift) & (nb - 1)], 1u);
        }
        __syncthreads();
        const uint32_t per = nb / kPSelThreads; // 8 or 4 bins per thread
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

// Block bitonic sort of n2 (power of two) u64 keys in shared memory, ascending.
__device__ __forceinline__ void block_bitonic(uint64_t* sq, uint32_t n2) {
    for (uint32_t size = 2; size <= n2; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < n2 / 2; i += kPSelThreads) {
                const uint32_t lo = 2 * i - (i & (stride - 1));
                const uint32_t hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t a = sq[lo], b = sq[hi];
                if ((a > b) == up) {
                    sq[lo] = b;
                    sq[hi] = a;
                }
            }
            __syncthreads();
        }
}

// One CTA (kPSelThreads) per query.
__global__ void __launch_bounds__(kPSelThreads)
trim_probe_select_kernel(DevIndex ix, const float* __restrict__ queries, uint64_t nq, uint32_t np,
                         const float* __restrict__ approx, const float* __restrict__ cn2,
                         const float* __restrict__ cn, uint32_t* __restrict__ probe_out) {
    extern __shared__ __align__(16) unsigned char ps_smem[];
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint64_t q = blockIdx.x;
    if (q >= nq)
        return;
    const uint32_t nlist = ix.nlist;
    uint64_t* sq = reinterpret_cast<uint64_t*>(ps_smem);          // [kSelCap]
    uint32_t* keys = reinterpret_cast<uint32_t*>(sq + kSelCap);   // [nlist]
    uint32_t* hist = keys + nlist;                                // [2048]
    float* qv = reinterpret_cast<float*>(hist + 2048);            // [dim_stride]
    uint32_t* sc = reinterpret_cast<uint32_t*>(qv + ix.dim_stride); // [16] scalars
    const float* qrow = queries + q * ix.dim_stride;
    const float* arow = approx + q * mma_ld(nlist);

    float qp = 0.0f;
    for (uint32_t i = tid; i < ix.dim_stride; i += kPSelThreads) {
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
    for (uint32_t w = 0; w < kPSelThreads / 32; ++w)
        qn2 = __fadd_ru(qn2, __uint_as_float(hist[w]));
    qn2 = __fmul_ru(qn2, 1.0f + 1.0f / 65536.0f); // >= |q|^2
    const float qn = __fsqrt_ru(qn2);
    __syncthreads();

    // upper bounds U_c = D~_c + E_c as orderable keys
    for (uint32_t c = tid; c < nlist; c += kPSelThreads) {
        const float e = __fadd_ru(__fmul_ru(__fmul_ru(qn, __ldg(cn + c)), 1.0f / 64.0f),
                                  __fmul_ru(__fadd_ru(qn2, __ldg(cn2 + c)), 1.0f / 16384.0f));
        keys[c] = f2key(__fadd_ru(arow[c], e));
    }
    __syncthreads();
    // tau' >= np-th smallest U: the top 22 key bits, bucket upper edge
    const float tau = key2f(block_radix_select(keys, nlist, np, hist, sc, 2) | 0x3FFu);
    if (tid == 0)
        sc[2] = 0;
    __syncthreads();
    // candidates: lower bound L_c = D~_c - E_c <= tau'
    for (uint32_t c = tid; c < nlist; c += kPSelThreads) {
        const float e = __fadd_ru(__fmul_ru(__fmul_ru(qn, __ldg(cn + c)), 1.0f / 64.0f),
                                  __fmul_ru(__fadd_ru(qn2, __ldg(cn2 + c)), 1.0f / 16384.0f));
        if (__fsub_rd(arow[c], e) <= tau) {
            const uint32_t slot = atomicAdd(&sc[2], 1u);
            if (slot < kSelCap)
                keys[slot] = c; // (U keys are no longer needed)
        }
    }
    __syncthreads();
    const uint32_t ncand = sc[2];
    uint32_t* out = probe_out + q * np;
    if (ncand <= kSelCap) {
        uint32_t n2 = 1;
        while (n2 < ncand)
            n2 <<= 1;
        for (uint32_t i = tid; i < n2; i += kPSelThreads) {
            uint64_t kk = ~0ull;
            if (i < ncand) {
                const uint32_t c = keys[i];
                const float d = euclid_sq_vec4(qv, ix.coarse + static_cast<size_t>(c) * ix.dim_stride, ix.dim);
                kk = (static_cast<uint64_t>(__float_as_uint(d)) << 32) | c;
            }
            sq[i] = kk;
        }
        __syncthreads();
        block_bitonic(sq, n2);
        for (uint32_t i = tid; i < np; i += kPSelThreads)
            out[i] = static_cast<uint32_t>(sq[i] & 0xffffffffu);
        return;
    }
    // degenerate (too many candidates): exact distances of every list
    for (uint32_t c = tid; c < nlist; c += kPSelThreads)
        keys[c] = __float_as_uint(euclid_sq_vec4(qv, ix.coarse + static_cast<size_t>(c) * ix.dim_stride, ix.dim));
    __syncthreads();
    const uint32_t kth = block_radix_select(keys, nlist, np, hist, sc, 3);
    if (tid == 0)
        sc[2] = 0;
    __syncthreads();
    for (uint32_t c = tid; c < nlist; c += kPSelThreads) // keys below the np-th: fewer than np
        if (keys[c] < kth)
            sq[atomicAdd(&sc[2], 1u)] = (static_cast<uint64_t>(keys[c]) << 32) | c;
    __syncthreads();
    const uint32_t n_lt = sc[2];
    if (warp == 0) { // ties at the np-th distance: the lowest list ids, in order
        uint32_t n_eq = 0;
        const uint32_t need = np - n_lt;
        for (uint32_t c0 = 0; c0 < nlist && n_eq < need; c0 += 32) {
            const uint32_t c = c0 + lane;
            const bool eq = c < nlist && keys[c] == kth;
            const uint32_t beq = __ballot_sync(0xffffffffu, eq);
            const uint32_t r = n_eq + __popc(beq & ((1u << lane) - 1u));
            if (eq && r < need)
                sq[n_lt + r] = (static_cast<uint64_t>(kth) << 32) | c;
            n_eq += __popc(beq);
        }
    }
    uint32_t n2 = 1;
    while (n2 < np)
        n2 <<= 1;
    for (uint32_t i = np + tid; i < n2; i += kPSelThreads)
        sq[i] = ~0ull;
    __syncthreads();
    block_bitonic(sq, n2);
    for (uint32_t i = tid; i < np; i += kPSelThreads)
        out[i] = static_cast<uint32_t>(sq[i] & 0xffffffffu);
}

} // namespace trimgpu
