// trim_build.cu — device-side index build.
//
// The reference builds its index on host threads (pq::train pq/pq.hpp:65-113,
// trim::build_landmarks trim/landmarks.hpp:57-72, ivf::build_ivf
// ivf/ivf.hpp:112-154). At 10M-800M vectors that is hours of CPU, so the
// B200 build runs here:
//   * seeded synthetic data (Philox4x32-10 + Box-Muller; blob rows are
//     assigned round-robin like make_blob_dataset, core/synthetic.hpp:21-33);
//   * k-means, bit-identical to pq::kmeans (kmeans.hpp:89-158): k-means++
//     seeding with the reference's std::mt19937_64 draws and sequential D^2
//     sums/scan on the host, distance updates on the device; Lloyd steps with
//     the reference's exact nearest-centroid arithmetic and ties
//     (pq/kmeans.hpp:27-41), per-cluster double sums in ascending point order
//     (kmeans.hpp:129-140) and the reference's empty-cluster repair
//     (kmeans.hpp:111-127) — so pq::train and build_ivf reproduce the
//     reference's codebook, coarse quantizer and lists from the same rows;
//   * PQ encode + Γ(l,x) bit-exact with pq::encode / build_landmarks;
//   * lists in ascending id order (stable radix sort by list id, ivf.hpp:147-152).
// Row samples use the reference's own Fisher-Yates sampler with std::mt19937_64
// (pq.hpp:72-80, ivf.hpp:121-126), so sampled row sets match the reference.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "../../include/trim_gpu.h"
#include "trim_common.cuh"

using namespace trimgpu;

namespace {

} // namespace
extern "C" void trim__set_last_error(const char* msg); // trim_capi.cu (thread-local)
namespace {

// Builder errors land in the same thread-local slot trim_last_error() reads.
int berr(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    trim__set_last_error(buf);
    return code;
}

struct BErr {
    int code;
};

#define BK(call)                                                                          \
    do {                                                                                  \
        cudaError_t _e = (call);                                                          \
        if (_e != cudaSuccess) {                                                          \
            berr(TRIM_ECUDA, "CUDA error %s (%s) at %s:%d", cudaGetErrorName(_e),         \
                 cudaGetErrorString(_e), __FILE__, __LINE__);                             \
            throw BErr{TRIM_ECUDA};                                                       \
        }                                                                                 \
    } while (0)

template <typename Fn>
int bguard(Fn&& fn) {
    try {
        return fn();
    } catch (const BErr& e) {
        return e.code;
    } catch (const std::bad_alloc&) {
        return berr(TRIM_ENOMEM, "host allocation failed");
    }
}

struct BDevice {
    int prev = 0;
    explicit BDevice(int d) {
        BK(cudaGetDevice(&prev));
        if (prev != d)
            BK(cudaSetDevice(d));
    }
    ~BDevice() { cudaSetDevice(prev); }
};

template <typename T>
struct DArr {
    T* p = nullptr;
    explicit DArr(size_t n) {
        if (n)
            BK(cudaMalloc(&p, sizeof(T) * n));
    }
    ~DArr() {
        if (p)
            cudaFree(p);
    }
    DArr(const DArr&) = delete;
    DArr& operator=(const DArr&) = delete;
};

// ---------------------------------------------------------------- Philox
__device__ __forceinline__ uint4 philox4x32(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

__device__ __forceinline__ float u01(uint32_t v) { // (0, 1]
    return (static_cast<float>(v >> 8) + 1.0f) * (1.0f / 16777216.0f);
}

// 4 standard normals per counter (Box-Muller on two pairs).
__device__ __forceinline__ float4 normal4(uint64_t seed, uint64_t ctr) {
    const uint4 r = philox4x32(make_uint4(static_cast<uint32_t>(ctr), static_cast<uint32_t>(ctr >> 32),
                                          0x6A09E667u, 0xF3BCC908u),
                               make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)));
    const float r0 = sqrtf(-2.0f * logf(u01(r.x))), r1 = sqrtf(-2.0f * logf(u01(r.z)));
    const float t0 = 6.283185307179586f * u01(r.y), t1 = 6.283185307179586f * u01(r.w);
    return make_float4(r0 * cosf(t0), r0 * sinf(t0), r1 * cosf(t1), r1 * sinf(t1));
}

// out[i][j] = centers[i % nc][j] + sigma * z(i,j)   (centers == null: z)
__global__ void synth_kernel(const float* centers, uint32_t nc, uint32_t dim, uint64_t n, float sigma,
                             uint64_t seed, float* out) {
    const uint64_t total = n * dim;
    for (uint64_t g = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4; g < total;
         g += static_cast<uint64_t>(gridDim.x) * blockDim.x * 4) {
        const float4 z = normal4(seed, g >> 2);
        const float zz[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const uint64_t e = g + t;
            if (e < total) {
                if (centers) {
                    const uint64_t i = e / dim;
                    const uint32_t j = static_cast<uint32_t>(e - i * dim);
                    out[e] = __fadd_rn(centers[(i % nc) * dim + j], __fmul_rn(sigma, zz[t]));
                } else {
                    out[e] = zz[t];
                }
            }
        }
    }
}

// uniform [0,1) rows, optionally L2-normalised (VectorDataset::normalize_rows,
// core/dataset.hpp:44-56: double sum of squares, float(1/sqrt), scale).
__global__ void synth_uniform_kernel(uint64_t n, uint32_t dim, uint64_t seed, int normalize, float* out) {
    const uint64_t row = static_cast<uint64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
    const uint32_t lane = threadIdx.x & 31u;
    if (row >= n)
        return;
    float* r = out + row * dim;
    double sq = 0.0;
    for (uint32_t j = lane; j < dim; j += 32) {
        const uint64_t e = row * dim + j;
        const uint4 v = philox4x32(make_uint4(static_cast<uint32_t>(e), static_cast<uint32_t>(e >> 32),
                                              0x3C6EF372u, 0xA54FF53Au),
                                   make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)));
        const float u = static_cast<float>(v.x >> 8) * (1.0f / 16777216.0f);
        r[j] = u;
        sq += static_cast<double>(u) * u;
    }
    if (!normalize)
        return;
    for (int o = 16; o > 0; o >>= 1)
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if (sq <= 0.0)
        return;
    const float inv = static_cast<float>(1.0 / sqrt(sq));
    for (uint32_t j = lane; j < dim; j += 32)
        r[j] = __fmul_rn(r[j], inv);
}

// ------------------------------------------------------ nearest centroid
// One CTA = 32 points (lane) x all k centroids; warp w takes centroids
// w*8..w*8+7 of every 64-centroid tile. Distances in the reference order
// (euclid 4-accumulator), argmin ties -> lowest index (kmeans.hpp:27-41).
constexpr int kAsgPts = 32;
constexpr int kAsgTile = 64;

__global__ void __launch_bounds__(256)
assign_kernel(const float* __restrict__ x, uint64_t n, uint32_t dim, const float* __restrict__ cent,
              uint32_t k, uint32_t* assign, float* best_out) {
    extern __shared__ __align__(16) float sm[];
    const uint32_t pstride = ((dim + 3) & ~3u) + 4; // padded point rows (conflict-free LDS.128)
    const uint32_t cstride = (dim + 3) & ~3u;
    float* xs = sm;                        // kAsgPts * pstride
    float* cs = xs + kAsgPts * pstride;    // kAsgTile * cstride
    __shared__ float rd[8][kAsgPts];
    __shared__ uint32_t ri[8][kAsgPts];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint64_t p0 = static_cast<uint64_t>(blockIdx.x) * kAsgPts;
    for (uint32_t i = threadIdx.x; i < kAsgPts * pstride; i += blockDim.x) {
        const uint32_t p = i / pstride, j = i - p * pstride;
        xs[i] = (p0 + p < n && j < dim) ? x[(p0 + p) * dim + j] : 0.0f;
    }
    const uint32_t dim4 = dim & ~3u;
    float best = 3.402823466e+38f;
    uint32_t bi = 0;
    for (uint32_t c0 = 0; c0 < k; c0 += kAsgTile) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < kAsgTile * cstride; i += blockDim.x) {
            const uint32_t c = i / cstride, j = i - c * cstride;
            cs[i] = (c0 + c < k && j < dim) ? cent[static_cast<size_t>(c0 + c) * dim + j] : 0.0f;
        }
        __syncthreads();
        float a[8][4];
#pragma unroll
        for (int t = 0; t < 8; ++t)
            a[t][0] = a[t][1] = a[t][2] = a[t][3] = 0.0f;
        const float* xp = xs + lane * pstride;
        for (uint32_t i = 0; i < dim4; i += 4) {
            const float4 xv = *reinterpret_cast<const float4*>(xp + i);
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const float4 cv = *reinterpret_cast<const float4*>(cs + (warp * 8 + t) * cstride + i);
                const float d0 = __fsub_rn(xv.x, cv.x), d1 = __fsub_rn(xv.y, cv.y);
                const float d2 = __fsub_rn(xv.z, cv.z), d3 = __fsub_rn(xv.w, cv.w);
                a[t][0] = __fadd_rn(a[t][0], __fmul_rn(d0, d0));
                a[t][1] = __fadd_rn(a[t][1], __fmul_rn(d1, d1));
                a[t][2] = __fadd_rn(a[t][2], __fmul_rn(d2, d2));
                a[t][3] = __fadd_rn(a[t][3], __fmul_rn(d3, d3));
            }
        }
        for (uint32_t i = dim4; i < dim; ++i) {
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const float d = __fsub_rn(xp[i], cs[(warp * 8 + t) * cstride + i]);
                a[t][0] = __fadd_rn(a[t][0], __fmul_rn(d, d));
            }
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const uint32_t c = c0 + warp * 8 + t;
            const float d = __fadd_rn(__fadd_rn(a[t][0], a[t][1]), __fadd_rn(a[t][2], a[t][3]));
            if (c < k && (d < best || (d == best && c < bi))) {
                best = d;
                bi = c;
            }
        }
    }
    rd[warp][lane] = best;
    ri[warp][lane] = bi;
    __syncthreads();
    if (warp == 0) {
        float b = rd[0][lane];
        uint32_t c = ri[0][lane];
        for (int w = 1; w < 8; ++w) {
            const float d = rd[w][lane];
            const uint32_t ci = ri[w][lane];
            if (d < b || (d == b && ci < c)) {
                b = d;
                c = ci;
            }
        }
        if (p0 + lane < n) {
            assign[p0 + lane] = c;
            if (best_out)
                best_out[p0 + lane] = b;
        }
    }
}

// Large-dim fallback: one warp per point, centroids strided over lanes.
__global__ void assign_kernel_wide(const float* __restrict__ x, uint64_t n, uint32_t dim,
                                   const float* __restrict__ cent, uint32_t k, uint32_t* assign,
                                   float* best_out) {
    const uint64_t p = static_cast<uint64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
    const uint32_t lane = threadIdx.x & 31u;
    if (p >= n)
        return;
    float best = 3.402823466e+38f;
    uint32_t bi = 0;
    for (uint32_t c = lane; c < k; c += 32) {
        const float d = euclid_sq_generic(x + p * dim, cent + static_cast<size_t>(c) * dim, dim);
        if (d < best || (d == best && c < bi)) {
            best = d;
            bi = c;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const float od = __shfl_xor_sync(0xffffffffu, best, o);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (od < best || (od == best && oi < bi)) {
            best = od;
            bi = oi;
        }
    }
    if (lane == 0) {
        assign[p] = bi;
        if (best_out)
            best_out[p] = best;
    }
}

void launch_assign(const float* x, uint64_t n, uint32_t dim, const float* cent, uint32_t k,
                   uint32_t* assign, float* best, cudaStream_t st) {
    if (n == 0)
        return;
    const uint32_t pstride = ((dim + 3) & ~3u) + 4, cstride = (dim + 3) & ~3u;
    const size_t smem = sizeof(float) * (kAsgPts * pstride + kAsgTile * cstride);
    if (smem <= 200 * 1024) {
        BK(cudaFuncSetAttribute(assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
        const uint64_t blocks = (n + kAsgPts - 1) / kAsgPts;
        assign_kernel<<<static_cast<unsigned>(blocks), 256, smem, st>>>(x, n, dim, cent, k, assign, best);
    } else {
        assign_kernel_wide<<<static_cast<unsigned>((n + 7) / 8), 256, 0, st>>>(x, n, dim, cent, k,
                                                                            assign, best);
    }
    BK(cudaGetLastError());
}

// ------------------------------------------------------------ k-means++
// detail::kmeanspp_init (kmeans.hpp:43-86), bit for bit: the draws come from
// the reference's own generator and distributions on the host
// (std::mt19937_64, uniform_int_distribution<size_t>, uniform_real_distribution
// <double> — the same libstdc++ as the reference build), the D^2 total is the
// reference's sequential double sum and the weighted pick its sequential
// subtraction scan (host, over the device-computed d2 copied back), and the
// O(n*dim) distance updates run on the device with the reference arithmetic
// (float euclidean_sq widened to double, d2 = min(d2, d)).
__global__ void kmeanspp_d2_kernel(const float* __restrict__ x, uint64_t n, uint32_t dim,
                                   const float* __restrict__ c, double* d2, int first) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const double d = euclid_sq_generic(x + i * dim, c, dim);
    d2[i] = first ? d : (d < d2[i] ? d : d2[i]);
}

// Lloyd update: cluster c's centroid = float(sum_{i in c, ascending} x_i * (1/size))
// with double sums (kmeans.hpp:129-140). order = point ids sorted by cluster
// (stable), seg = cluster start offsets (k+1).
__global__ void update_kernel(const float* __restrict__ x, uint32_t dim, const uint32_t* order,
                              const uint64_t* seg, uint32_t k, float* cent) {
    const uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= static_cast<uint64_t>(k) * dim)
        return;
    const uint32_t c = static_cast<uint32_t>(g / dim), j = static_cast<uint32_t>(g % dim);
    const uint64_t b = seg[c], e = seg[c + 1];
    if (e == b)
        return;
    double s = 0.0;
    for (uint64_t i = b; i < e; ++i)
        s += x[static_cast<uint64_t>(order[i]) * dim + j];
    const double inv = 1.0 / static_cast<double>(e - b);
    cent[g] = static_cast<float>(s * inv);
}

__global__ void iota_kernel(uint32_t* v, uint64_t n) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n)
        v[i] = static_cast<uint32_t>(i);
}

__global__ void gather_rows_kernel(const float* x, uint32_t dim, uint32_t col0, uint32_t cols,
                                   const uint64_t* rows, uint64_t nr, float* out) {
    const uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= nr * cols)
        return;
    const uint64_t r = g / cols;
    const uint32_t j = static_cast<uint32_t>(g - r * cols);
    out[g] = x[rows[r] * dim + col0 + j];
}

// --------------------------------------------------------- PQ encode
// Thread per row; codebook in shared memory when it fits (all lanes read
// the same centroid: broadcast). Ties keep the lowest index (pq.hpp:123-131).
__global__ void __launch_bounds__(256)
encode_kernel(const float* __restrict__ x, uint64_t n, uint32_t dim, uint32_t m, uint32_t ksub,
              const uint32_t* __restrict__ sub_dims, const uint32_t* __restrict__ sub_offsets,
              const float* __restrict__ cent_g, int cent_in_smem, uint8_t* codes, uint32_t code_stride) {
    extern __shared__ __align__(16) float cs[];
    if (cent_in_smem) {
        for (uint32_t i = threadIdx.x; i < ksub * dim; i += blockDim.x)
            cs[i] = cent_g[i];
        __syncthreads();
    }
    const float* cent = cent_in_smem ? cs : cent_g;
    const uint64_t row = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (row >= n)
        return;
    const float* xr = x + row * dim;
    for (uint32_t j = 0; j < m; ++j) {
        const uint32_t sd = sub_dims[j], off = sub_offsets[j];
        const float* cb = cent + static_cast<size_t>(ksub) * off;
        float xv[16];
        const uint32_t sdc = sd < 16 ? sd : 16;
        for (uint32_t t = 0; t < sdc; ++t)
            xv[t] = xr[off + t];
        uint32_t best = 0;
        float best_d = 3.402823466e+38f;
        for (uint32_t c = 0; c < ksub; ++c) {
            float d;
            if (sd <= 16) {
                float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
                const float* cp = cb + c * sd;
                uint32_t i = 0;
                for (; i + 4 <= sd; i += 4) {
                    const float d0 = __fsub_rn(xv[i], cp[i]), d1 = __fsub_rn(xv[i + 1], cp[i + 1]);
                    const float d2 = __fsub_rn(xv[i + 2], cp[i + 2]), d3 = __fsub_rn(xv[i + 3], cp[i + 3]);
                    a0 = __fadd_rn(a0, __fmul_rn(d0, d0));
                    a1 = __fadd_rn(a1, __fmul_rn(d1, d1));
                    a2 = __fadd_rn(a2, __fmul_rn(d2, d2));
                    a3 = __fadd_rn(a3, __fmul_rn(d3, d3));
                }
                for (; i < sd; ++i) {
                    const float dd = __fsub_rn(xv[i], cp[i]);
                    a0 = __fadd_rn(a0, __fmul_rn(dd, dd));
                }
                d = __fadd_rn(__fadd_rn(a0, a1), __fadd_rn(a2, a3));
            } else {
                d = euclid_sq_generic(xr + off, cb + c * sd, sd);
            }
            if (d < best_d) {
                best_d = d;
                best = c;
            }
        }
        codes[row * code_stride + j] = static_cast<uint8_t>(best);
    }
}

// Γ(l,x) = sqrt(euclidean_sq(x, decode(code))) (landmarks.hpp:66-70), thread per
// row, 4-accumulator order over the full dimension; dsub/dbase map a coordinate
// to its subspace and centroid element.
__global__ void __launch_bounds__(256)
landmark_dist_kernel(const float* __restrict__ x, uint64_t n, uint32_t dim, uint32_t ksub,
                     const uint16_t* __restrict__ dsub, const uint32_t* __restrict__ dbase,
                     const uint8_t* __restrict__ dsd, const float* __restrict__ cent,
                     const uint8_t* __restrict__ codes, uint32_t code_stride, float* lx) {
    const uint64_t row = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (row >= n)
        return;
    const float* xr = x + row * dim;
    const uint8_t* code = codes + row * code_stride;
    auto lval = [&](uint32_t i) { return cent[dbase[i] + static_cast<uint32_t>(code[dsub[i]]) * dsd[i]]; };
    float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
    uint32_t i = 0;
    for (; i + 4 <= dim; i += 4) {
        const float d0 = __fsub_rn(xr[i], lval(i)), d1 = __fsub_rn(xr[i + 1], lval(i + 1));
        const float d2 = __fsub_rn(xr[i + 2], lval(i + 2)), d3 = __fsub_rn(xr[i + 3], lval(i + 3));
        a0 = __fadd_rn(a0, __fmul_rn(d0, d0));
        a1 = __fadd_rn(a1, __fmul_rn(d1, d1));
        a2 = __fadd_rn(a2, __fmul_rn(d2, d2));
        a3 = __fadd_rn(a3, __fmul_rn(d3, d3));
    }
    for (; i < dim; ++i) {
        const float d = __fsub_rn(xr[i], lval(i));
        a0 = __fadd_rn(a0, __fmul_rn(d, d));
    }
    lx[row] = __fsqrt_rn(__fadd_rn(__fadd_rn(a0, a1), __fadd_rn(a2, a3)));
}

__global__ void list_offsets_kernel(const uint32_t* sorted_keys, uint64_t n, uint32_t nlist,
                                    uint64_t* offsets) {
    // offsets[l] = first position with key >= l (keys sorted ascending)
    const uint64_t l = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (l > nlist)
        return;
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (sorted_keys[mid] < l)
            lo = mid + 1;
        else
            hi = mid;
    }
    offsets[l] = lo;
}

// Stable sort of (key, iota) by key: order[] = ids grouped by key, ascending
// within a key.
void stable_group(const uint32_t* d_keys, uint64_t n, uint32_t nkeys, uint32_t* d_sorted_keys,
                  uint32_t* d_order, cudaStream_t st) {
    DArr<uint32_t> iota(n);
    iota_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(iota.p, n);
    BK(cudaGetLastError());
    int bits = 1;
    while ((1ull << bits) < nkeys)
        ++bits;
    size_t tb = 0;
    BK(cub::DeviceRadixSort::SortPairs(nullptr, tb, d_keys, d_sorted_keys, iota.p, d_order,
                                       static_cast<int64_t>(n), 0, bits, st));
    DArr<unsigned char> tmp(tb);
    BK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, d_keys, d_sorted_keys, iota.p, d_order,
                                       static_cast<int64_t>(n), 0, bits, st));
}

// The reference's row sampler (pq.hpp:72-80, ivf.hpp:121-126).
std::vector<uint64_t> sample_rows(uint64_t n, uint64_t sample_n, uint64_t seed) {
    std::vector<uint64_t> rows(n);
    std::iota(rows.begin(), rows.end(), 0);
    std::mt19937_64 rng(seed);
    for (uint64_t i = 0; i < sample_n; ++i) {
        std::uniform_int_distribution<std::size_t> pick(i, n - 1);
        std::swap(rows[i], rows[pick(rng)]);
    }
    rows.resize(sample_n);
    return rows;
}

// k-means on device x[n*dim] (kmeans.hpp:89-158 structure).
void kmeans_device(const float* x, uint64_t n, uint32_t dim, uint32_t k, uint32_t iters, uint64_t seed,
                   float* cent, cudaStream_t st) {
    {
        std::mt19937_64 rng(seed);
        std::uniform_int_distribution<std::size_t> uni(0, n - 1);
        const std::size_t first = uni(rng);
        BK(cudaMemcpyAsync(cent, x + first * dim, sizeof(float) * dim, cudaMemcpyDeviceToDevice, st));
        DArr<double> d2(n);
        double* hd2 = nullptr;
        BK(cudaMallocHost(&hd2, sizeof(double) * n));
        const unsigned nb = static_cast<unsigned>((n + 255) / 256);
        try {
            kmeanspp_d2_kernel<<<nb, 256, 0, st>>>(x, n, dim, cent, d2.p, 1);
            BK(cudaGetLastError());
            for (uint32_t c = 1; c < k; ++c) {
                BK(cudaMemcpyAsync(hd2, d2.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
                BK(cudaStreamSynchronize(st));
                double total = 0.0;
                for (uint64_t i = 0; i < n; ++i)
                    total += hd2[i];
                std::size_t chosen;
                if (total <= 0.0) {
                    chosen = uni(rng); // all mass collapsed; fall back to uniform
                } else {
                    std::uniform_real_distribution<double> ud(0.0, total);
                    double target = ud(rng);
                    chosen = n - 1;
                    for (uint64_t i = 0; i < n; ++i) {
                        target -= hd2[i];
                        if (target <= 0.0) {
                            chosen = i;
                            break;
                        }
                    }
                }
                float* dst = cent + static_cast<size_t>(c) * dim;
                BK(cudaMemcpyAsync(dst, x + chosen * dim, sizeof(float) * dim, cudaMemcpyDeviceToDevice, st));
                kmeanspp_d2_kernel<<<nb, 256, 0, st>>>(x, n, dim, dst, d2.p, 0);
                BK(cudaGetLastError());
            }
            BK(cudaStreamSynchronize(st));
        } catch (...) {
            cudaFreeHost(hd2);
            throw;
        }
        cudaFreeHost(hd2);
    }
    DArr<uint32_t> assign(n), skeys(n), order(n);
    DArr<float> pdist(n);
    DArr<uint64_t> seg(k + 1);
    std::vector<uint64_t> hseg(k + 1);
    std::vector<uint32_t> hassign;
    std::vector<float> hdist;
    for (uint32_t it = 0; it < iters; ++it) {
        launch_assign(x, n, dim, cent, k, assign.p, pdist.p, st);
        stable_group(assign.p, n, k, skeys.p, order.p, st);
        list_offsets_kernel<<<(k + 1 + 255) / 256, 256, 0, st>>>(skeys.p, n, k, seg.p);
        BK(cudaGetLastError());
        BK(cudaMemcpyAsync(hseg.data(), seg.p, sizeof(uint64_t) * (k + 1), cudaMemcpyDeviceToHost, st));
        BK(cudaStreamSynchronize(st));
        bool empty = false;
        for (uint32_t c = 0; c < k; ++c)
            empty |= hseg[c + 1] == hseg[c];
        if (empty) {
            // kmeans.hpp:111-127 on host: move the farthest point of a
            // non-singleton cluster into each empty cluster, in order.
            hassign.resize(n);
            hdist.resize(n);
            BK(cudaMemcpy(hassign.data(), assign.p, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost));
            BK(cudaMemcpy(hdist.data(), pdist.p, sizeof(float) * n, cudaMemcpyDeviceToHost));
            std::vector<uint64_t> sizes(k);
            for (uint32_t c = 0; c < k; ++c)
                sizes[c] = hseg[c + 1] - hseg[c];
            for (uint32_t c = 0; c < k; ++c) {
                if (sizes[c] != 0)
                    continue;
                uint64_t worst = 0;
                float worst_d = -1.0f;
                for (uint64_t i = 0; i < n; ++i)
                    if (sizes[hassign[i]] > 1 && hdist[i] > worst_d) {
                        worst_d = hdist[i];
                        worst = i;
                    }
                --sizes[hassign[worst]];
                hassign[worst] = c;
                sizes[c] = 1;
                hdist[worst] = 0.0f;
            }
            BK(cudaMemcpy(assign.p, hassign.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice));
            stable_group(assign.p, n, k, skeys.p, order.p, st);
            list_offsets_kernel<<<(k + 1 + 255) / 256, 256, 0, st>>>(skeys.p, n, k, seg.p);
            BK(cudaGetLastError());
        }
        const uint64_t tot = static_cast<uint64_t>(k) * dim;
        update_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, st>>>(x, dim, order.p, seg.p, k,
                                                                                cent);
        BK(cudaGetLastError());
    }
    BK(cudaStreamSynchronize(st));
}

} // namespace

extern "C" {

int trim_synth_normal_device(uint64_t n, uint32_t dim, uint64_t seed, float* d_out, int device,
                             void* stream) {
    return bguard([&]() -> int {
        BDevice g(device);
        const uint64_t tot = n * dim;
        const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((tot / 4 + 255) / 256 + 1, 148 * 64));
        synth_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(nullptr, 0, dim, n, 1.0f, seed,
                                                                           d_out);
        BK(cudaGetLastError());
        return TRIM_OK;
    });
}

int trim_synth_blobs_device(const float* d_centers, uint64_t nc, uint32_t dim, uint64_t n, float sigma,
                            uint64_t seed, float* d_out, int device, void* stream) {
    if (nc == 0)
        return berr(TRIM_EINVAL, "make_blob_dataset: no centers");
    return bguard([&]() -> int {
        BDevice g(device);
        const uint64_t tot = n * dim;
        const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((tot / 4 + 255) / 256 + 1, 148 * 64));
        synth_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
            d_centers, static_cast<uint32_t>(nc), dim, n, sigma, seed, d_out);
        BK(cudaGetLastError());
        return TRIM_OK;
    });
}

int trim_synth_uniform_device(uint64_t n, uint32_t dim, uint64_t seed, int normalize, float* d_out,
                              int device, void* stream) {
    return bguard([&]() -> int {
        BDevice g(device);
        synth_uniform_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
            n, dim, seed, normalize, d_out);
        BK(cudaGetLastError());
        return TRIM_OK;
    });
}

int trim_sample_rows(uint64_t n, uint64_t sample_n, uint64_t seed, uint64_t* rows_out) {
    if (sample_n > n)
        return berr(TRIM_EINVAL, "trim_sample_rows: sample_n > n");
    return bguard([&]() -> int {
        const auto r = sample_rows(n, sample_n, seed);
        std::memcpy(rows_out, r.data(), sizeof(uint64_t) * sample_n);
        return TRIM_OK;
    });
}

int trim_assign_device(const float* d_x, uint64_t n, uint32_t dim, const float* d_cent, uint32_t k,
                       uint32_t* d_assign, float* d_dist, int device, void* stream) {
    if (k == 0 || dim == 0)
        return berr(TRIM_EINVAL, "nearest_centroid: need k >= 1 and dim >= 1");
    return bguard([&]() -> int {
        BDevice g(device);
        launch_assign(d_x, n, dim, d_cent, k, d_assign, d_dist, static_cast<cudaStream_t>(stream));
        return TRIM_OK;
    });
}

int trim_kmeans_device(const float* d_x, uint64_t n, uint32_t dim, uint32_t k, uint32_t iters,
                       uint64_t seed, float* d_centroids, int device) {
    if (k == 0 || n < k)
        return berr(TRIM_EINVAL, "kmeans: need at least k training points");
    return bguard([&]() -> int {
        BDevice g(device);
        cudaStream_t st;
        BK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        try {
            kmeans_device(d_x, n, dim, k, iters, seed, d_centroids, st);
        } catch (...) {
            cudaStreamDestroy(st);
            throw;
        }
        cudaStreamDestroy(st);
        return TRIM_OK;
    });
}

int trim_pq_train_device(const float* d_x, uint64_t n, uint32_t dim, uint32_t m, uint32_t ksub,
                         uint32_t iters, uint64_t seed, uint64_t train_sample, uint32_t* sub_dims_out,
                         float* d_centroids_out, int device) {
    if (m == 0 || m > dim)
        return berr(TRIM_EINVAL, "PqParams: need 1 <= m <= dim");
    if (ksub == 0 || ksub > 256)
        return berr(TRIM_EINVAL, "PqParams: need 1 <= c <= 256 for byte codes");
    if (iters == 0)
        return berr(TRIM_EINVAL, "PqParams: kmeans_iters must be positive");
    uint64_t sn = train_sample ? train_sample : std::min<uint64_t>(n, 100ull * ksub);
    sn = std::min(sn, n);
    if (sn < ksub)
        return berr(TRIM_EINVAL, "pq::train: need at least c training rows");
    return bguard([&]() -> int {
        BDevice g(device);
        // pq.hpp:56-62 split; pq.hpp:72-80 sample
        std::vector<uint32_t> sub(m, dim / m);
        for (uint32_t j = 0; j < dim % m; ++j)
            ++sub[j];
        std::vector<uint64_t> rows;
        if (sn < n) {
            rows = sample_rows(n, sn, seed ^ 0x9e3779b97f4a7c15ull);
        } else {
            rows.resize(n);
            std::iota(rows.begin(), rows.end(), 0);
        }
        cudaStream_t st;
        BK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        try {
            DArr<uint64_t> drows(sn);
            BK(cudaMemcpy(drows.p, rows.data(), sizeof(uint64_t) * sn, cudaMemcpyHostToDevice));
            uint32_t off = 0;
            const uint32_t maxsd = *std::max_element(sub.begin(), sub.end());
            DArr<float> slice(sn * maxsd);
            for (uint32_t j = 0; j < m; ++j) {
                const uint32_t sd = sub[j];
                gather_rows_kernel<<<static_cast<unsigned>((sn * sd + 255) / 256), 256, 0, st>>>(
                    d_x, dim, off, sd, drows.p, sn, slice.p);
                BK(cudaGetLastError());
                kmeans_device(slice.p, sn, sd, ksub, iters, seed + 0x51edull * j,
                              d_centroids_out + static_cast<size_t>(ksub) * off, st);
                off += sd;
            }
        } catch (...) {
            cudaStreamDestroy(st);
            throw;
        }
        BK(cudaStreamSynchronize(st));
        cudaStreamDestroy(st);
        std::memcpy(sub_dims_out, sub.data(), sizeof(uint32_t) * m);
        return TRIM_OK;
    });
}

int trim_pq_encode_device(const float* d_x, uint64_t n, uint32_t dim, uint32_t m, uint32_t ksub,
                          const uint32_t* sub_dims, const float* d_centroids, uint8_t* d_codes,
                          uint32_t code_stride, float* d_lx, int device, void* stream) {
    if (m == 0 || ksub == 0 || ksub > 256 || code_stride < m)
        return berr(TRIM_EINVAL, "pq::encode: bad codebook shape");
    return bguard([&]() -> int {
        BDevice g(device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        std::vector<uint32_t> off(m);
        uint32_t s = 0;
        for (uint32_t j = 0; j < m; ++j) {
            off[j] = s;
            s += sub_dims[j];
        }
        if (s != dim)
            return berr(TRIM_EDATA, "codebook sub_dims do not sum to dim");
        std::vector<uint16_t> dsub(dim);
        std::vector<uint32_t> dbase(dim);
        std::vector<uint8_t> dsd(dim);
        for (uint32_t j = 0; j < m; ++j)
            for (uint32_t t = 0; t < sub_dims[j]; ++t) {
                dsub[off[j] + t] = static_cast<uint16_t>(j);
                dbase[off[j] + t] = ksub * off[j] + t;
                dsd[off[j] + t] = static_cast<uint8_t>(sub_dims[j]);
            }
        for (uint32_t j = 0; j < m; ++j)
            if (sub_dims[j] > 255)
                return berr(TRIM_EINVAL, "pq::encode: sub_dim > 255 unsupported");
        DArr<uint32_t> dsubd(m), doff(m), ddbase(dim);
        DArr<uint16_t> ddsub(dim);
        DArr<uint8_t> ddsd(dim);
        BK(cudaMemcpy(dsubd.p, sub_dims, sizeof(uint32_t) * m, cudaMemcpyHostToDevice));
        BK(cudaMemcpy(doff.p, off.data(), sizeof(uint32_t) * m, cudaMemcpyHostToDevice));
        BK(cudaMemcpy(ddsub.p, dsub.data(), sizeof(uint16_t) * dim, cudaMemcpyHostToDevice));
        BK(cudaMemcpy(ddbase.p, dbase.data(), sizeof(uint32_t) * dim, cudaMemcpyHostToDevice));
        BK(cudaMemcpy(ddsd.p, dsd.data(), dim, cudaMemcpyHostToDevice));
        const size_t cb_bytes = sizeof(float) * ksub * dim;
        const int in_smem = cb_bytes <= 200 * 1024;
        const size_t smem = in_smem ? cb_bytes : 0;
        BK(cudaFuncSetAttribute(encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
        encode_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, smem, st>>>(
            d_x, n, dim, m, ksub, dsubd.p, doff.p, d_centroids, in_smem, d_codes, code_stride);
        BK(cudaGetLastError());
        if (d_lx) {
            landmark_dist_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(
                d_x, n, dim, ksub, ddsub.p, ddbase.p, ddsd.p, d_centroids, d_codes, code_stride, d_lx);
            BK(cudaGetLastError());
        }
        BK(cudaStreamSynchronize(st));
        return TRIM_OK;
    });
}

int trim_ivf_lists_device(const uint32_t* d_assign, uint64_t n, uint32_t nlist, uint64_t* d_offsets,
                          uint32_t* d_ids, int device, void* stream) {
    if (nlist == 0)
        return berr(TRIM_EINVAL, "build_ivf: need 1 <= nlist <= n");
    return bguard([&]() -> int {
        BDevice g(device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        DArr<uint32_t> sk(n);
        stable_group(d_assign, n, nlist, sk.p, d_ids, st);
        list_offsets_kernel<<<(nlist + 1 + 255) / 256, 256, 0, st>>>(sk.p, n, nlist, d_offsets);
        BK(cudaGetLastError());
        BK(cudaStreamSynchronize(st));
        return TRIM_OK;
    });
}

} // extern "C"
