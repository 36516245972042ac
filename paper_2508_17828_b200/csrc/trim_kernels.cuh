// trim_kernels.cuh — sm_100a kernels of the TRIM candidate filter.
//
//   trim_probe_kernel     detail_ivf::probe_order      (ivf/ivf.hpp:173-187)
//   trim_lut_kernel       pq::build_distance_table     (pq/pq.hpp:158-172)
//   trim_knn_kernel       ivf::search_trim_ivf_knn     (ivf/ivf.hpp:243-304)
//   trim_range_kernel     ivf::search_trim_ivf_range   (ivf/ivf.hpp:308-347)
//   trim_adc_est_kernel + select/refine kernels
//                         ivf::search_baseline_ivfpq   (ivf/ivf.hpp:193-237)
//   trim_merge_kernel     top-k merge after the multi-GPU all-gather
//
// Paths are relative to /root/reference/proj/include/trimsearch.
#pragma once

#include "trim_common.cuh"

namespace trimgpu {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / kWarp;
constexpr int kChunkU = 4;                      // candidates per thread per chunk
constexpr int kChunkMax = kThreads * kChunkU;   // 1024 stream positions per chunk
constexpr int kBins = kChunkU * kWarps;         // 32 survivor bins of 32 slots
constexpr int kMaxSeg = 32;                     // lists touched by one chunk

// --------------------------------------------------------------------------
// Shared helpers: the per-query candidate stream.
//
// A query's stream is its probed lists in probe order, each list in stored
// (ascending id) order (ivf.hpp:259-262). cum[li] is the stream position of
// list li's first entry; base[li] the list's first global entry index.
// --------------------------------------------------------------------------
struct StreamSmem {
    uint32_t* cum;  // np+1
    uint64_t* base; // np
};

// Fills cum/base for the query's probe lists (warp 0 scans; others load).
__device__ __forceinline__ uint32_t load_stream(const DevIndex& ix, const uint32_t* probe,
                                                uint32_t np, StreamSmem s) {
    for (uint32_t li = threadIdx.x; li < np; li += blockDim.x) {
        const uint32_t l = probe ? probe[li] : li;
        s.base[li] = ix.list_offsets[l];
        s.cum[li + 1] = static_cast<uint32_t>(ix.list_offsets[l + 1] - ix.list_offsets[l]);
    }
    __syncthreads();
    if (threadIdx.x < kWarp) {
        const uint32_t lane = threadIdx.x;
        uint32_t carry = 0;
        for (uint32_t b = 0; b < np; b += kWarp) {
            const uint32_t li = b + lane;
            uint32_t v = li < np ? s.cum[li + 1] : 0u;
#pragma unroll
            for (int o = 1; o < kWarp; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= static_cast<uint32_t>(o))
                    v += t;
            }
            if (li < np)
                s.cum[li + 1] = carry + v;
            carry += __shfl_sync(0xffffffffu, v, kWarp - 1);
        }
        if (lane == 0)
            s.cum[0] = 0;
    }
    __syncthreads();
    return s.cum[np];
}

// ADC (pq/pq.hpp:186-192): sequential fp32 sum from 0 over j = 0..m-1 of
// lut[j][code_j]; code bytes come in 16-byte vectors.
template <int M, int KS>
__device__ __forceinline__ float adc_sum(const float* __restrict__ lut,
                                         const uint8_t* __restrict__ code, uint32_t m,
                                         uint32_t ksub) {
    constexpr int kBlocks = M > 0 ? (M + 15) / 16 : 8;
    const uint32_t mm = M > 0 ? static_cast<uint32_t>(M) : m;
    const uint32_t ks = KS > 0 ? static_cast<uint32_t>(KS) : ksub;
    const uint4* cw = reinterpret_cast<const uint4*>(code);
    float acc = 0.0f;
#pragma unroll
    for (int b = 0; b < kBlocks; ++b) {
        if (M == 0 && static_cast<uint32_t>(b * 16) >= mm)
            break;
        const uint4 w = __ldg(cw + b);
        const uint32_t words[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            const uint32_t j = static_cast<uint32_t>(b * 16 + t);
            if (j < mm) {
                const uint32_t c = (words[t >> 2] >> (8 * (t & 3))) & 0xFFu;
                acc = __fadd_rn(acc, lut[j * ks + c]);
            }
        }
    }
    return acc;
}

// --------------------------------------------------------------------------
// Warp-register top-k (replaces std::priority_queue<ScoredId>, ivf.hpp:256).
// Slot s lives in lane s%32, register s/32. Slots s >= k are disabled
// (d = -1 never wins a max); live slots start as (+inf, 0xFFFFFFFF) sentinels,
// so the first k inserts are unconditional exactly like the reference's
// seeding (ivf.hpp:264-271) and max_dis stays +inf until they are filled.
// --------------------------------------------------------------------------
template <int S>
struct WarpTopK {
    float d[S];
    uint32_t id[S];
    float wd;       // current worst (the heap top)
    uint32_t wid;
    uint32_t wslot;

    __device__ __forceinline__ void init(uint32_t k) {
        const uint32_t lane = lane_id();
#pragma unroll
        for (int r = 0; r < S; ++r) {
            const uint32_t slot = static_cast<uint32_t>(r) * kWarp + lane;
            d[r] = slot < k ? __int_as_float(0x7f800000) : -1.0f;
            id[r] = kInvalidId;
        }
        reduce_worst();
    }

    static __device__ __forceinline__ bool less3(float da, uint32_t ia, uint32_t sa, float db,
                                                 uint32_t ib, uint32_t sb) {
        return da < db || (da == db && (ia < ib || (ia == ib && sa < sb)));
    }

    __device__ __forceinline__ void reduce_worst() {
        const uint32_t lane = lane_id();
        float bd = d[0];
        uint32_t bi = id[0], bs = lane;
#pragma unroll
        for (int r = 1; r < S; ++r) {
            const uint32_t s = static_cast<uint32_t>(r) * kWarp + lane;
            if (less3(bd, bi, bs, d[r], id[r], s)) {
                bd = d[r];
                bi = id[r];
                bs = s;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float od = __shfl_xor_sync(0xffffffffu, bd, o);
            const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
            const uint32_t os = __shfl_xor_sync(0xffffffffu, bs, o);
            if (less3(bd, bi, bs, od, oi, os)) {
                bd = od;
                bi = oi;
                bs = os;
            }
        }
        wd = bd;
        wid = bi;
        wslot = bs;
    }

    // `cand < result.top()` then pop/push (ivf.hpp:277-282). Warp-uniform.
    __device__ __forceinline__ void offer(float cd, uint32_t cid) {
        if (!scored_less(cd, cid, wd, wid))
            return;
        const uint32_t lane = lane_id();
#pragma unroll
        for (int r = 0; r < S; ++r) {
            if (wslot == static_cast<uint32_t>(r) * kWarp + lane) {
                d[r] = cd;
                id[r] = cid;
            }
        }
        reduce_worst();
    }

    // Rows ascending by (dist, id) (ivf.hpp:292-302).
    __device__ __forceinline__ void store_sorted(uint32_t k, uint32_t* ids_out, float* dist_out) {
        const uint32_t lane = lane_id();
#pragma unroll
        for (int r = 0; r < S; ++r) {
            const uint32_t slot = static_cast<uint32_t>(r) * kWarp + lane;
            uint32_t rank = 0;
#pragma unroll
            for (int r2 = 0; r2 < S; ++r2) {
                for (int l = 0; l < kWarp; ++l) {
                    const float od = __shfl_sync(0xffffffffu, d[r2], l);
                    const uint32_t oi = __shfl_sync(0xffffffffu, id[r2], l);
                    const uint32_t os = static_cast<uint32_t>(r2) * kWarp + l;
                    if (os < k && scored_less(od, oi, d[r], id[r]))
                        ++rank;
                }
            }
            if (slot < k) {
                ids_out[rank] = id[r];
                dist_out[rank] = d[r];
            }
        }
    }
};

// --------------------------------------------------------------------------
// trim_knn_kernel — one CTA owns one query's candidate stream.
//
// The reference threshold max_dis is sequential state (ivf.hpp:256-287,
// SPEC.md:500). The stream is processed in chunks: the whole CTA computes
// ADC + relaxed bound for a chunk with the threshold T frozen at the chunk
// start, keeps the superset {est < T} (T only decreases, so everything the
// reference evaluates is kept), computes exact distances for the superset,
// then warp 0 replays the superset in stream order with the live threshold:
// evaluate iff est < T_live, replace iff (d,id) < top. The evaluate/prune
// decisions, counters and result set are therefore those of the reference,
// for any gamma.
// --------------------------------------------------------------------------
struct KnnParams {
    const float* queries; // nq*dim_stride
    uint64_t nq;
    uint32_t k;
    uint32_t np;             // probed lists per query
    const uint32_t* probe;   // nq*np list ids, or null when nlist == 1
    float two_gamma;
    uint32_t* ids_out;       // nq*k
    float* dist_out;         // nq*k
    unsigned long long* counters; // nq*6
    uint32_t* status;        // bit0: some query had < k probed entries
    uint32_t first_chunk;    // ramp: first chunk after the seeds
};

__host__ __device__ inline size_t knn_smem_bytes(uint32_t m, uint32_t ksub, uint32_t dim_stride,
                                                 uint32_t np) {
    size_t b = 0;
    b += sizeof(float) * m * ksub;               // lut
    b += sizeof(float) * dim_stride;             // query
    b = (b + 15) & ~size_t(15);
    b += sizeof(uint64_t) * np;                  // base
    b += sizeof(uint32_t) * (np + 1);            // cum
    b = (b + 15) & ~size_t(15);
    b += sizeof(uint32_t) * kChunkMax * 3;       // survivors: entry/id, est, d
    b += sizeof(int64_t) * kMaxSeg + sizeof(uint32_t) * kMaxSeg; // segments
    b += sizeof(uint32_t) * (kBins + 8);         // bin counts + scalars
    return b;
}

template <int M, int KS, int S>
__global__ void __launch_bounds__(kThreads)
trim_knn_kernel(DevIndex ix, KnnParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t q = blockIdx.x;
    if (q >= p.nq)
        return;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;

    float* qv = reinterpret_cast<float*>(smem); // dim_stride % 4 == 0: lut stays 16B-aligned
    float* lut = qv + ix.dim_stride;
    size_t off = sizeof(float) * (ix.m * ix.ksub + ix.dim_stride);
    off = (off + 15) & ~size_t(15);
    StreamSmem st;
    st.base = reinterpret_cast<uint64_t*>(smem + off);
    off += sizeof(uint64_t) * p.np;
    st.cum = reinterpret_cast<uint32_t*>(smem + off);
    off += sizeof(uint32_t) * (p.np + 1);
    off = (off + 15) & ~size_t(15);
    uint32_t* s_e = reinterpret_cast<uint32_t*>(smem + off); // entry index, then id
    float* s_est = reinterpret_cast<float*>(s_e + kChunkMax);
    float* s_d = s_est + kChunkMax;
    int64_t* seg_delta = reinterpret_cast<int64_t*>(s_d + kChunkMax);
    uint32_t* seg_rel = reinterpret_cast<uint32_t*>(seg_delta + kMaxSeg);
    uint32_t* bin_cnt = seg_rel + kMaxSeg;
    uint32_t* scal = bin_cnt + kBins; // [0]=T bits [1]=cn [2]=nseg [3]=li cursor

    // query vector (rows padded to dim_stride with zeros)
    const float* qg = p.queries + static_cast<size_t>(q) * ix.dim_stride;
    for (uint32_t i = tid; i < ix.dim_stride; i += kThreads)
        qv[i] = qg[i];
    __syncthreads();
    build_lut_smem(ix, qv, lut);
    const uint32_t total = load_stream(ix, p.probe ? p.probe + static_cast<size_t>(q) * p.np : nullptr,
                                       p.np, st); // includes a barrier

    WarpTopK<S> topk;
    uint64_t dc = 0;
    if (warp == 0)
        topk.init(p.k);
    if (tid == 0) {
        scal[0] = __float_as_uint(__int_as_float(0x7f800000));
        scal[3] = 0;
    }
    __syncthreads();

    uint32_t pos = 0;
    uint32_t chunk_want = p.first_chunk;
    while (pos < total) {
        // ---- segment table for [pos, pos+cn): warp 0 ----
        if (warp == 0) {
            const uint32_t first = pos < p.k ? max(p.k - pos, chunk_want) : chunk_want;
            const uint32_t want_end = min(total, pos + min(first, static_cast<uint32_t>(kChunkMax)));
            const uint32_t li0 = scal[3];
            const uint32_t li = li0 + lane;
            const bool in = li < p.np;
            const uint32_t c0 = in ? st.cum[li] : total;
            const uint32_t c1 = in ? st.cum[li + 1] : total;
            const uint32_t sb = max(c0, pos);
            const bool nonempty = in && c0 < want_end && c1 > sb;
            const uint32_t mask = __ballot_sync(0xffffffffu, nonempty);
            const uint32_t cover = (li0 + kWarp < p.np) ? st.cum[li0 + kWarp] : total;
            const uint32_t end = min(want_end, cover);
            if (nonempty) {
                const uint32_t slot = __popc(mask & ((1u << lane) - 1u));
                seg_rel[slot] = sb - pos;
                seg_delta[slot] = static_cast<int64_t>(st.base[li]) - static_cast<int64_t>(c0);
            }
            const uint32_t consumed = __popc(__ballot_sync(0xffffffffu, in && c1 <= end));
            if (lane == 0) {
                scal[1] = end - pos;
                scal[2] = __popc(mask);
                scal[3] = li0 + consumed;
            }
        }
        __syncthreads(); // (A) segments, cn, T

        const uint32_t cn = scal[1];
        const uint32_t nseg = scal[2];
        const float T = __uint_as_float(scal[0]);

        // ---- ADC + relaxed bound for the chunk, threshold frozen ----
        uint32_t e_u[kChunkU];
        float est_u[kChunkU];
        uint32_t bal_u[kChunkU];
#pragma unroll
        for (int u = 0; u < kChunkU; ++u) {
            const uint32_t r = static_cast<uint32_t>(u) * kThreads + tid;
            bool surv = false;
            e_u[u] = 0;
            est_u[u] = 0.0f;
            if (r < cn) {
                uint32_t s = 0;
                while (s + 1 < nseg && seg_rel[s + 1] <= r)
                    ++s;
                const uint32_t pp = pos + r;
                const uint32_t e = static_cast<uint32_t>(static_cast<int64_t>(pp) + seg_delta[s]);
                e_u[u] = e;
                if (pp < p.k) {
                    // seed (ivf.hpp:264-271): evaluated unconditionally, no ADC
                    est_u[u] = __int_as_float(0xff800000);
                    surv = true;
                } else {
                    const float a = adc_sum<M, KS>(lut, ix.codes + static_cast<size_t>(e) * ix.code_stride,
                                                   ix.m, ix.ksub);
                    const float est = relaxed_lb(__fsqrt_rn(a), __ldg(ix.lx + e), p.two_gamma);
                    est_u[u] = est;
                    surv = est < T;
                }
            }
            bal_u[u] = __ballot_sync(0xffffffffu, surv);
            if (surv) {
                const uint32_t slot = (static_cast<uint32_t>(u) * kWarps + warp) * kWarp +
                                      __popc(bal_u[u] & ((1u << lane) - 1u));
                s_e[slot] = e_u[u];
                s_est[slot] = est_u[u];
            }
            if (lane == 0)
                bin_cnt[u * kWarps + warp] = __popc(bal_u[u]);
        }
        __syncthreads(); // (B) survivors + bin counts

        // ---- exact distances of the superset (lane per survivor) ----
#pragma unroll
        for (int u = 0; u < kChunkU; ++u) {
            const uint32_t g = static_cast<uint32_t>(u) * kThreads + tid;
            const uint32_t b = g >> 5;
            if ((g & 31u) < bin_cnt[b]) {
                const uint32_t id = __ldg(ix.list_ids + s_e[g]);
                const float* row = ix.vectors + static_cast<size_t>(id - ix.id_base) * ix.dim_stride;
                s_d[g] = euclid_sq_vec4(qv, row, ix.dim);
                s_e[g] = id;
            }
        }
        __syncthreads(); // (C) distances

        // ---- in-order replay with the live threshold: warp 0 ----
        if (warp == 0) {
            const uint32_t nz = __ballot_sync(0xffffffffu, bin_cnt[lane] != 0);
            uint32_t bins = nz;
            while (bins) {
                const uint32_t b = __ffs(bins) - 1;
                bins &= bins - 1;
                const uint32_t cnt = bin_cnt[b];
                for (uint32_t i = 0; i < cnt; ++i) {
                    const uint32_t g = b * kWarp + i;
                    const float est = s_est[g];
                    if (est < topk.wd) { // ivf.hpp:275 — prune on tie
                        ++dc;
                        topk.offer(s_d[g], s_e[g]);
                    }
                }
            }
            if (lane == 0)
                scal[0] = __float_as_uint(topk.wd);
        }
        pos += cn;
        chunk_want = min(chunk_want * 2u, static_cast<uint32_t>(kChunkMax));
        __syncthreads(); // (D) T published, buffers free
    }

    if (warp == 0) {
        uint32_t* io = p.ids_out + static_cast<size_t>(q) * p.k;
        float* dout = p.dist_out + static_cast<size_t>(q) * p.k;
        if (total < p.k) {
            for (uint32_t i = lane; i < p.k; i += kWarp) {
                io[i] = kInvalidId;
                dout[i] = __int_as_float(0x7f800000);
            }
            if (lane == 0 && p.status)
                atomicOr(p.status, 1u);
        } else {
            topk.store_sorted(p.k, io, dout);
        }
        if (lane == 0 && p.counters) {
            unsigned long long* c = p.counters + static_cast<size_t>(q) * 6;
            const uint64_t evaluated = total;
            const uint64_t seeds = min(static_cast<uint64_t>(p.k), evaluated);
            c[0] = dc;                       // dc
            c[1] = evaluated - seeds;        // edc
            c[2] = evaluated - dc;           // pruned
            c[3] = evaluated;                // evaluated
            c[4] = 0;                        // hops
            c[5] = ix.nlist;                 // coarse_dc (probe_order always runs)
        }
    }
}

// --------------------------------------------------------------------------
// trim_range_kernel — order-free (ivf.hpp:323-340 has no running state).
// grid (slices, nq). Each CTA scans one slice of one query's stream:
// evaluate iff est <= r^2, member iff d <= r^2; members are appended as
// sortable (d,id) keys to the query's result pool.
// --------------------------------------------------------------------------
struct RangeParams {
    const float* queries;
    uint64_t nq;
    const float* radius_sq; // nq
    uint32_t np;
    const uint32_t* probe;
    float two_gamma;
    uint32_t slice;          // stream positions per CTA
    uint32_t cap;            // pool entries per query
    unsigned long long* keys;  // nq*cap
    unsigned int* count;       // nq (members)
    unsigned long long* dc;    // nq (exact evaluations)
    unsigned long long* evaluated; // nq (stream length), written by slice 0
};

__host__ __device__ inline size_t range_smem_bytes(uint32_t m, uint32_t ksub, uint32_t dim_stride,
                                                   uint32_t np) {
    size_t b = 0;
    b += sizeof(float) * m * ksub;
    b += sizeof(float) * dim_stride;
    b = (b + 15) & ~size_t(15);
    b += sizeof(uint64_t) * np;
    b += sizeof(uint32_t) * (np + 1);
    b = (b + 15) & ~size_t(15);
    b += sizeof(uint32_t) * kChunkMax; // survivor entries
    b += sizeof(uint32_t) * 8;
    return b;
}

template <int M, int KS>
__global__ void __launch_bounds__(kThreads)
trim_range_kernel(DevIndex ix, RangeParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t q = blockIdx.y;
    const uint32_t tid = threadIdx.x;
    float* qv = reinterpret_cast<float*>(smem); // dim_stride % 4 == 0: lut stays 16B-aligned
    float* lut = qv + ix.dim_stride;
    size_t off = sizeof(float) * (ix.m * ix.ksub + ix.dim_stride);
    off = (off + 15) & ~size_t(15);
    StreamSmem st;
    st.base = reinterpret_cast<uint64_t*>(smem + off);
    off += sizeof(uint64_t) * p.np;
    st.cum = reinterpret_cast<uint32_t*>(smem + off);
    off += sizeof(uint32_t) * (p.np + 1);
    off = (off + 15) & ~size_t(15);
    uint32_t* s_e = reinterpret_cast<uint32_t*>(smem + off);
    uint32_t* scal = s_e + kChunkMax; // [0] survivor count

    const float* qg = p.queries + static_cast<size_t>(q) * ix.dim_stride;
    for (uint32_t i = tid; i < ix.dim_stride; i += kThreads)
        qv[i] = qg[i];
    const uint32_t total = load_stream(ix, p.probe ? p.probe + static_cast<size_t>(q) * p.np : nullptr,
                                       p.np, st);
    const uint32_t begin = blockIdx.x * p.slice;
    if (blockIdx.x == 0 && tid == 0)
        p.evaluated[q] = total;
    if (begin >= total)
        return;
    const uint32_t end = min(total, begin + p.slice);
    build_lut_smem(ix, qv, lut);
    const float r2 = p.radius_sq[q];

    // list cursor: first list whose range contains `begin`
    uint32_t li = 0;
    {
        uint32_t lo = 0, hi = p.np; // find last li with cum[li] <= begin
        while (lo + 1 < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (st.cum[mid] <= begin)
                lo = mid;
            else
                hi = mid;
        }
        li = lo;
    }
    uint32_t dc_local = 0;
    if (tid == 0)
        scal[0] = 0;
    __syncthreads();

    for (uint32_t pos = begin; pos < end; pos += kChunkMax) {
        const uint32_t cn = min(static_cast<uint32_t>(kChunkMax), end - pos);
#pragma unroll
        for (int u = 0; u < kChunkU; ++u) {
            const uint32_t r = static_cast<uint32_t>(u) * kThreads + tid;
            if (r < cn) {
                const uint32_t pp = pos + r;
                uint32_t l = li;
                while (st.cum[l + 1] <= pp)
                    ++l;
                const uint32_t e = static_cast<uint32_t>(st.base[l] + (pp - st.cum[l]));
                const float a = adc_sum<M, KS>(lut, ix.codes + static_cast<size_t>(e) * ix.code_stride,
                                               ix.m, ix.ksub);
                const float est = relaxed_lb(__fsqrt_rn(a), __ldg(ix.lx + e), p.two_gamma);
                if (est <= r2) {
                    const uint32_t slot = atomicAdd(&scal[0], 1u);
                    s_e[slot] = e;
                }
            }
        }
        __syncthreads();
        const uint32_t ns = scal[0];
        dc_local += ns;
        for (uint32_t i = tid; i < ns; i += kThreads) {
            const uint32_t id = __ldg(ix.list_ids + s_e[i]);
            const float* row = ix.vectors + static_cast<size_t>(id - ix.id_base) * ix.dim_stride;
            const float d = euclid_sq_vec4(qv, row, ix.dim);
            if (d <= r2) {
                const uint32_t slot = atomicAdd(p.count + q, 1u);
                if (slot < p.cap)
                    p.keys[static_cast<size_t>(q) * p.cap + slot] = scored_key(d, id);
            }
        }
        // advance the list cursor past lists fully before the next chunk
        while (li + 1 < p.np && st.cum[li + 1] <= pos + cn)
            ++li;
        __syncthreads();
        if (tid == 0)
            scal[0] = 0;
        __syncthreads();
    }
    if (tid == 0 && dc_local)
        atomicAdd(p.dc + q, static_cast<unsigned long long>(dc_local));
}

#ifndef TRIM_M // non-template kernels: compiled once, in trim_capi.cu
// --------------------------------------------------------------------------
// trim_probe_kernel — probe_order (ivf.hpp:173-187): coarse distances in the
// reference's arithmetic, sorted by (dist, list id) in shared memory, first
// np ids out. One CTA per query.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
trim_probe_kernel(DevIndex ix, const float* queries, uint64_t nq, uint32_t np, uint32_t nl_pow2,
                  uint32_t* probe_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t q = blockIdx.x;
    float* qv = reinterpret_cast<float*>(smem);
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem + sizeof(float) * ((ix.dim_stride + 3) & ~3u));
    const float* qg = queries + static_cast<size_t>(q) * ix.dim_stride;
    for (uint32_t i = threadIdx.x; i < ix.dim_stride; i += blockDim.x)
        qv[i] = qg[i];
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < nl_pow2; c += blockDim.x) {
        if (c < ix.nlist) {
            const float d = euclid_sq_vec4(qv, ix.coarse + static_cast<size_t>(c) * ix.dim_stride, ix.dim);
            keys[c] = scored_key(d, c);
        } else {
            keys[c] = ~0ull;
        }
    }
    __syncthreads();
    // bitonic sort, ascending
    for (uint32_t size = 2; size <= nl_pow2; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < nl_pow2 / 2; i += blockDim.x) {
                const uint32_t lo = 2 * i - (i & (stride - 1));
                const uint32_t hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t a = keys[lo], b = keys[hi];
                if ((a > b) == up) {
                    keys[lo] = b;
                    keys[hi] = a;
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t i = threadIdx.x; i < np; i += blockDim.x)
        probe_out[static_cast<size_t>(q) * np + i] = static_cast<uint32_t>(keys[i] & 0xffffffffu);
}

// pq::build_distance_table to global memory (one CTA per query).
__global__ void __launch_bounds__(kThreads)
trim_lut_kernel(DevIndex ix, const float* queries, float* lut_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    float* qv = reinterpret_cast<float*>(smem);
    const uint32_t q = blockIdx.x;
    for (uint32_t i = threadIdx.x; i < ix.dim_stride; i += blockDim.x)
        qv[i] = queries[static_cast<size_t>(q) * ix.dim_stride + i];
    __syncthreads();
    build_lut_smem(ix, qv, lut_out + static_cast<size_t>(q) * ix.m * ix.ksub);
}

// Unpack sorted keys into (ids, dist) at the compacted offsets.
__global__ void trim_unpack_keys_kernel(const unsigned long long* keys, uint32_t cap,
                                        const uint64_t* offsets, uint64_t nq, uint32_t* ids,
                                        float* dist) {
    const uint32_t q = blockIdx.x;
    const uint64_t o = offsets[q], n = offsets[q + 1] - o;
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const unsigned long long key = keys[static_cast<size_t>(q) * cap + i];
        ids[o + i] = static_cast<uint32_t>(key & 0xffffffffu);
        dist[o + i] = __uint_as_float(static_cast<uint32_t>(key >> 32));
    }
}

// Multi-GPU merge: k smallest (dist, id) of nshards*k candidates per query.
__global__ void __launch_bounds__(kThreads)
trim_merge_kernel(const float* dist, const uint32_t* ids, uint32_t nshards, uint64_t nq,
                  uint32_t k, uint32_t n_pow2, float* dist_out, uint32_t* ids_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
    const uint32_t q = blockIdx.x;
    const uint32_t n = nshards * k;
    for (uint32_t i = threadIdx.x; i < n_pow2; i += blockDim.x) {
        uint64_t key = ~0ull;
        if (i < n) {
            const uint32_t s = i / k, j = i % k;
            const size_t src = (static_cast<size_t>(s) * nq + q) * k + j;
            if (ids[src] != kInvalidId)
                key = scored_key(dist[src], ids[src]);
        }
        keys[i] = key;
    }
    __syncthreads();
    for (uint32_t size = 2; size <= n_pow2; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < n_pow2 / 2; i += blockDim.x) {
                const uint32_t lo = 2 * i - (i & (stride - 1));
                const uint32_t hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t a = keys[lo], b = keys[hi];
                if ((a > b) == up) {
                    keys[lo] = b;
                    keys[hi] = a;
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
        const uint64_t key = keys[i];
        ids_out[static_cast<size_t>(q) * k + i] = key == ~0ull ? kInvalidId : static_cast<uint32_t>(key);
        dist_out[static_cast<size_t>(q) * k + i] =
            key == ~0ull ? __int_as_float(0x7f800000) : __uint_as_float(static_cast<uint32_t>(key >> 32));
    }
}

#endif // TRIM_M

} // namespace trimgpu
