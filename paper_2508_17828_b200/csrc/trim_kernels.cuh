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

#include "trim_adc.cuh"
#include "trim_common.cuh"

namespace trimgpu {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / kWarp;
constexpr int kBaselineSlice = 512;             // IVFPQ baseline: stream positions per slice unit
constexpr int kRangeU = 4;                      // range: candidates per thread per chunk
constexpr int kRangeChunk = kThreads * kRangeU; // 1024

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

    __device__ __forceinline__ void init(uint32_t k, void* = nullptr) {
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

    // Rows ascending by (dist, id) (ivf.hpp:292-302). Unfilled slots (fewer
    // than k entries offered: a shard whose stream is shorter than k) keep their
    // (+inf, 0xFFFFFFFF) sentinels and sort last; the slot index breaks their ties.
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
                    if (os < k && less3(od, oi, os, d[r], id[r], slot))
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
// Shared-memory top-k for k > 256 (the reference's priority_queue has no cap,
// ivf.hpp:256-302). Entries are 64-bit keys (dist bits << 32 | id): dist >= 0,
// so key order is ScoredId order (core/ground_truth.hpp:39-50) and
// `(d, id) < top` is `key < worst key`. Slots start as (+inf, 0xFFFFFFFF)
// sentinels like WarpTopK's; the replay warp owns the array (slot s: lane
// s % 32), tracks the worst by a lane scan + butterfly, and sorts the final
// rows with a warp bitonic sort in place (padding keys ~0 sort last).
// --------------------------------------------------------------------------
constexpr uint32_t kSmemTopKMax = 4096;
__host__ __device__ inline uint32_t smem_topk_slots(uint32_t k) {
    uint32_t p = 32;
    while (p < k)
        p <<= 1;
    return p;
}

struct SmemTopK {
    unsigned long long* key; // smem_topk_slots(k) entries
    uint32_t k, P;
    float wd;
    uint32_t wid;
    uint32_t wslot;
    unsigned long long wkey;

    __device__ __forceinline__ void init(uint32_t k_, void* buf) {
        key = static_cast<unsigned long long*>(buf);
        k = k_;
        P = smem_topk_slots(k_);
        const uint32_t lane = lane_id();
        for (uint32_t s = lane; s < P; s += kWarp)
            key[s] = s < k ? (static_cast<unsigned long long>(0x7f800000u) << 32) | kInvalidId : ~0ull;
        __syncwarp();
        reduce_worst();
    }
    __device__ __forceinline__ void reduce_worst() {
        const uint32_t lane = lane_id();
        unsigned long long b = 0;
        uint32_t bs = lane;
        for (uint32_t s = lane; s < k; s += kWarp) {
            const unsigned long long v = key[s];
            if (v > b || s == lane) {
                b = v;
                bs = s;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ob = __shfl_xor_sync(0xffffffffu, b, o);
            const uint32_t os = __shfl_xor_sync(0xffffffffu, bs, o);
            if (ob > b || (ob == b && os > bs)) {
                b = ob;
                bs = os;
            }
        }
        wkey = b;
        wslot = bs;
        wd = __uint_as_float(static_cast<uint32_t>(b >> 32));
        wid = static_cast<uint32_t>(b);
    }
    // `cand < result.top()` then pop/push (ivf.hpp:277-282). Warp-uniform.
    __device__ __forceinline__ void offer(float cd, uint32_t cid) {
        const unsigned long long c = (static_cast<unsigned long long>(__float_as_uint(cd)) << 32) | cid;
        if (!(c < wkey))
            return;
        if (lane_id() == (wslot & 31u))
            key[wslot] = c;
        __syncwarp();
        reduce_worst();
    }
    // Rows ascending by (dist, id) (ivf.hpp:292-302), sentinels last.
    __device__ __forceinline__ void store_sorted(uint32_t, uint32_t* ids_out, float* dist_out) {
        const uint32_t lane = lane_id();
        for (uint32_t size = 2; size <= P; size <<= 1)
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                for (uint32_t i = lane; i < P / 2; i += kWarp) {
                    const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                    const bool up = (lo & size) == 0;
                    const unsigned long long a = key[lo], b = key[hi];
                    if ((a > b) == up) {
                        key[lo] = b;
                        key[hi] = a;
                    }
                }
                __syncwarp();
            }
        for (uint32_t s = lane; s < k; s += kWarp) {
            ids_out[s] = static_cast<uint32_t>(key[s]);
            dist_out[s] = __uint_as_float(static_cast<uint32_t>(key[s] >> 32));
        }
    }
};

template <int S>
struct TopKOf {
    using type = WarpTopK<S>;
};
template <>
struct TopKOf<0> {
    using type = SmemTopK;
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
    float adc_eps;           // adc_rel_eps(m)
    float omg_hi;            // 1 - gamma, rounded up
    uint32_t* ids_out;       // nq*k
    float* dist_out;         // nq*k
    unsigned long long* counters; // nq*6
    uint32_t* status;        // bit0: some query had < k probed entries
    uint32_t skip_lists;     // 1: apply the list-level bound (list_lower_bound)
    float omg_lo;            // 1 - gamma, rounded down
    float kq1;               // 1 - relative error bound of the fp32 coarse distance
    float kq2;               // 1 - relative error bound of sqrt(reference ADC)
    float kest;              // 1 - relative error bound of relaxed_lb's evaluation
    unsigned long long* skipped; // positions skipped by the list bound (diagnostic)
    unsigned long long* timeline; // nq*kTimeline phase stamps/cycle counts (perf probe only), or null
    // flat scans: tensor-core distance bounds (trim_flat_mma.cuh), or null
    const __nv_bfloat16* dap; // nq x dap_ld: rigorous lower bound of |q - x|^2 (tf32 D~ - E, rounded down)
    uint64_t dap_ld;
    const uint32_t* plan;  // per-query setup records (trim_knn_setup_kernel), or null: set up in the kernel
    uint32_t topk_off;     // k > 256: byte offset of the SmemTopK keys in dynamic shared memory
    // segmented flat scans (trim_knn_seg_plan_kernel): per-query entry tables, tab_cap words each
    const uint32_t* tab;
    uint32_t tab_cap;
    uint32_t mode_sel; // PRE kernel without SEG: the record mode this launch serves (0, or 2 = a continue round)
    float stage_c1;    // <= γ(2-γ) (StageCut)
    float stage_ka;    // >= 1 / ((1 - adc_eps)(1 - 2^-24)^2), +inf when adc_eps >= 1 (StageCut)
};

// Per-query setup record written by trim_knn_setup_kernel (u32 words): the
// stream length, the seeds' (d, id) in stream order, the seeded threshold and
// the compacted stream after the list-level plan — what the replay warp of
// trim_knn_kernel otherwise computes itself before the workers may start.
struct KnnPlanLayout {
    uint32_t cum, base, sd, sid, words;
    // header: [0] total [1] nseed [2] nk [3] total2 [4] T0 bits [5] dc so far (the seeds, or
    // everything before a resumed scan) [6] entries evaluated unconditionally (edc = evaluated
    // - this) [7] mode: 0 = runs in cum/base, 1 = entry table of a segmented block stream (SEG kernel),
    // 2 = runs in cum/base of a continue round (more rows in order, then planned again)
    __host__ __device__ static KnnPlanLayout of(uint32_t np, uint32_t k) {
        KnnPlanLayout o;
        o.cum = 8;
        o.base = (o.cum + np + 1 + 1) & ~1u; // u64-aligned
        o.sd = o.base + 2 * np;
        o.sid = o.sd + k;
        o.words = (o.sid + k + 1) & ~1u;
        return o;
    }
};

constexpr uint32_t kTimeline = 32;
// Phase instrumentation of trim_knn_kernel, compiled only into the perf-probe
// build of the library (make timeline -> libtrim_b200_tl.so).
#ifdef TRIM_TIMELINE
#define TRIM_TL(...) __VA_ARGS__
#else
#define TRIM_TL(...)
#endif
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Warp-specialised pipeline: warp 0 replays, warps 1..kWorkers filter.
constexpr uint32_t kWorkers = kWarps - 1;          // 7
constexpr uint32_t kLaneU = 1;                     // candidates per worker lane per chunk
constexpr uint32_t kPerWorker = kWarp * kLaneU;    // 32 stream positions per worker per chunk
constexpr uint32_t kChunkW = kWorkers * kPerWorker; // 224 stream positions per chunk
#ifndef TRIM_KRING
#define TRIM_KRING 6
#endif
constexpr uint32_t kRing = TRIM_KRING;             // chunk buffers in flight
#ifndef TRIM_STAGE_CUT
#define TRIM_STAGE_CUT 1   // kNN workers: one-compare stage tests every 8 lookups (StageCut); 0: StageCheck
#endif
#ifndef TRIM_SEG_NOSTAGE
#define TRIM_SEG_NOSTAGE 0 // 1: the table-driven flat kernel (SEG) also runs without stages (spills at m = 48)
#endif
#ifndef TRIM_QUAD_L2
#define TRIM_QUAD_L2 1     // members' exact L2 by lane quads (euclid_sq_quad), 8 rows per warp pass
#endif
static_assert(kLaneU == 1, "bin_mask records one ballot per worker chunk");

// Warps per filter CTA by code length: a long code (m = 120: a 128 KB LUT, one
// CTA per SM) gets 16 warps (15 workers, 128 registers: measured best of 8/16/24/32)
// so the SM is not left with 8 warps; otherwise 8 (3 CTAs per SM).
#ifndef TRIM_WIDE_WARPS
#define TRIM_WIDE_WARPS 16
#endif
#ifndef TRIM_NARROW_WARPS
#define TRIM_NARROW_WARPS 8
#endif
#ifndef TRIM_M16_WARPS
#define TRIM_M16_WARPS 6 // config 1 (m = 16): 4 CTAs x 6 warps measured 3% over 3 x 8, 4 warps 24% slower
#endif
__host__ __device__ constexpr uint32_t knn_warps(int mt) {
    return mt > 64 ? TRIM_WIDE_WARPS : (mt == 0 ? kWarps : (mt == 16 ? TRIM_M16_WARPS : TRIM_NARROW_WARPS));
}
// CTAs per SM the register budget is set for (24 warps per SM in total)
#ifndef TRIM_NARROW_MINB
#define TRIM_NARROW_MINB 0 // > 0: CTAs per SM the register budget of the narrow (m = 48-class) shape targets
#endif
__host__ __device__ constexpr uint32_t knn_min_blocks(int mt) {
    return mt == 0 ? 2u
                   : (TRIM_NARROW_MINB > 0 && mt <= 64 && mt != 16
                          ? static_cast<uint32_t>(TRIM_NARROW_MINB)
                          : (24u / knn_warps(mt) > 0 ? 24u / knn_warps(mt) : 1u));
}
__host__ __device__ constexpr uint32_t knn_threads(int mt) { return knn_warps(mt) * kWarp; }
__host__ __device__ constexpr uint32_t knn_chunk(int mt) { return (knn_warps(mt) - 1) * kPerWorker; }

__host__ __device__ inline size_t knn_smem_bytes(int mt, uint32_t m, uint32_t dim_stride,
                                                 uint32_t np) {
    const size_t kChunkW = knn_chunk(mt), kWorkers = knn_warps(mt) - 1;
    size_t b = lut_bytes(mt, m);                 // blocked lut at offset 0
    b += sizeof(float) * dim_stride;             // query
    b += sizeof(uint64_t) * np;                  // base
    b += sizeof(uint32_t) * (np + 1);            // cum
    b = (b + 15) & ~size_t(15);
    b += sizeof(uint32_t) * kRing * kChunkW * 4; // superset bins: id, est_lo, est_hi, d
    b += sizeof(uint32_t) * kRing * kWorkers * 2; // bin counts, bin lane masks
    b = (b + 15) & ~size_t(15);
    b += sizeof(uint64_t) * (2 * kRing + 2);     // full/empty mbarriers (+2 spare)
    b += 16;                                     // published threshold, plan length
    return b;
}

__device__ __forceinline__ uint32_t saddr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(saddr(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    for (;;) {
        // suspend-time hint: the warp may sleep in hardware until the phase completes
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done)
                     : "r"(saddr(bar)), "r"(parity), "r"(1000000u)
                     : "memory");
        if (done)
            break;
    }
}
// Named hardware barriers between the replay warp and the workers (a warp
// blocked in bar.sync issues nothing, unlike an mbarrier poll).
constexpr uint32_t kBarWorkers = 1;   // workers only: LUT complete
constexpr uint32_t kBarPlan = 2;      // replay arrives: seeds + plan published
constexpr uint32_t kBarChunk0 = 3;    // replay arrives: chunk 0 replayed
__device__ __forceinline__ void named_arrive(uint32_t id, uint32_t n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_sync(uint32_t id, uint32_t n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ float ld_volatile(const float* p) {
    return *reinterpret_cast<const volatile float*>(p);
}

// --------------------------------------------------------------------------
// List-level bound. For every entry x of inverted list l the reference computes
// est = relaxed_lb(g, lx) with g = fl(sqrt(adc)) (ivf.hpp:273-275). With
// D <= |q - c_l| (coarse distance, rounded down), R_l >= |c_l - landmark(x)|
// (trim_list_meta_kernel) and the ADC's relative error folded into kq2,
// g >= G := (D - R_l) * kq2 by the triangle inequality. relaxed_lb(g, x) =
// (x - (1-γ)g)^2 + γ(2-γ)g^2 is increasing in g once g >= (1-γ)x, so if
// G >= (1-γ) xmax_l every entry of the list has
//     est >= min_{x in [xmin, xmax]} relaxed_lb(G, x)
//         =  γ(2-γ)G^2 + dist((1-γ)G, [xmin, xmax])^2
// up to the evaluation error folded into kest. Every product and sum below is
// rounded toward the safe side, so the returned L is a rigorous lower bound on
// est for all of the list's entries (0 when no bound holds).
// --------------------------------------------------------------------------
__device__ __forceinline__ float list_lower_bound(float dq, float R, float xmin, float xmax,
                                                  const KnnParams& p) {
    const float omg_hi = p.omg_hi, omg_lo = p.omg_lo;
    const float D = __fsqrt_rd(__fmul_rd(dq, p.kq1));
    const float G0 = __fsub_rd(D, R);
    if (!(G0 > 0.0f))
        return 0.0f;
    const float g = __fmul_rd(G0, p.kq2);
    if (!(g >= __fmul_ru(omg_hi, xmax))) // outside the monotone region
        return 0.0f;
    const float omg2 = fmaxf(__fmul_ru(omg_lo, omg_lo), __fmul_ru(omg_hi, omg_hi));
    if (!(omg2 <= 1.0f)) // γ(2-γ) may be negative (γ >= 2): no bound
        return 0.0f;
    const float c1 = __fsub_rd(1.0f, omg2); // γ(2-γ), rounded down
    const float t1 = __fmul_rd(__fmul_rd(g, g), c1);
    const float plo = __fmul_rd(omg_lo, g), phi = __fmul_ru(omg_hi, g); // (1-γ)g
    const float gap = fmaxf(0.0f, fmaxf(__fsub_rd(xmin, phi), __fsub_rd(plo, xmax)));
    return __fmul_rd(__fadd_rd(t1, __fmul_rd(gap, gap)), p.kest);
}

// --------------------------------------------------------------------------
// trim_knn_kernel — one CTA owns one query's candidate stream.
//
// The reference threshold max_dis is sequential state (ivf.hpp:256-287,
// SPEC.md:500). Worker warps (1..7) stream the query's candidates in chunks
// of 224 positions (warp w, lane l: position c*224 + (w-1)*32 + l), each with
// the latest threshold T the replay warp has published — any published T is
// >= the reference's running threshold at every later position, because the
// threshold only decreases. From the any-order ADC a worker derives a
// rigorous interval [lo, hi] around the reference's est (trim_adc.cuh), keeps
// the members {lo < T} and computes their exact L2. Warp 0 replays the
// chunk's members in stream order with the live threshold: evaluate iff
// est < T_live (prune on tie, ivf.hpp:275) — decided by lo >= T_live (prune)
// or hi < T_live (evaluate), and only when the interval straddles T_live by
// the reference-order ADC itself (adc_serial) — and replace iff
// (d, id) < top (ivf.hpp:277-282). The evaluate /
// prune decisions, counters and result set are therefore the reference's,
// for any gamma. Chunks flow through a ring of kRing buffers guarded by
// mbarriers (full: 224 worker-lane arrivals; empty: 32 replay-lane arrivals),
// so workers never wait for the replay except when the ring is full; the
// next chunk's codes are prefetched into registers while the current one is
// filtered.
//
// The replay warp first evaluates the k seeds (ivf.hpp:264-271) itself and
// publishes the seeded threshold, so no chunk is filtered against +inf.
// After chunk 0 (positions [0, 224)) it plans the rest of the stream from
// p0 = max(224, k): a probed list that starts at or after p0 and whose
// list_lower_bound is >= the published T is pruned as a whole (every entry
// has est >= L >= T >= T_live: the reference prunes each of them,
// ivf.hpp:275), and the remaining positions are compacted in place into
// cum/base. Chunks c >= 1 walk the compacted stream. Counters are unchanged:
// skipped entries are evaluated-and-pruned positions.
// --------------------------------------------------------------------------
// PRE: the seeds and the plan come from trim_knn_setup_kernel's record
// (p.plan); the in-kernel setup code is compiled out (fewer live registers).
//
// SEG (with PRE): a segmented block stream over a flat index
// (trim_knn_seg_plan_kernel). `ix` holds the rows regrouped by (segment of
// consecutive ids, block); the record resumes the scan after the first rows
// (top-k, counters) and the query's entry table (p.tab) lists the rows of the
// blocks the list-level bound could not prune, merged back into ascending-id
// order — the reference's stream order with the pruned blocks' rows removed —
// so stream position pp is entry tab[pp] and the pipeline below runs unchanged.
// A CTA whose record is of the other mode exits at once (both kernels are
// launched over the batch).
//
// HARD (with PRE, without SEG): the launch for the records whose bit 8 is set — the
// list-level bound dropped at least 3/4 of the stream, so what is left are the lists
// around the query, every candidate is near the threshold and the ADC runs without
// early-exit stages (StageNone); the other records are served by the HARD = false launch.
template <int M, int KS, int S, bool PRE, bool SEG = false, bool HARD = false>
__global__ void __launch_bounds__(knn_threads(M), knn_min_blocks(M))
trim_knn_kernel(DevIndex ix, KnnParams p) {
    static_assert(PRE || !SEG, "segmented streams come from a plan record");
    static_assert(!HARD || (PRE && !SEG), "HARD is a flavour of the PRE kernel");
    // this instantiation's CTA shape (knn_warps): warp 0 replays, the rest filter
    constexpr uint32_t kThreads = knn_threads(M);
    constexpr uint32_t kWorkers = knn_warps(M) - 1;
    constexpr uint32_t kChunkW = knn_chunk(M);
    unsigned char* smem = trim_dyn_smem;
    const uint32_t q = blockIdx.x;
    if (q >= p.nq)
        return;
    if constexpr (PRE) { // a record of another launch's mode or flavour: nothing to do here
        const uint32_t md = __ldg(p.plan + static_cast<size_t>(q) * KnnPlanLayout::of(p.np, p.k).words + 7);
        if ((md & 0xffu) != (SEG ? 1u : p.mode_sel) || (!SEG && ((md >> 8) & 1u) != (HARD ? 1u : 0u)))
            return;
    }
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t m = M > 0 ? static_cast<uint32_t>(M) : ix.m;

    float* lut = reinterpret_cast<float*>(smem); // offset 0
    float* qv = lut + lut_bytes(M, m) / sizeof(float);
    size_t off = lut_bytes(M, m) + sizeof(float) * ix.dim_stride;
    StreamSmem st;
    st.base = reinterpret_cast<uint64_t*>(smem + off);
    off += sizeof(uint64_t) * p.np;
    st.cum = reinterpret_cast<uint32_t*>(smem + off);
    off += sizeof(uint32_t) * (p.np + 1);
    off = (off + 15) & ~size_t(15);
    uint32_t* s_e = reinterpret_cast<uint32_t*>(smem + off);  // [kRing][kChunkW]: id
    float* s_lo = reinterpret_cast<float*>(s_e + kRing * kChunkW); // est interval
    float* s_hi = s_lo + kRing * kChunkW;
    float* s_d = s_hi + kRing * kChunkW;
    uint32_t* bin_cnt = reinterpret_cast<uint32_t*>(s_d + kRing * kChunkW); // [kRing][kWorkers]
    uint32_t* bin_mask = bin_cnt + kRing * kWorkers; // lanes of the members, [kRing][kWorkers]
    // (bins: worker w of ring slot s owns s_*[s*kChunkW + w*kPerWorker ...], in stream order)
    off = reinterpret_cast<unsigned char*>(bin_mask + kRing * kWorkers) - smem;
    off = (off + 15) & ~size_t(15);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + off);
    uint64_t* empty = full + kRing;
    uint64_t* plan = empty + kRing;
    float* s_T = reinterpret_cast<float*>(plan + 2);
    uint32_t* s_total2 = reinterpret_cast<uint32_t*>(s_T + 1);

    const float kInf = __int_as_float(0x7f800000);
    const float kNegInf = __int_as_float(0xff800000);

    TRIM_TL(unsigned long long* tl = p.timeline ? p.timeline + static_cast<size_t>(q) * kTimeline : nullptr;
            if (tl && tid == 0) {
                uint32_t smid;
                asm("mov.u32 %0, %smid;" : "=r"(smid));
                tl[0] = gtime();
                tl[6] = smid;
            })
    const float* qg = p.queries + static_cast<size_t>(q) * ix.dim_stride;
    for (uint32_t i = tid; i < ix.dim_stride; i += kThreads)
        qv[i] = qg[i];
    if (tid == 0) {
        for (uint32_t s = 0; s < kRing; ++s) {
            mbar_init(full + s, kWorkers * kWarp);
            mbar_init(empty + s, kWarp);
        }
        *s_T = kInf;
    }
    __syncthreads();
    // the stream (probe order, ascending ids) — from the setup record when
    // trim_knn_setup_kernel ran, else built here
    const uint32_t* rec = PRE ? p.plan + static_cast<size_t>(q) * KnnPlanLayout::of(p.np, p.k).words : nullptr;
    // SEG: the query's entry table (stream position -> entry of the regrouped arrays)
    [[maybe_unused]] const uint32_t* tab = SEG ? p.tab + static_cast<size_t>(q) * p.tab_cap : nullptr;
    uint32_t total;
    if constexpr (PRE) {
        const KnnPlanLayout lo = KnnPlanLayout::of(p.np, p.k);
        const uint32_t nk = __ldg(rec + 2);
        for (uint32_t i = tid; i <= nk; i += kThreads)
            st.cum[i] = __ldg(rec + lo.cum + i);
        const uint64_t* rb = reinterpret_cast<const uint64_t*>(rec + lo.base);
        for (uint32_t i = tid; i < nk; i += kThreads)
            st.base[i] = __ldg(rb + i);
        total = __ldg(rec);
        __syncthreads();
    } else {
        total = load_stream(ix, p.probe ? p.probe + static_cast<size_t>(q) * p.np : nullptr,
                            p.np, st); // ends with a barrier
    }
    // seeds [0, nseed) are the replay warp's; the candidate stream is the kept
    // part of [nseed, total), compacted into cum/base by the plan
    const uint32_t nseed = min(p.k, total);

    if (warp == 0) {
        // ------------------------------------------------ replay warp
        // (the worker warps build the LUT meanwhile)
        TRIM_TL(if (tl && lane == 0) tl[1] = gtime();)
        typename TopKOf<S>::type topk; // S = 0: k > 256, the shared-memory top-k
        topk.init(p.k, smem + p.topk_off);
        uint32_t carry = 0, nk = 0;
        if constexpr (PRE) { // seeds and plan from trim_knn_setup_kernel
            const KnnPlanLayout lo = KnnPlanLayout::of(p.np, p.k);
            for (uint32_t j = 0; j < nseed; ++j)
                topk.offer(__uint_as_float(__ldg(rec + lo.sd + j)), __ldg(rec + lo.sid + j));
            nk = __ldg(rec + 2);
            carry = __ldg(rec + 3);
            if (lane == 0) {
                *s_total2 = carry;
                *reinterpret_cast<volatile float*>(s_T) = topk.wd;
            }
        }
        // seeds (ivf.hpp:264-271): evaluated unconditionally, in stream order
        for (uint32_t b0 = 0; !PRE && b0 < nseed; b0 += kWarp) {
            const uint32_t i = b0 + lane;
            float d = 0.0f;
            uint32_t id = 0;
            if (i < nseed) {
                uint32_t li = 0;
                while (st.cum[li + 1] <= i)
                    ++li;
                const uint64_t e = st.base[li] + (i - st.cum[li]);
                id = __ldg(ix.list_ids + e);
                d = euclid_sq_vec4(qv, ix.vectors + static_cast<size_t>(id - ix.id_base) * ix.dim_stride, ix.dim,
                                   true); // the whole row in one round trip: the seeds gate every chunk
            }
            const uint32_t cnt = min(static_cast<uint32_t>(kWarp), nseed - b0);
            for (uint32_t j = 0; j < cnt; ++j)
                topk.offer(__shfl_sync(0xffffffffu, d, j), __shfl_sync(0xffffffffu, id, j));
        }
        const float T0 = topk.wd; // max_dis after the seeds
        TRIM_TL(if (tl && lane == 0) tl[2] = gtime();)
        // plan: drop every probed list after the seeds whose list_lower_bound
        // is >= T0 (>= T_live at all its positions), compact the rest in place
        const bool skip = p.skip_lists && p.probe && total > nseed;
        const uint32_t* pl = p.probe ? p.probe + static_cast<size_t>(q) * p.np : nullptr;
        for (uint32_t b0 = 0; !PRE && b0 < p.np; b0 += kWarp) {
            const uint32_t i = b0 + lane;
            uint32_t len = 0;
            uint64_t bs = 0;
            if (i < p.np) {
                const uint32_t c0 = st.cum[i], c1 = st.cum[i + 1];
                bool drop = c1 <= nseed;
                if (!drop && skip && c0 >= nseed) {
                    const uint32_t l = __ldg(pl + i);
                    const float dq = euclid_sq_vec4(qv, ix.coarse + static_cast<size_t>(l) * ix.dim_stride, ix.dim);
                    drop = list_lower_bound(dq, __ldg(ix.list_R + l), __ldg(ix.list_xmin + l),
                                            __ldg(ix.list_xmax + l), p) >= T0;
                }
                if (!drop) {
                    const uint32_t s0 = max(c0, nseed);
                    len = c1 - s0;
                    bs = st.base[i] + (s0 - c0);
                }
            }
            const uint32_t keep = __ballot_sync(0xffffffffu, len != 0);
            uint32_t v = len;
#pragma unroll
            for (int o = 1; o < kWarp; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= static_cast<uint32_t>(o))
                    v += t;
            }
            __syncwarp(); // this batch's reads precede its (lower-index) writes
            if (len != 0) {
                const uint32_t j = nk + __popc(keep & ((1u << lane) - 1u));
                st.base[j] = bs;
                st.cum[j] = carry + v - len;
            }
            carry += __shfl_sync(0xffffffffu, v, kWarp - 1);
            nk += __popc(keep);
            __syncwarp();
        }
        if (lane == 0 && !PRE) {
            st.cum[nk] = carry;
            *s_total2 = carry;
            *reinterpret_cast<volatile float*>(s_T) = T0;
            const uint32_t rest = total - nseed;
            if (p.skipped && rest != carry)
                atomicAdd(p.skipped, static_cast<unsigned long long>(rest - carry));
        }
        const uint32_t nchunks = (carry + kChunkW - 1) / kChunkW;
        const uint32_t ncum = nk;
        TRIM_TL(if (tl && lane == 0) tl[3] = gtime();)
        __syncwarp();
        named_arrive(kBarPlan, kThreads);

        uint64_t dc = PRE ? __ldg(rec + 5) : nseed;
        const uint32_t nuncond = PRE ? __ldg(rec + 6) : nseed;
        TRIM_TL(uint32_t members = 0;)
        // The reference-order est of a member whose interval straddles the live
        // threshold (rare): its compacted position from the bin's lane mask, its
        // entry from cum/base, then pq::adc_lookup + relaxed_lb.
        auto exact_est = [&](uint32_t c, uint32_t w, uint32_t i, uint32_t mask) -> float {
            for (uint32_t r = 0; r < i; ++r)
                mask &= mask - 1;
            const uint32_t pp = c * kChunkW + w * kPerWorker + (__ffs(mask) - 1);
            uint64_t e;
            if constexpr (SEG) {
                e = __ldg(tab + pp);
            } else {
                uint32_t lo = 0, hi = ncum; // largest li with cum[li] <= pp
                while (hi - lo > 1) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (st.cum[mid] <= pp)
                        lo = mid;
                    else
                        hi = mid;
                }
                e = st.base[lo] + (pp - st.cum[lo]);
            }
            const float a = adc_serial<M>(ix.codes + e * ix.code_stride, m);
            return relaxed_lb(__fsqrt_rn(a), __ldg(ix.lx + e), p.two_gamma);
        };
        TRIM_TL(unsigned long long cyc_wait = 0, cyc_busy = 0;)
        for (uint32_t c = 0; c < nchunks; ++c) {
            const uint32_t s = c % kRing;
            TRIM_TL(const unsigned long long k0 = tl ? clock64() : 0;)
            mbar_wait(full + s, (c / kRing) & 1u);
            TRIM_TL(const unsigned long long k1 = tl ? clock64() : 0;)
            // the chunk's members of all kWorkers bins, in stream order (bin w
            // before bin w+1, bin order inside), 32 at a time: lane i holds
            // member base+i of bin w at rank r
            const uint32_t* cnts = bin_cnt + s * kWorkers;
            uint32_t inc = lane < kWorkers ? cnts[lane] : 0u;
#pragma unroll
            for (uint32_t o = 1; o < kWarp; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o)
                    inc += t;
            }
            const uint32_t nmem = __shfl_sync(0xffffffffu, inc, kWorkers - 1);
            for (uint32_t base = 0; base < nmem; base += kWarp) {
                const uint32_t i = base + lane;
                const uint32_t cnt = min(static_cast<uint32_t>(kWarp), nmem - base);
                uint32_t w = 0, before = 0;
#pragma unroll
                for (uint32_t x = 0; x < kWorkers; ++x) {
                    const uint32_t ix_ = __shfl_sync(0xffffffffu, inc, x);
                    if (i >= ix_) {
                        w = x + 1;
                        before = ix_;
                    }
                }
                const uint32_t r = i - before;
                const uint32_t g = s * kChunkW + w * kPerWorker + r;
                TRIM_TL(members += cnt;)
                // Warp-parallel replay (lane i <-> member base+i): with the live
                // threshold T, a member is pruned iff lo >= T, evaluated iff hi < T
                // (ivf.hpp:275) and replaces the top iff also (d, id) < top
                // (ivf.hpp:277-282). Members up to the first one that replaces (or
                // whose interval straddles T) are decided at once; that one is
                // handled alone (it may lower T), then the rest again.
                const bool valid = lane < cnt;
                const float lo = valid ? s_lo[g] : kInf;
                const float hi = valid ? s_hi[g] : kInf;
                const float dd = valid ? s_d[g] : kInf;
                const uint32_t did = valid ? s_e[g] : kInvalidId;
                uint32_t start = 0;
                while (start < cnt) {
                    const bool mine = valid && lane >= start;
                    const bool maybe = mine && lo < topk.wd;
                    const bool sure = maybe && hi < topk.wd;
                    const bool hard = maybe && (!sure || scored_less(dd, did, topk.wd, topk.wid));
                    const uint32_t hb = __ballot_sync(0xffffffffu, hard);
                    const uint32_t f = hb ? static_cast<uint32_t>(__ffs(hb) - 1) : cnt;
                    dc += __popc(__ballot_sync(0xffffffffu, sure && lane < f));
                    if (f >= cnt)
                        break;
                    const float hf = __shfl_sync(0xffffffffu, hi, f);
                    bool ev = true;
                    if (!(hf < topk.wd)) {
                        const uint32_t wf = __shfl_sync(0xffffffffu, w, f);
                        const uint32_t rf = __shfl_sync(0xffffffffu, r, f);
                        ev = exact_est(c, wf, rf, bin_mask[s * kWorkers + wf]) < topk.wd;
                    }
                    if (ev) {
                        ++dc;
                        topk.offer(__shfl_sync(0xffffffffu, dd, f), __shfl_sync(0xffffffffu, did, f));
                    }
                    start = f + 1;
                }
            }
            if (lane == 0)
                *reinterpret_cast<volatile float*>(s_T) = topk.wd;
            __syncwarp();
            mbar_arrive(empty + s);
            if (!SEG && c == 0 && nchunks > 1) // the workers filter chunk 1 on against this threshold
                named_arrive(kBarChunk0, kThreads);
            TRIM_TL(if (tl) {
                cyc_wait += k1 - k0;
                cyc_busy += clock64() - k1;
            })
        }
        TRIM_TL(if (tl && lane == 0) {
            tl[4] = gtime();
            tl[5] = nchunks;
            tl[7] = members;
            tl[8] = cyc_wait;
            tl[9] = cyc_busy;
        })
        uint32_t* io = p.ids_out + static_cast<size_t>(q) * p.k;
        float* dout = p.dist_out + static_cast<size_t>(q) * p.k;
        // a stream shorter than k: the reference throws after the scan
        // (ivf.hpp:289-290) — status bit 0; the rows keep the partial sorted
        // top-k padded with (+inf, 0xFFFFFFFF), which an id-sharded caller merges
        // (the error is then decided on the total over the shards)
        if (total < p.k && lane == 0 && p.status)
            atomicOr(p.status, 1u);
        topk.store_sorted(p.k, io, dout);
        if (lane == 0 && p.counters) {
            unsigned long long* cc = p.counters + static_cast<size_t>(q) * 6;
            const uint64_t evaluated = total;
            cc[0] = dc;                // dc
            cc[1] = evaluated - nuncond; // edc
            cc[2] = evaluated - dc;    // pruned (including skipped lists)
            cc[3] = evaluated;         // evaluated
            cc[4] = 0;                 // hops
            cc[5] = ix.nlist;          // coarse_dc (probe_order always runs)
        }
        return;
    }

    // ---------------------------------------------------- worker warps
    TRIM_TL(const bool wtl = tl && lane == 0; // lane 0 of every worker records (worker 0: slots 10-15)
            unsigned long long wc[6] = {0, 0, 0, 0, 0, 0}; // lut, plan wait, ring wait, adc, l2, total
            unsigned long long wk = wtl ? clock64() : 0;)
    const uint32_t w = warp - 1;
    uint32_t bound = 0, nchunks = 0; // the compacted stream length, published with the plan
    uint32_t li = 0; // list cursor (positions of a lane only increase)
    struct Cand {
        FastCode<M> fc;
        float lx;
        uint32_t e;
        uint32_t kind; // 0: past the end, 2: candidate
    };
    struct Slot {
        Cand c[kLaneU];
    };
    Slot sa, sb; // double buffer in registers (static names: no local-memory indexing)
    auto fetch = [&](uint32_t c, Slot& d) {
#pragma unroll
        for (uint32_t u = 0; u < kLaneU; ++u) {
            const uint32_t pp = c * kChunkW + w * kPerWorker + u * kWarp + lane;
            Cand& x = d.c[u];
            x.kind = 0;
            x.e = 0;
            x.lx = 0.0f;
            if (c < nchunks && pp < bound) {
                if constexpr (SEG) { // the plan's entry table: the kept rows in ascending-id order
                    x.e = __ldg(tab + pp);
                } else {
                    while (st.cum[li + 1] <= pp)
                        ++li;
                    x.e = static_cast<uint32_t>(st.base[li] + (pp - st.cum[li]));
                }
                x.kind = 2u;
#ifdef TRIM_DEBUG_BOUNDS
                if (x.e >= ix.list_offsets[ix.nlist] || li >= p.np) {
                    printf("DBG fetch q=%u w=%u lane=%u c=%u pp=%u bound=%u li=%u e=%u\n", q, w, lane, c, pp, bound, li, x.e);
                    __trap();
                }
#endif
                x.fc.load(ix.codes + static_cast<size_t>(x.e) * ix.code_stride, m, lane);
                x.lx = __ldg(ix.lx + x.e);
            } else { // dead lanes still step through the schedule: valid rows
                x.fc.zero(m);
            }
        }
    };
    build_lut_blocked<M>(ix, qv, lut, tid - kWarp, kThreads - kWarp);
    named_sync(kBarWorkers, kThreads - kWarp); // workers only
    LaneAdc la;
    la.init(lane, LutShape::of(m));
    TRIM_TL(if (wtl) {
        const unsigned long long t = clock64();
        wc[0] = t - wk;
        wk = t;
    })
    named_sync(kBarPlan, kThreads); // seeds done, compacted stream ready
    TRIM_TL(if (wtl) {
        const unsigned long long t = clock64();
        wc[1] = t - wk;
        wk = t;
    })
    bound = *reinterpret_cast<volatile uint32_t*>(s_total2);
    nchunks = (bound + kChunkW - 1) / kChunkW;
    fetch(0, sa);
    auto process = [&](uint32_t c, Slot& cur) {
        const uint32_t s = c % kRing;
        TRIM_TL(const unsigned long long k0 = wtl ? clock64() : 0;)
        if (c >= kRing)
            mbar_wait(empty + s, ((c / kRing) - 1) & 1u);
        if (!SEG && c == 1) // filter the rest against the threshold after chunk 0, not the seeds'
            named_sync(kBarChunk0, kThreads);
        const float T = ld_volatile(s_T);
        TRIM_TL(const unsigned long long k1 = wtl ? clock64() : 0;)
        const uint32_t g0 = s * kChunkW + w * kPerWorker;
        Cand& x = cur.c[0];
#if TRIM_STAGE_CUT
        float a; // warp-collective
        if constexpr (HARD || (SEG && TRIM_SEG_NOSTAGE)) { // every candidate is near the threshold: no early-exit stages
            a = x.fc.template sum_staged<true, StageNone>(m, la, StageNone{}, x.kind == 2u);
        } else {
            const StageCut ck = StageCut::make(x.lx, p.stage_c1, p.omg_hi, p.stage_ka, T);
            a = x.fc.template sum_staged<true, StageCut>(m, la, ck, x.kind == 2u);
        }
#else
        const StageCheck ck{x.lx, p.two_gamma, p.omg_hi, p.adc_eps, T};
        const float a = x.fc.sum_staged(m, la, ck, x.kind == 2u); // warp-collective
#endif
        // member = a candidate whose est interval [lo, hi] starts below T
        float lo = kNegInf, hi = kNegInf;
        bool keep = false;
        if (x.kind == 2u && a >= 0.0f) {
            lo = est_lower_bound(a, x.lx, p.two_gamma, p.adc_eps);
            keep = lo < ld_volatile(s_T); // the freshest published threshold
            if (keep)
                hi = est_upper_bound(a, x.lx, p.two_gamma, p.adc_eps);
        }
        TRIM_TL(const unsigned long long k2 = wtl ? clock64() : 0;)
        uint32_t id = 0;
        float d = 0.0f;
        bool exact = false;
        uint64_t rw = 0;
        if (keep) { // exact L2 (ivf.hpp:276) of every member the replay may evaluate
            id = __ldg(ix.list_ids + x.e);
            rw = id - ix.id_base;
#ifdef TRIM_DEBUG_BOUNDS
            if (rw >= ix.n) {
                printf("DBG keep q=%u w=%u lane=%u e=%u id=%u kind=%u\n", q, w, lane, x.e, id, x.kind);
                __trap();
            }
#endif
            exact = true;
            if (p.dap) { // d >= D~ - E > T_pub >= T_live: cannot replace the top (ivf.hpp:277)
                const float dl = __bfloat162float(p.dap[static_cast<size_t>(q) * p.dap_ld + rw]);
                if (dl > ld_volatile(s_T)) {
                    d = dl;
                    exact = false;
                }
            }
        }
        // the members' exact distances, 8 rows per warp pass: quad g = lane / 4
        // takes the g-th remaining member (euclid_sq_quad, the reference's
        // accumulator chains one per lane of the quad)
        if (!TRIM_QUAD_L2 && exact) // one lane walks the whole row (A/B: TRIM_QUAD_L2=0)
            d = euclid_sq_vec4(qv, ix.vectors + rw * ix.dim_stride, ix.dim, true);
        for (uint32_t em = TRIM_QUAD_L2 ? __ballot_sync(0xffffffffu, exact) : 0u; em;) {
            const uint32_t g = lane >> 2;
            uint32_t mm = em;
            for (uint32_t i = 0; i < g; ++i)
                mm &= mm - 1;
            const int src = mm ? __ffs(mm) - 1 : -1;
            const uint64_t rs = __shfl_sync(0xffffffffu, rw, src < 0 ? 0 : src);
#ifdef TRIM_DEBUG_BOUNDS
            if (src >= 0 && rs >= ix.n) {
                printf("DBG quad q=%u w=%u lane=%u src=%d rs=%llu em=%x\n", q, w, lane, src, (unsigned long long)rs, em);
                __trap();
            }
#endif
            const float dq = euclid_sq_quad(qv, src < 0 ? nullptr : ix.vectors + rs * ix.dim_stride, ix.dim,
                                            lane & 3u);
            const uint32_t rank = __popc(em & ((1u << lane) - 1u));
            const float mine = __shfl_sync(0xffffffffu, dq, (rank & 7u) * 4u);
            if (exact && rank < 8)
                d = mine;
            for (int i = 0; i < 8 && em; ++i) // drop this pass's members
                em &= em - 1;
            exact = exact && rank >= 8;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            const uint32_t r = __popc(bal & ((1u << lane) - 1u));
            s_e[g0 + r] = id;
            s_lo[g0 + r] = lo;
            s_hi[g0 + r] = hi;
            s_d[g0 + r] = d;
        }
        if (lane == 0) {
            bin_cnt[s * kWorkers + w] = __popc(bal);
            bin_mask[s * kWorkers + w] = bal;
        }
        mbar_arrive(full + s);
        TRIM_TL(if (wtl) {
            wc[2] += k1 - k0;
            wc[3] += k2 - k1;
            wc[4] += clock64() - k2;
        })
    };
    for (uint32_t c = 0; c < nchunks; c += 2) {
        fetch(c + 1, sb); // prefetch: loads in flight while chunk c is filtered
        process(c, sa);
        if (c + 1 >= nchunks)
            break;
        fetch(c + 2, sa);
        process(c + 1, sb);
    }
    TRIM_TL(if (wtl) {
        wc[5] = clock64() - wk;
        if (w == 0)
            for (int i = 0; i < 6; ++i)
                tl[10 + i] = wc[i];
        if (w < 7) {
            tl[16 + w] = wc[2];          // per worker: ring / chunk-0 waits
            tl[23 + w] = wc[3] + wc[4];  // per worker: ADC + exact L2
        }
    })
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
    float adc_eps;
    float omg_hi;            // 1 - gamma, rounded up
    uint32_t slice;          // stream positions per CTA
    uint32_t cap;            // pool entries per query
    unsigned long long* keys;  // nq*cap
    unsigned int* count;       // nq (members)
    unsigned long long* dc;    // nq (exact evaluations)
    unsigned long long* evaluated; // nq (stream length), written by slice 0
    // flat indexes with a block partition: per-query kept block count (probe
    // stride np), the stream split evenly over gridDim.x slices, and the
    // reference's stream length (every row) reported as evaluated
    const uint32_t* np_q;
    uint64_t eval_override;
};

__host__ __device__ inline size_t range_smem_bytes(int mt, uint32_t m, uint32_t dim_stride,
                                                   uint32_t np) {
    size_t b = lut_bytes(mt, m);
    b += sizeof(float) * dim_stride;
    b += sizeof(uint64_t) * np;
    b += sizeof(uint32_t) * (np + 1);
    b = (b + 15) & ~size_t(15);
    b += sizeof(uint32_t) * kRangeChunk; // superset entries
    b += sizeof(uint32_t) * 8;
    return b;
}

template <int M, int KS>
__global__ void __launch_bounds__(kThreads)
trim_range_kernel(DevIndex ix, RangeParams p) {
    unsigned char* smem = trim_dyn_smem;
    const uint32_t q = blockIdx.y;
    const uint32_t tid = threadIdx.x, lane = tid & 31u;
    const uint32_t m = M > 0 ? static_cast<uint32_t>(M) : ix.m;
    float* lut = reinterpret_cast<float*>(smem);
    float* qv = lut + lut_bytes(M, m) / sizeof(float);
    size_t off = lut_bytes(M, m) + sizeof(float) * ix.dim_stride;
    StreamSmem st;
    st.base = reinterpret_cast<uint64_t*>(smem + off);
    off += sizeof(uint64_t) * p.np;
    st.cum = reinterpret_cast<uint32_t*>(smem + off);
    off += sizeof(uint32_t) * (p.np + 1);
    off = (off + 15) & ~size_t(15);
    uint32_t* s_e = reinterpret_cast<uint32_t*>(smem + off);
    uint32_t* scal = s_e + kRangeChunk; // [0] superset count

    const float* qg = p.queries + static_cast<size_t>(q) * ix.dim_stride;
    for (uint32_t i = tid; i < ix.dim_stride; i += kThreads)
        qv[i] = qg[i];
    const uint32_t npq = p.np_q ? p.np_q[q] : p.np;
    const uint32_t total = load_stream(ix, p.probe ? p.probe + static_cast<size_t>(q) * p.np : nullptr,
                                       npq, st);
    uint32_t slice = p.slice;
    if (p.np_q) // the kept blocks' positions, split evenly over the CTAs of this query
        slice = max(static_cast<uint32_t>(kRangeChunk),
                    ((total + gridDim.x - 1) / gridDim.x + kRangeChunk - 1) / kRangeChunk * kRangeChunk);
    const uint32_t begin = blockIdx.x * slice;
    if (blockIdx.x == 0 && tid == 0)
        p.evaluated[q] = p.eval_override ? p.eval_override : total;
    if (begin >= total)
        return;
    const uint32_t end = min(total, begin + slice);
    build_lut_blocked<M>(ix, qv, lut);
    const float r2 = p.radius_sq[q];
    LaneAdc la;
    la.init(lane, LutShape::of(m));
    const float r2_excl = __int_as_float(__float_as_int(r2) + 1); // smallest float > r2 (r2 >= 0)

    // first list whose range contains `begin`
    uint32_t lo = 0, hi = npq;
    while (lo + 1 < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (st.cum[mid] <= begin)
            lo = mid;
        else
            hi = mid;
    }
    uint32_t li[kRangeU];
#pragma unroll
    for (int u = 0; u < kRangeU; ++u)
        li[u] = lo;
    uint32_t dc_local = 0;
    if (tid == 0)
        scal[0] = 0;
    __syncthreads();

    for (uint32_t pos = begin; pos < end; pos += kRangeChunk) {
        const uint32_t cn = min(static_cast<uint32_t>(kRangeChunk), end - pos);
#pragma unroll
        for (int u = 0; u < kRangeU; ++u) {
            const uint32_t r = static_cast<uint32_t>(u) * kThreads + tid;
            const bool valid = r < cn;
            uint32_t e = 0;
            float glx = 0.0f;
            FastCode<M> fc;
            fc.zero(m);
            if (valid) {
                const uint32_t pp = pos + r;
                while (st.cum[li[u] + 1] <= pp)
                    ++li[u];
                e = static_cast<uint32_t>(st.base[li[u]] + (pp - st.cum[li[u]]));
                fc.load(ix.codes + static_cast<size_t>(e) * ix.code_stride, m, lane);
                glx = __ldg(ix.lx + e);
            }
            const StageCheck ck{glx, p.two_gamma, p.omg_hi, p.adc_eps, r2_excl};
            const float a = fc.sum_staged(m, la, ck, valid); // warp-collective: every lane calls
            // evaluate iff est <= r^2 (ivf.hpp:331): decided by the rigorous interval
            // [lo, hi] around the reference's est, or, when it straddles r^2 (rare),
            // by the reference-order ADC itself
            if (valid && a >= 0.0f && est_lower_bound(a, glx, p.two_gamma, p.adc_eps) <= r2) {
                bool ev = est_upper_bound(a, glx, p.two_gamma, p.adc_eps) <= r2;
                if (!ev) {
                    const float ax = adc_serial<M>(ix.codes + static_cast<size_t>(e) * ix.code_stride, m);
                    ev = relaxed_lb(__fsqrt_rn(ax), glx, p.two_gamma) <= r2;
                }
                if (ev) {
                    const uint32_t slot = atomicAdd(&scal[0], 1u);
                    s_e[slot] = e;
                }
            }
        }
        __syncthreads();
        const uint32_t ns = scal[0];
        for (uint32_t i = tid; i < ns; i += kThreads) {
            const uint32_t e = s_e[i];
            {
                ++dc_local;
                const uint32_t id = __ldg(ix.list_ids + e);
                const float* row = ix.vectors + static_cast<size_t>(id - ix.id_base) * ix.dim_stride;
                const float d = euclid_sq_vec4(qv, row, ix.dim);
                if (d <= r2) { // ivf.hpp:334
                    const uint32_t slot = atomicAdd(p.count + q, 1u);
                    if (slot < p.cap)
                        p.keys[static_cast<size_t>(q) * p.cap + slot] = scored_key(d, id);
                }
            }
        }
        __syncthreads();
        if (tid == 0)
            scal[0] = 0;
        __syncthreads();
    }
    // block-wide sum of exact evaluations
    for (int o = 16; o > 0; o >>= 1)
        dc_local += __shfl_xor_sync(0xffffffffu, dc_local, o);
    if (lane == 0 && dc_local)
        atomicAdd(p.dc + q, static_cast<unsigned long long>(dc_local));
}

// --------------------------------------------------------------------------
// trim_range_flat_kernel — the flat scan (nlist = 1: every query's stream is
// the whole single list, ivf.hpp:318-320) with query tiling: a CTA holds the
// LUTs of up to kFlatMaxQ queries and evaluates each code it streams against
// all of them, so the codes are read from HBM once per query tile instead of
// once per query. Per (candidate, query) the decisions are trim_range_kernel's.
// grid (ceil(nq / qt), slices): consecutive CTAs are different query tiles
// over the same slice, so a slice's codes are read from HBM about once per
// wave of resident CTAs and served from L2 to the rest.
// --------------------------------------------------------------------------
constexpr uint32_t kFlatMaxQ = 8;
constexpr uint32_t kFlatThreads = 512; // 16 warps: one CTA per SM holds up to 6 LUTs of 32 KB

__host__ __device__ inline size_t range_flat_smem(int mt, uint32_t m, uint32_t dim_stride, uint32_t qt) {
    size_t b = lut_bytes(mt, m) * qt;            // LUTs (multiples of 128 B) at offset 0
    b += sizeof(float) * dim_stride * qt;        // query rows
    b += sizeof(uint32_t) * (2 * kFlatMaxQ);     // r^2, dc per query
    return b;
}

template <int M, int KS>
__global__ void __launch_bounds__(kFlatThreads)
trim_range_flat_kernel(DevIndex ix, RangeParams p, uint32_t qt) {
    unsigned char* smem = trim_dyn_smem;
    const uint32_t tid = threadIdx.x, lane = tid & 31u;
    const uint32_t m = M > 0 ? static_cast<uint32_t>(M) : ix.m;
    const uint64_t q0 = static_cast<uint64_t>(blockIdx.x) * qt;
    const uint32_t nqt = static_cast<uint32_t>(min(static_cast<uint64_t>(qt), p.nq - q0));
    const uint32_t lutb = static_cast<uint32_t>(lut_bytes(M, m));
    float* qvs = reinterpret_cast<float*>(smem + static_cast<size_t>(lutb) * qt);
    float* s_r2 = qvs + ix.dim_stride * qt;
    uint32_t* s_dc = reinterpret_cast<uint32_t*>(s_r2 + kFlatMaxQ);

    for (uint32_t i = tid; i < ix.dim_stride * qt; i += kFlatThreads) {
        const uint32_t t = i / ix.dim_stride;
        qvs[i] = t < nqt ? p.queries[(q0 + t) * ix.dim_stride + i % ix.dim_stride] : 0.0f;
    }
    if (tid < kFlatMaxQ) {
        s_r2[tid] = tid < nqt ? p.radius_sq[q0 + tid] : -1.0f;
        s_dc[tid] = 0;
    }
    const uint64_t lbeg = ix.list_offsets[0];
    const uint32_t total = static_cast<uint32_t>(ix.list_offsets[1] - lbeg);
    if (blockIdx.y == 0 && tid < nqt)
        p.evaluated[q0 + tid] = total;
    const uint32_t begin = blockIdx.y * p.slice;
    if (begin >= total)
        return;
    const uint32_t end = min(total, begin + p.slice);
    __syncthreads();
    for (uint32_t t = 0; t < nqt; ++t)
        build_lut_blocked<M>(ix, qvs + t * ix.dim_stride, reinterpret_cast<float*>(smem + static_cast<size_t>(t) * lutb));
    __syncthreads();
    LaneAdc la;
    la.init(lane, LutShape::of(m));

    FastCode<M> fa, fb;
    float xa = 0.0f, xb = 0.0f;
    auto fetch = [&](uint32_t pos, FastCode<M>& fc, float& glx) {
        const uint32_t pp = pos + tid;
        if (pp < end) {
            const uint64_t e = lbeg + pp;
            fc.load(ix.codes + e * ix.code_stride, m, lane);
            glx = __ldg(ix.lx + e);
        } else {
            fc.zero(m);
            glx = 0.0f;
        }
    };
    // No block barriers in the scan: a member (rare) is evaluated by its own lane
    // at once — exact L2 (ivf.hpp:332), then kept iff d <= r^2 (ivf.hpp:334).
    auto step = [&](uint32_t pos, FastCode<M>& fc, float glx) {
        const bool valid = pos + tid < end;
        const uint64_t e = lbeg + pos + tid;
        fc.permute_all(m, la);
#pragma unroll 1
        for (uint32_t t = 0; t < nqt; ++t) {
            const float r2 = s_r2[t];
            const float r2x = __int_as_float(__float_as_int(r2) + 1); // smallest float > r^2
            const StageCheck ck{glx, p.two_gamma, p.omg_hi, p.adc_eps, r2x};
            const float a = fc.template sum_staged<false>(m, la, ck, valid, t * lutb); // warp-collective
            // evaluate iff est <= r^2 (ivf.hpp:331): the interval decides, or the
            // reference-order ADC when it straddles r^2
            if (valid && a >= 0.0f && est_lower_bound(a, glx, p.two_gamma, p.adc_eps) <= r2) {
                bool ev = est_upper_bound(a, glx, p.two_gamma, p.adc_eps) <= r2;
                if (!ev) {
                    const float ax = adc_serial<M>(ix.codes + e * ix.code_stride, m, t * lutb);
                    ev = relaxed_lb(__fsqrt_rn(ax), glx, p.two_gamma) <= r2;
                }
                if (ev) {
                    atomicAdd(s_dc + t, 1u);
                    const uint32_t id = __ldg(ix.list_ids + e);
                    const float* row = ix.vectors + static_cast<size_t>(id - ix.id_base) * ix.dim_stride;
                    const float d = euclid_sq_vec4(qvs + t * ix.dim_stride, row, ix.dim, true);
                    if (d <= r2) {
                        const uint64_t q = q0 + t;
                        const uint32_t slot = atomicAdd(p.count + q, 1u);
                        if (slot < p.cap)
                            p.keys[q * p.cap + slot] = scored_key(d, id);
                    }
                }
            }
        }
    };
    fetch(begin, fa, xa);
    for (uint32_t pos = begin; pos < end; pos += 2 * kFlatThreads) {
        fetch(pos + kFlatThreads, fb, xb); // next step's codes in flight
        step(pos, fa, xa);
        if (pos + kFlatThreads >= end)
            break;
        fetch(pos + 2 * kFlatThreads, fa, xa);
        step(pos + kFlatThreads, fb, xb);
    }
    __syncthreads();
    if (tid < nqt && s_dc[tid])
        atomicAdd(p.dc + q0 + tid, static_cast<unsigned long long>(s_dc[tid]));
}

#ifndef TRIM_M // non-template kernels: compiled once, in trim_capi.cu
} // namespace trimgpu
#include "trim_probe_mma.cuh"
#include "trim_flat_mma.cuh"
namespace trimgpu {
// --------------------------------------------------------------------------
// trim_knn_setup_kernel — what trim_knn_kernel's replay warp does before its
// workers may start (ivf.hpp:256-271 and the list-level plan), for a batch,
// one warp per query: the stream of the probed lists, the k seeds' exact
// distances in stream order (evaluated unconditionally, ivf.hpp:264-271), the
// seeded threshold T0 = max_dis, and the plan — every probed list after the
// seeds whose list_lower_bound is >= T0 is dropped (the reference prunes each
// of its entries, ivf.hpp:275), the rest compacted. Moving it out of the
// filter kernel frees that kernel's shared-memory slot ~25 us sooner per query.
// Dynamic shared memory: (np + 1) u32 + np u64.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(kWarp) trim_knn_setup_kernel(DevIndex ix, KnnParams p, uint32_t* recs) {
    const uint32_t q = blockIdx.x;
    if (q >= p.nq)
        return;
    const uint32_t lane = threadIdx.x;
    StreamSmem st;
    st.base = reinterpret_cast<uint64_t*>(trim_dyn_smem);
    st.cum = reinterpret_cast<uint32_t*>(st.base + p.np);
    const uint32_t* pl = p.probe + static_cast<size_t>(q) * p.np;
    const float* qv = p.queries + static_cast<size_t>(q) * ix.dim_stride;
    uint32_t carry = 0;
    for (uint32_t b0 = 0; b0 < p.np; b0 += kWarp) { // load_stream, one warp
        const uint32_t li = b0 + lane;
        uint32_t v = 0;
        if (li < p.np) {
            const uint32_t l = __ldg(pl + li);
            st.base[li] = __ldg(ix.list_offsets + l);
            v = static_cast<uint32_t>(__ldg(ix.list_offsets + l + 1) - st.base[li]);
        }
#pragma unroll
        for (int o = 1; o < kWarp; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= static_cast<uint32_t>(o))
                v += t;
        }
        if (li < p.np)
            st.cum[li + 1] = carry + v;
        carry += __shfl_sync(0xffffffffu, v, kWarp - 1);
    }
    if (lane == 0)
        st.cum[0] = 0;
    __syncwarp();
    const uint32_t total = carry;
    const uint32_t nseed = min(p.k, total);
    const KnnPlanLayout lo = KnnPlanLayout::of(p.np, p.k);
    uint32_t* rec = recs + static_cast<size_t>(q) * lo.words;
    // seeds (ivf.hpp:264-271): exact distances in stream order; T0 = max_dis
    // after them (the largest (d, id), or +inf when fewer than k)
    float T0 = nseed < p.k ? __int_as_float(0x7f800000) : 0.0f;
    for (uint32_t b0 = 0; b0 < nseed; b0 += kWarp) {
        const uint32_t i = b0 + lane;
        if (i < nseed) {
            uint32_t li = 0;
            while (st.cum[li + 1] <= i)
                ++li;
            const uint64_t e = st.base[li] + (i - st.cum[li]);
            const uint32_t id = __ldg(ix.list_ids + e);
            const float d = euclid_sq_vec4(qv, ix.vectors + static_cast<size_t>(id - ix.id_base) * ix.dim_stride,
                                           ix.dim, true);
            rec[lo.sd + i] = __float_as_uint(d);
            rec[lo.sid + i] = id;
            if (nseed == p.k)
                T0 = fmaxf(T0, d);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        T0 = fmaxf(T0, __shfl_xor_sync(0xffffffffu, T0, o));
    // plan (as trim_knn_kernel's replay warp)
    const bool skip = p.skip_lists && total > nseed;
    uint32_t kept = 0, nk = 0;
    for (uint32_t b0 = 0; b0 < p.np; b0 += kWarp) {
        const uint32_t i = b0 + lane;
        uint32_t len = 0;
        uint64_t bs = 0;
        if (i < p.np) {
            const uint32_t c0 = st.cum[i], c1 = st.cum[i + 1];
            bool drop = c1 <= nseed;
            if (!drop && skip && c0 >= nseed) {
                const uint32_t l = __ldg(pl + i);
                const float dq = euclid_sq_vec4(qv, ix.coarse + static_cast<size_t>(l) * ix.dim_stride, ix.dim);
                drop = list_lower_bound(dq, __ldg(ix.list_R + l), __ldg(ix.list_xmin + l), __ldg(ix.list_xmax + l),
                                        p) >= T0;
            }
            if (!drop) {
                const uint32_t s0 = max(c0, nseed);
                len = c1 - s0;
                bs = st.base[i] + (s0 - c0);
            }
        }
        const uint32_t keep = __ballot_sync(0xffffffffu, len != 0);
        uint32_t v = len;
#pragma unroll
        for (int o = 1; o < kWarp; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= static_cast<uint32_t>(o))
                v += t;
        }
        if (len != 0) {
            const uint32_t j = nk + __popc(keep & ((1u << lane) - 1u));
            reinterpret_cast<uint64_t*>(rec + lo.base)[j] = bs;
            rec[lo.cum + j] = kept + v - len;
        }
        kept += __shfl_sync(0xffffffffu, v, kWarp - 1);
        nk += __popc(keep);
    }
    if (lane == 0) {
        rec[lo.cum + nk] = kept;
        rec[0] = total;
        rec[1] = nseed;
        rec[2] = nk;
        rec[3] = kept;
        rec[4] = __float_as_uint(T0);
        rec[5] = nseed; // dc so far
        rec[6] = nseed; // evaluated unconditionally
        const uint32_t rest = total - nseed;
        // stream in order; bit 8: the list-level bound dropped at least 3/4 of it, so what is
        // left are the lists around the query — no early-exit stages (StageNone)
        rec[7] = kept && static_cast<uint64_t>(kept) * 4 <= rest ? 0x100u : 0u;
        if (p.skipped && rest != kept)
            atomicAdd(p.skipped, static_cast<unsigned long long>(rest - kept));
    }
}

// --------------------------------------------------------------------------
// trim_knn_seg_plan_kernel — the plan of a segmented flat kNN scan
// (ivf.hpp:243-304 with nlist = 1), one CTA per query.
//
// The flat stream is the rows in id order and the running threshold only
// falls, so once the first n0 rows are scanned (an ordinary launch over
// [0, n0): top-k `ids_a`/`dist_a`, counters `ct_a`) every later row x has
// est(x) >= T_live(x) whenever the list-level bound L_b of its block
// (list_lower_bound over the partition's block b, D~ - E from
// trim_probe_mma_kernel as the coarse distance) is >= T_A = max_dis after n0
// rows: the reference prunes it (ivf.hpp:275). Rows n0.. are stored regrouped
// by (segment of `seg_len` consecutive ids, block), ascending ids inside
// (seg_off: S * nb + 1 offsets). For each segment the kept blocks' runs (each
// ascending in id) are merged by id in shared memory (rank = own offset + the
// counts of smaller ids in the other runs) and the entries appended to the query's table: the
// reference's stream with the pruned blocks' rows removed, in order. The record
// resumes the top-k and the counters; trim_knn_kernel<SEG> walks the table. A
// query whose plan does not fit (more than kSegMaxKept blocks, kSegSortCap rows
// of one segment, `tab_cap` rows in all) is planned as one in-order run over
// rows [n0, n) of the original arrays (mode 0, the PRE kernel without SEG).
// --------------------------------------------------------------------------
// list_lower_bound for a block of a flat partition
__device__ __forceinline__ float block_lower_bound(float dq, float R, float xmin, float xmax, float omg_lo, float omg_hi,
                                                   float kq1, float kq2, float kest) {
    KnnParams p{};
    p.omg_lo = omg_lo;
    p.omg_hi = omg_hi;
    p.kq1 = kq1;
    p.kq2 = kq2;
    p.kest = kest;
    return list_lower_bound(dq, R, xmin, xmax, p);
}

struct SegPlanParams {
    const float* queries;
    uint64_t nq;
    uint32_t k, np;          // np: the record layout's run capacity (1)
    uint32_t tab_cap;        // table words per query
    uint64_t n, n0;      // n0: rows scanned in order so far (= the start of segment seg0)
    uint64_t n_next;     // a plan that does not fit continues in order up to here and is planned again (0: last round)
    uint32_t nseg, seg0; // segments [seg0, nseg) remain
    uint32_t round;      // > 0: queries already planned (mode 1) are left alone
    const uint64_t* seg_off;
    const uint32_t* ids;  // ids of the regrouped entries
    const float* approx;  // nq x mma_ld(nb): tf32 |q - c_b|^2
    const float* cn2;     // |c_b|^2
    const float* cn;      // |c_b|
    const uint32_t* ids_a;
    const float* dist_a;
    const unsigned long long* ct_a;
    float omg_lo, omg_hi, kq1, kq2, kest;
    uint32_t* recs;
    uint32_t* tab;
    unsigned long long* skipped;
    uint32_t force_plain;
    uint32_t* dbg; // TRIM_SEG_DEBUG: per query {kept blocks, plain, table rows, segments sorted}, or null
};
constexpr uint32_t kSegMaxKept = 64;   // kept blocks per query in block mode
constexpr uint32_t kSegSortCap = 8192; // rows of one segment's kept blocks (their ids in shared memory)

__global__ void __launch_bounds__(kThreads) trim_knn_seg_plan_kernel(DevIndex aux, SegPlanParams p) {
    __shared__ uint32_t s_id[kSegSortCap];
    __shared__ uint32_t ws[16];
    __shared__ uint32_t s_kept[kSegMaxKept];
    __shared__ uint32_t s_roff[kSegMaxKept + 1];
    __shared__ unsigned long long s_rbase[kSegMaxKept];
    __shared__ uint32_t s_nkept, s_bad;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint64_t q = blockIdx.x;
    if (q >= p.nq)
        return;
    const uint32_t nb = aux.nlist;
    const KnnPlanLayout lo = KnnPlanLayout::of(p.np, p.k);
    uint32_t* rec = p.recs + q * lo.words;
    if (p.round && (rec[7] & 0xffu) == 1u)
        return;
    uint32_t* tab = p.tab + q * p.tab_cap;
    const float* qrow = p.queries + q * aux.dim_stride;
    float qp = 0.0f;
    for (uint32_t i = tid; i < aux.dim; i += kThreads)
        qp = __fadd_ru(qp, __fmul_ru(qrow[i], qrow[i]));
    for (int o = 16; o > 0; o >>= 1)
        qp = __fadd_ru(qp, __shfl_xor_sync(0xffffffffu, qp, o));
    if (lane == 0)
        ws[warp] = __float_as_uint(qp);
    if (tid == 0) {
        s_nkept = 0;
        s_bad = p.force_plain;
    }
    __syncthreads();
    float qn2 = 0.0f;
    for (uint32_t w = 0; w < kWarps; ++w)
        qn2 = __fadd_ru(qn2, __uint_as_float(ws[w]));
    qn2 = __fmul_ru(qn2, 1.0f + 1.0f / 65536.0f);
    const float qn = __fsqrt_ru(qn2);
    const float T = p.dist_a[q * p.k + (p.k - 1)]; // max_dis after the first n0 rows
    const float* arow = p.approx + q * mma_ld(nb);
    // the blocks the bound cannot prune, ascending
    for (uint32_t b0 = 0; b0 < nb; b0 += kThreads) {
        const uint32_t b = b0 + tid;
        bool keep = false;
        if (b < nb) {
            const float e = __fadd_ru(__fmul_ru(__fmul_ru(qn, __ldg(p.cn + b)), 1.0f / 64.0f),
                                      __fmul_ru(__fadd_ru(qn2, __ldg(p.cn2 + b)), 1.0f / 16384.0f));
            const float dq = fmaxf(__fsub_rd(arow[b], e), 0.0f); // <= |q - c_b|^2
            keep = !(block_lower_bound(dq, __ldg(aux.list_R + b), __ldg(aux.list_xmin + b), __ldg(aux.list_xmax + b),
                                       p.omg_lo, p.omg_hi, p.kq1, p.kq2, p.kest) >= T);
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0)
            ws[warp] = __popc(bal);
        __syncthreads();
        uint32_t before = s_nkept, tot = 0;
        for (uint32_t w = 0; w < kWarps; ++w) {
            before += w < warp ? ws[w] : 0u;
            tot += ws[w];
        }
        if (keep) {
            const uint32_t j = before + __popc(bal & ((1u << lane) - 1u));
            if (j < kSegMaxKept)
                s_kept[j] = b;
        }
        __syncthreads();
        if (tid == 0) {
            s_nkept += tot;
            if (s_nkept > kSegMaxKept)
                s_bad = 1;
        }
        __syncthreads();
    }
    const uint32_t nkept = min(s_nkept, kSegMaxKept);
    // segment by segment: the kept blocks' runs merged by id into the table
    uint32_t total = 0, sorted = 0;
    for (uint32_t g = p.seg0; g < p.nseg; ++g) {
        if (s_bad)
            break;
        const uint64_t* so = p.seg_off + static_cast<size_t>(g) * nb;
        if (tid < kWarp) { // run starts and the prefix of their lengths (nkept <= 64: two per lane)
            uint32_t carry = 0;
            for (uint32_t j0 = 0; j0 < nkept; j0 += kWarp) {
                const uint32_t j = j0 + lane;
                uint32_t len = 0;
                if (j < nkept) {
                    const uint64_t b0 = __ldg(so + s_kept[j]);
                    len = static_cast<uint32_t>(__ldg(so + s_kept[j] + 1) - b0);
                    s_rbase[j] = b0;
                }
                uint32_t v = len;
#pragma unroll
                for (int o = 1; o < kWarp; o <<= 1) {
                    const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
                    if (lane >= static_cast<uint32_t>(o))
                        v += t;
                }
                if (j < nkept)
                    s_roff[j] = carry + v - len;
                carry += __shfl_sync(0xffffffffu, v, kWarp - 1);
            }
            if (lane == 0)
                s_roff[nkept] = carry;
        }
        __syncthreads();
        const uint32_t rows = s_roff[nkept];
        if (rows == 0) {
            __syncthreads();
            continue;
        }
        if (rows > kSegSortCap || total + rows > p.tab_cap) {
            __syncthreads();
            if (tid == 0)
                s_bad = 1;
            __syncthreads();
            break;
        }
        uint32_t nonempty = 0;
        for (uint32_t j = 0; j < nkept; ++j)
            nonempty += s_roff[j + 1] != s_roff[j];
        if (nonempty == 1) { // one run: already in id order
            uint32_t j = 0;
            while (s_roff[j + 1] == s_roff[j])
                ++j;
            const uint32_t b0 = static_cast<uint32_t>(s_rbase[j]);
            for (uint32_t i = tid; i < rows; i += kThreads)
                tab[total + i] = b0 + i;
        } else {
            // merge the runs by id: every run is ascending and ids are unique, so a row's
            // place is its offset in its own run plus, for every other run, the number of
            // that run's ids below it (a binary search in shared memory)
            for (uint32_t i = tid; i < rows; i += kThreads) {
                uint32_t a = 0, b = nkept; // the run holding merge-input index i
                while (b - a > 1) {
                    const uint32_t mid = (a + b) >> 1;
                    if (s_roff[mid] <= i)
                        a = mid;
                    else
                        b = mid;
                }
                s_id[i] = __ldg(p.ids + static_cast<uint32_t>(s_rbase[a]) + (i - s_roff[a]));
            }
            __syncthreads();
            for (uint32_t i = tid; i < rows; i += kThreads) {
                uint32_t a = 0, b = nkept;
                while (b - a > 1) {
                    const uint32_t mid = (a + b) >> 1;
                    if (s_roff[mid] <= i)
                        a = mid;
                    else
                        b = mid;
                }
                const uint32_t id = s_id[i];
                uint32_t rank = i - s_roff[a];
                for (uint32_t j = 0; j < nkept; ++j) {
                    if (j == a)
                        continue;
                    uint32_t l0 = s_roff[j], h0 = s_roff[j + 1]; // first index in run j with id above `id`
                    while (l0 < h0) {
                        const uint32_t mid = (l0 + h0) >> 1;
                        if (s_id[mid] < id)
                            l0 = mid + 1;
                        else
                            h0 = mid;
                    }
                    rank += l0 - s_roff[j];
                }
                tab[total + rank] = static_cast<uint32_t>(s_rbase[a]) + (i - s_roff[a]);
            }
            ++sorted;
        }
        total += rows;
        __syncthreads();
    }
    // resume state: the top-k after n0 rows as the seeds, its counters
    for (uint32_t i = tid; i < p.k; i += kThreads) {
        rec[lo.sd + i] = __float_as_uint(p.dist_a[q * p.k + i]);
        rec[lo.sid + i] = p.ids_a[q * p.k + i];
    }
    if (tid == 0) {
        const bool plain = s_bad != 0;
        if (p.dbg) {
            p.dbg[q * 4 + 0] = s_nkept;
            p.dbg[q * 4 + 1] = plain;
            p.dbg[q * 4 + 2] = total;
            p.dbg[q * 4 + 3] = sorted;
        }
        rec[0] = static_cast<uint32_t>(p.n);                // evaluated
        rec[1] = p.k;                                       // entries offered to the top-k
        rec[4] = __float_as_uint(T);
        rec[5] = static_cast<uint32_t>(p.ct_a[q * 6 + 0]);  // dc over [0, n0)
        rec[6] = static_cast<uint32_t>(min(static_cast<uint64_t>(p.k), p.n)); // the seeds
        rec[lo.cum] = 0;
        if (plain) { // in order: up to n_next and planned again, or (last round) the rest
            const uint64_t end = p.n_next ? p.n_next : p.n;
            rec[2] = 1;
            rec[3] = static_cast<uint32_t>(end - p.n0);
            rec[7] = p.n_next ? 2 : 0;
            rec[lo.cum + 1] = static_cast<uint32_t>(end - p.n0);
            reinterpret_cast<uint64_t*>(rec + lo.base)[0] = p.n0;
        } else {
            rec[2] = 0; // no runs: the stream is the table
            rec[3] = total;
            rec[7] = 1;
            if (p.skipped)
                atomicAdd(p.skipped, static_cast<unsigned long long>(p.n - p.n0) - total);
        }
    }
}

// --------------------------------------------------------------------------
// trim_probe_kernel — probe_order (ivf.hpp:173-187): coarse distances in the
// reference's arithmetic, sorted by (dist, list id) in shared memory, first
// np ids out. One CTA per query.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
trim_probe_kernel(DevIndex ix, const float* queries, uint64_t nq, uint32_t np, uint32_t nl_pow2,
                  uint32_t* probe_out) {
    unsigned char* smem = trim_dyn_smem;
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

// --------------------------------------------------------------------------
// trim_probe_tiled_kernel — probe_order (ivf.hpp:173-187) for kProbeQ queries
// per CTA: centroid tiles are staged transposed in shared memory
// ([dim/4][tile][float4], conflict-free float4 reads), every (query,
// centroid) distance uses the reference's 4-accumulator order, and warp w
// then selects query w's np smallest (dist, list id) by an 8-bit radix
// select over the distance bits (ties resolved by ascending list id, as
// std::sort on ScoredId does) and sorts them with a warp bitonic sort.
// Requires np <= kProbeMaxNp.
// --------------------------------------------------------------------------
constexpr uint32_t kProbeQ = 8;        // queries per CTA (one selecting warp each)
constexpr uint32_t kProbeMaxNp = 256;

__host__ __device__ inline size_t probe_tiled_smem(uint32_t nlist, uint32_t dim_stride, uint32_t tile) {
    return sizeof(float) * kProbeQ * dim_stride          // queries
         + sizeof(float) * dim_stride * tile              // centroid tile (transposed)
         + sizeof(uint32_t) * kProbeQ * nlist             // distance bits
         + kProbeQ * (sizeof(uint32_t) * 256 + sizeof(uint64_t) * kProbeMaxNp); // hist + sort
}

__global__ void __launch_bounds__(kThreads)
trim_probe_tiled_kernel(DevIndex ix, const float* queries, uint64_t nq, uint32_t np, uint32_t tile,
                        uint32_t* probe_out) {
    unsigned char* smem = trim_dyn_smem;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint64_t q0 = static_cast<uint64_t>(blockIdx.x) * kProbeQ;
    const uint32_t ds = ix.dim_stride, nv = ds >> 2, nlist = ix.nlist;
    const uint32_t full4 = ix.dim >> 2, tail = ix.dim & 3u;
    float* qs = reinterpret_cast<float*>(smem);
    float4* ct = reinterpret_cast<float4*>(qs + kProbeQ * ds); // [nv][tile]
    uint32_t* keys = reinterpret_cast<uint32_t*>(ct + static_cast<size_t>(nv) * tile); // [kProbeQ][nlist]
    uint32_t* hist = keys + static_cast<size_t>(kProbeQ) * nlist;                        // [kProbeQ][256]
    uint64_t* sel = reinterpret_cast<uint64_t*>(hist + kProbeQ * 256);                   // [kProbeQ][kProbeMaxNp]

    for (uint32_t i = tid; i < kProbeQ * ds; i += kThreads) {
        const uint64_t qq = q0 + i / ds;
        qs[i] = qq < nq ? queries[qq * ds + i % ds] : 0.0f;
    }
    // ---- distances: warp w -> query w, lane -> centroids lane + 32j of the tile
    const float4* qv4 = reinterpret_cast<const float4*>(qs + warp * ds);
    const uint32_t per = tile / 32;
    for (uint32_t c0 = 0; c0 < nlist; c0 += tile) {
        __syncthreads();
        for (uint32_t i = tid; i < nv * tile; i += kThreads) {
            const uint32_t c = i % tile, v = i / tile;
            ct[v * tile + c] = (c0 + c < nlist)
                ? *reinterpret_cast<const float4*>(ix.coarse + static_cast<size_t>(c0 + c) * ds + 4 * v)
                : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncthreads();
        for (uint32_t j = 0; j < per; ++j) {
            const uint32_t c = lane + 32 * j;
            float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
            for (uint32_t v = 0; v < full4; ++v) {
                const float4 a = qv4[v];
                const float4 b = ct[v * tile + c];
                const float d0 = __fsub_rn(a.x, b.x), d1 = __fsub_rn(a.y, b.y);
                const float d2 = __fsub_rn(a.z, b.z), d3 = __fsub_rn(a.w, b.w);
                a0 = __fadd_rn(a0, __fmul_rn(d0, d0));
                a1 = __fadd_rn(a1, __fmul_rn(d1, d1));
                a2 = __fadd_rn(a2, __fmul_rn(d2, d2));
                a3 = __fadd_rn(a3, __fmul_rn(d3, d3));
            }
            if (tail) { // distance.hpp:23-26: the remainder goes into acc0, in order
                const float4 a = qv4[full4];
                const float4 b = ct[full4 * tile + c];
                const float d0 = __fsub_rn(a.x, b.x);
                a0 = __fadd_rn(a0, __fmul_rn(d0, d0));
                if (tail > 1) {
                    const float d1 = __fsub_rn(a.y, b.y);
                    a0 = __fadd_rn(a0, __fmul_rn(d1, d1));
                }
                if (tail > 2) {
                    const float d2 = __fsub_rn(a.z, b.z);
                    a0 = __fadd_rn(a0, __fmul_rn(d2, d2));
                }
            }
            if (c0 + c < nlist)
                keys[warp * nlist + c0 + c] = __float_as_uint(__fadd_rn(__fadd_rn(a0, a1), __fadd_rn(a2, a3)));
        }
    }
    __syncthreads();
    const uint64_t q = q0 + warp;
    if (q >= nq)
        return;
    // ---- radix select of the np-th smallest distance bits (non-negative floats
    // order like their bit patterns)
    const uint32_t* kq = keys + warp * nlist;
    uint32_t* h = hist + warp * 256;
    uint32_t prefix = 0, pmask = 0, rank = np; // rank: 1-based among keys matching prefix
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (uint32_t i = lane; i < 256; i += 32)
            h[i] = 0;
        __syncwarp();
        for (uint32_t c = lane; c < nlist; c += 32) {
            const uint32_t kk = kq[c];
            if ((kk & pmask) == prefix)
                atomicAdd(&h[(kk >> shift) & 0xFFu], 1u);
        }
        __syncwarp();
        // bucket b with cum(b) < rank <= cum(b) + h[b]: lane owns bins 8*lane..8*lane+7
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
    // prefix = the np-th smallest distance bits; take every key below it and
    // the first `rank` keys equal to it in ascending list-id order
    uint64_t* sq = sel + warp * kProbeMaxNp;
    uint32_t n_lt = 0, n_eq = 0;
    for (uint32_t c0 = 0; c0 < nlist; c0 += 32) {
        const uint32_t c = c0 + lane;
        const uint32_t kk = c < nlist ? kq[c] : 0xFFFFFFFFu;
        const bool lt = c < nlist && kk < prefix;
        const bool eq = c < nlist && kk == prefix;
        const uint32_t blt = __ballot_sync(0xffffffffu, lt);
        const uint32_t beq = __ballot_sync(0xffffffffu, eq);
        const uint32_t below = (1u << lane) - 1u;
        if (lt)
            sq[n_lt + __popc(blt & below)] = (static_cast<uint64_t>(kk) << 32) | c;
        if (eq) {
            const uint32_t r = n_eq + __popc(beq & below);
            if (r < rank)
                sq[np - rank + r] = (static_cast<uint64_t>(kk) << 32) | c;
        }
        n_lt += __popc(blt);
        n_eq += __popc(beq);
    }
    // pad to a power of two and bitonic-sort (warp, shared memory)
    uint32_t n2 = 1;
    while (n2 < np)
        n2 <<= 1;
    for (uint32_t i = np + lane; i < n2; i += 32)
        sq[i] = ~0ull;
    __syncwarp();
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
    for (uint32_t i = lane; i < np; i += 32)
        probe_out[q * np + i] = static_cast<uint32_t>(sq[i] & 0xffffffffu);
}

// pq::build_distance_table to global memory (one CTA per query).
__global__ void __launch_bounds__(kThreads)
trim_lut_kernel(DevIndex ix, const float* queries, float* lut_out) {
    unsigned char* smem = trim_dyn_smem;
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

// trim_search_range_device helpers. r^2 = r*r in fp32 (ivf.hpp:315).
__global__ void trim_range_r2_kernel(const float* radius, uint64_t nq, float* r2, uint32_t* status) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nq)
        return;
    const float r = radius[i];
    if (r < 0.0f) { // ivf.hpp:311-312 throws; here: empty result + status bit 1
        r2[i] = -1.0f;
        if (status)
            atomicOr(status, 2u);
    } else {
        r2[i] = __fmul_rn(r, r);
    }
}

// Segment bounds of the per-query pools for the segmented sort.
__global__ void trim_range_seg_kernel(const unsigned int* cnt, uint64_t nq, uint32_t cap, uint64_t* beg,
                                      uint64_t* end, uint32_t* status) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nq)
        return;
    const unsigned int c = cnt[i];
    beg[i] = i * cap;
    end[i] = i * cap + min(c, cap);
    if (c > cap && status)
        atomicOr(status, 1u);
}

// Sorted (d, id) keys -> per-query slots; counts and counters
// (ivf.hpp:327-338: evaluated = stream length, edc = evaluated, dc exact).
__global__ void trim_range_finish_kernel(const unsigned long long* sorted, const unsigned int* cnt,
                                         const unsigned long long* dc, const unsigned long long* ev,
                                         uint64_t nq, uint32_t cap, uint32_t nlist, uint32_t* counts,
                                         uint32_t* ids, float* dist, unsigned long long* counters) {
    const uint64_t q = blockIdx.x;
    const uint32_t n = min(cnt[q], cap);
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const unsigned long long key = sorted[q * cap + i];
        ids[q * cap + i] = static_cast<uint32_t>(key & 0xffffffffu);
        dist[q * cap + i] = __uint_as_float(static_cast<uint32_t>(key >> 32));
    }
    if (threadIdx.x == 0) {
        counts[q] = cnt[q];
        if (counters) {
            unsigned long long* c = counters + q * 6;
            c[0] = dc[q];
            c[1] = ev[q];
            c[2] = ev[q] - dc[q];
            c[3] = ev[q];
            c[4] = 0;
            c[5] = nlist;
        }
    }
}

// Multi-GPU merge: k smallest (dist, id) of nshards*k candidates per query.
__global__ void __launch_bounds__(kThreads)
trim_merge_kernel(const float* dist, const uint32_t* ids, uint32_t nshards, uint64_t nq,
                  uint32_t k, uint32_t n_pow2, float* dist_out, uint32_t* ids_out) {
    unsigned char* smem = trim_dyn_smem;
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

// Per inverted list (one CTA each): R_l >= max_x |c_l - landmark(x)|, where
// landmark(x) is the PQ reconstruction of x's code (the point lx measures to,
// ivf.hpp:137-145), computed in fp64 and rounded up; and [xmin, xmax] of the
// stored lx. Feeds list_lower_bound. Empty lists get R = 0, xmin = +inf,
// xmax = -inf (they contribute no positions).
__global__ void __launch_bounds__(kThreads)
trim_list_meta_kernel(DevIndex ix, float* list_R, float* list_xmin, float* list_xmax) {
    __shared__ double s_r[kWarps];
    __shared__ float s_lo[kWarps], s_hi[kWarps];
    const uint32_t l = blockIdx.x;
    const uint64_t b = ix.list_offsets[l], e = ix.list_offsets[l + 1];
    const float* c = ix.coarse + static_cast<size_t>(l) * ix.dim_stride;
    double r2 = 0.0;
    float lo = __int_as_float(0x7f800000), hi = __int_as_float(0xff800000);
    for (uint64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
        const uint8_t* code = ix.codes + i * ix.code_stride;
        double acc = 0.0;
        for (uint32_t j = 0; j < ix.m; ++j) {
            const uint32_t sd = ix.sub_dims[j], so = ix.sub_offsets[j];
            const float* cen = ix.centroids + static_cast<size_t>(ix.ksub) * so + static_cast<size_t>(code[j]) * sd;
            for (uint32_t t = 0; t < sd; ++t) {
                const double d = static_cast<double>(cen[t]) - static_cast<double>(c[so + t]);
                acc += d * d;
            }
        }
        r2 = fmax(r2, acc);
        const float x = ix.lx[i];
        lo = fminf(lo, x);
        hi = fmaxf(hi, x);
    }
    for (int o = 16; o > 0; o >>= 1) {
        r2 = fmax(r2, __shfl_xor_sync(0xffffffffu, r2, o));
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    if (lane == 0) {
        s_r[warp] = r2;
        s_lo[warp] = lo;
        s_hi[warp] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kWarps; ++w) {
            r2 = fmax(r2, s_r[w]);
            lo = fminf(lo, s_lo[w]);
            hi = fmaxf(hi, s_hi[w]);
        }
        // fp64 sum of <= 2^12 squares: relative error < 2^-40; the margin covers it
        list_R[l] = __double2float_ru(sqrt(r2) * (1.0 + 1e-9));
        list_xmin[l] = lo;
        list_xmax[l] = hi;
    }
}

// --------------------------------------------------------------------------
// Flat range search over a block partition of the rows (trim_capi.cu
// build_flat_partition): the range filter is order-free (ivf.hpp:323-340), so
// scanning the blocks instead of the rows in id order gives the reference's
// members and counters exactly, and a block whose list-level bound proves
// est > r^2 for all its rows is pruned whole. One CTA per query; D~ to the
// block centroids comes from trim_probe_mma_kernel. Output: the kept blocks in
// ascending order (probe stride nb) and their count.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
trim_block_select_kernel(DevIndex aux, const float* __restrict__ queries, uint64_t nq, const float* __restrict__ r2,
                         const float* __restrict__ approx, const float* __restrict__ cn2, const float* __restrict__ cn,
                         float omg_lo, float omg_hi, float kq1, float kq2, float kest, uint32_t* __restrict__ kept,
                         uint32_t* __restrict__ nkept, unsigned long long* skipped) {
    __shared__ uint32_t ws[16];
    __shared__ unsigned long long s_len;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint64_t q = blockIdx.x;
    if (q >= nq)
        return;
    const uint32_t nb = aux.nlist;
    const float* qrow = queries + q * aux.dim_stride;
    float qp = 0.0f;
    for (uint32_t i = tid; i < aux.dim; i += kThreads)
        qp = __fadd_ru(qp, __fmul_ru(qrow[i], qrow[i]));
    for (int o = 16; o > 0; o >>= 1)
        qp = __fadd_ru(qp, __shfl_xor_sync(0xffffffffu, qp, o));
    if (lane == 0)
        ws[warp] = __float_as_uint(qp);
    __syncthreads();
    float qn2 = 0.0f;
    for (uint32_t w = 0; w < kWarps; ++w)
        qn2 = __fadd_ru(qn2, __uint_as_float(ws[w]));
    qn2 = __fmul_ru(qn2, 1.0f + 1.0f / 65536.0f);
    const float qn = __fsqrt_ru(qn2);
    const float rr = r2[q];
    const float T = __int_as_float(__float_as_int(rr) + 1); // pruned iff est >= the float after r^2
    const float* arow = approx + q * mma_ld(nb);
    if (tid == 0)
        s_len = 0;
    __syncthreads();
    uint32_t carry = 0;
    unsigned long long my_len = 0;
    for (uint32_t b0 = 0; b0 < nb; b0 += kThreads) {
        const uint32_t b = b0 + tid;
        bool keep = false;
        if (b < nb && aux.list_offsets[b + 1] > aux.list_offsets[b]) {
            keep = true;
            if (rr >= 0.0f) {
                const float e = __fadd_ru(__fmul_ru(__fmul_ru(qn, __ldg(cn + b)), 1.0f / 64.0f),
                                          __fmul_ru(__fadd_ru(qn2, __ldg(cn2 + b)), 1.0f / 16384.0f));
                const float dq = fmaxf(__fsub_rd(arow[b], e), 0.0f); // <= |q - c_b|^2
                keep = !(block_lower_bound(dq, __ldg(aux.list_R + b), __ldg(aux.list_xmin + b),
                                           __ldg(aux.list_xmax + b), omg_lo, omg_hi, kq1, kq2, kest) >= T);
            } else {
                keep = false; // negative radius: nothing (status reported by the caller)
            }
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0)
            ws[warp] = __popc(bal);
        __syncthreads();
        uint32_t before = carry, tot = 0;
        for (uint32_t w = 0; w < kWarps; ++w) {
            before += w < warp ? ws[w] : 0u;
            tot += ws[w];
        }
        if (keep) {
            kept[q * nb + before + __popc(bal & ((1u << lane) - 1u))] = b;
            my_len += aux.list_offsets[b + 1] - aux.list_offsets[b];
        }
        carry += tot;
        __syncthreads();
    }
    if (my_len)
        atomicAdd(&s_len, my_len);
    __syncthreads();
    if (tid == 0) {
        nkept[q] = carry;
        const unsigned long long all = aux.list_offsets[nb];
        if (skipped && all > s_len)
            atomicAdd(skipped, all - s_len); // rows pruned as whole blocks (diagnostic)
    }
}

// entry rows -> block order: codes, lx and ids gathered by the sorted rows.
__global__ void trim_partition_gather_kernel(const uint32_t* __restrict__ rows, uint64_t n, const uint8_t* __restrict__ codes,
                                             uint32_t cs, const float* __restrict__ lx, const uint32_t* __restrict__ ids,
                                             uint8_t* __restrict__ codes_o, float* __restrict__ lx_o,
                                             uint32_t* __restrict__ ids_o) {
    const uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= n)
        return;
    const uint32_t r = rows[e];
    const uint4* src = reinterpret_cast<const uint4*>(codes + static_cast<size_t>(r) * cs);
    uint4* dst = reinterpret_cast<uint4*>(codes_o + e * cs);
    for (uint32_t i = 0; i < cs / 16; ++i)
        dst[i] = src[i];
    lx_o[e] = lx[r];
    ids_o[e] = ids[r];
}

// argmin over D~ rows (block assignment of a row chunk; any partition is valid,
// the per-block bounds are computed from the actual members).
__global__ void trim_argmin_kernel(const float* __restrict__ approx, uint64_t n, uint32_t nb, uint64_t ld,
                                   uint32_t* __restrict__ out) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
    const uint32_t lane = threadIdx.x & 31u;
    if (r >= n)
        return;
    float best = __int_as_float(0x7f800000);
    uint32_t bi = 0;
    for (uint32_t b = lane; b < nb; b += 32) {
        const float d = approx[r * ld + b];
        if (d < best) {
            best = d;
            bi = b;
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
    if (lane == 0)
        out[r] = bi;
}

// rows (stride floats apart, given by index) -> a contiguous [ns x dim] sample
__global__ void trim_gather_rows_kernel(const float* __restrict__ src, uint32_t stride, const uint64_t* __restrict__ rows,
                                        uint64_t ns, uint32_t dim, float* __restrict__ dst) {
    const uint64_t i = blockIdx.x;
    if (i >= ns)
        return;
    for (uint32_t j = threadIdx.x; j < dim; j += blockDim.x)
        dst[i * dim + j] = src[rows[i] * stride + j];
}

// (segment, block) key of rows n0.. for the segmented flat kNN layout: row n0 + i
// belongs to the segment g with bounds[g] <= n0 + i < bounds[g + 1] (bounds[0] = n0) and to
// the partition's block assign[i] (`assign` points at row n0).
__global__ void trim_seg_key_kernel(const uint32_t* __restrict__ assign, uint64_t cnt, const uint64_t* __restrict__ bounds,
                                    uint32_t nseg, uint32_t nb, uint32_t* __restrict__ keys) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= cnt)
        return;
    const uint64_t r = bounds[0] + i;
    uint32_t a = 0, b = nseg; // largest g with bounds[g] <= r
    while (b - a > 1) {
        const uint32_t mid = (a + b) >> 1;
        if (bounds[mid] <= r)
            a = mid;
        else
            b = mid;
    }
    keys[i] = a * nb + assign[i];
}

// the same with 32-bit row indices
__global__ void trim_gather_rows32_kernel(const float* __restrict__ src, uint32_t stride, const uint32_t* __restrict__ rows,
                                          uint64_t ns, uint32_t dim, float* __restrict__ dst) {
    const uint64_t i = blockIdx.x;
    if (i >= ns)
        return;
    for (uint32_t j = threadIdx.x; j < dim; j += blockDim.x)
        dst[i * dim + j] = src[static_cast<size_t>(rows[i]) * stride + j];
}

// 1 if list entry e holds row e (id_base + e) for every e (flat lists in row order).
__global__ void trim_identity_check_kernel(const uint32_t* __restrict__ ids, uint64_t n, uint64_t id_base,
                                           uint32_t* __restrict__ bad) {
    const uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e < n && ids[e] != id_base + e)
        atomicOr(bad, 1u);
}

#endif // TRIM_M

} // namespace trimgpu
