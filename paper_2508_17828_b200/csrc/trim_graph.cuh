// trim_graph.cuh — sm_100a TRIM filter over an HNSW graph.
//
//   trim_graph_kernel   graph::search_trim_knn    (graph/search.hpp:188-264)
//                       graph::search_trim_range  (graph/search.hpp:267-347)
//   (both start with detail_search::descend_to_level0, graph/search.hpp:37-58)
//
// Paths are relative to /root/reference/proj/include/trimsearch.
//
// One warp per query (a graph search is a sequential best-first walk). Per hop
// the warp filters the expanded node's level-0 neighbour list in parallel —
// visited test-and-set, reference-order ADC from the query's LUT in shared
// memory, relaxed TRIM bound, and the exact L2 of every neighbour that can be
// evaluated — and then replays the neighbours in list order with the live
// thresholds, exactly as the reference's loop does (so counters, queue keys
// and results are the reference's bit for bit):
//   * the candidate queue C (capacity ef, hybrid keys) and the result queue R
//     (capacity k) are WarpTopK register sets: push + pop-if-over-capacity of
//     std::priority_queue<ScoredId> keeps the ef (k) smallest (key, id), and
//     the keys are unique (every node is pushed at most once), so the kept set
//     and the heap top are those of the reference whatever the heap layout;
//   * the search queue S (unbounded min-heap by bound) is a binary heap of
//     (key bits << 32 | id) words owned by lane 0, in shared memory; u64
//     order = ScoredId order for non-negative keys. Once C is full its top
//     max_can_dis only falls, so an entry keyed above it can never be popped
//     before the search stops (the reference breaks on the first such pop,
//     search.hpp:222-223, and stops identically on an empty queue): such
//     entries are not pushed, and are purged when the heap fills.
// Queries whose S still outgrows the shared-memory heap set status bit 0 and
// are re-run by the host with a global-memory heap of capacity n + 1
// (trim_capi.cu).
#pragma once

#include "trim_adc.cuh"
#include "trim_common.cuh"
#include "trim_kernels.cuh"

namespace trimgpu {

// GraphIndex (graph/hnsw.hpp:22-35) as per-level CSR + the LandmarkStore
// (trim/landmarks.hpp:18-28) in `ix` (codes by node id, lx, codebook, vectors).
struct GraphDev {
    DevIndex ix;
    uint32_t levels;
    uint32_t entry;
    const uint64_t* offsets;  // levels x (n + 1)
    const uint64_t* nbr_base; // levels: start of level l's adjacency in nbrs
    const uint32_t* nbrs;
};

struct GraphParams {
    const float* queries; // nq x dim_stride
    uint64_t nq;
    uint32_t k;       // kNN: result capacity
    uint32_t ef;      // candidate queue capacity
    float two_gamma;  // 2 * float(profile.gamma)
    uint32_t range;   // 0: search_trim_knn, 1: search_trim_range
    const float* r2;  // range: nq squared radii (radius * radius in fp32, search.hpp:278)
    uint32_t* ids_out;   // kNN: nq x k
    float* dist_out;     // kNN: nq x k
    unsigned long long* pool; // range: nq x cap (dist bits << 32 | id)
    uint64_t cap;
    unsigned long long* counts;   // range: nq result counts (may exceed cap)
    unsigned long long* counters; // nq x 6
    uint32_t* visited;   // nq x vwords bitmap, zeroed
    uint64_t vwords;
    unsigned long long* heap; // nq x heap_cap in global memory, or null: heap_cap entries in shared memory
    uint64_t heap_cap;
    uint32_t* status;    // nq flags: bit 0 = search queue overflow (re-run)
    const uint32_t* qmap; // null, or the query index of each CTA (re-runs of a subset)
};

constexpr uint32_t kGraphThreads = 32;

// The graph kernel's LUT is the reference's own m x ksub table (pq.hpp:158-172),
// row-major: all lanes look up the same subspace j at once, so bank = code mod
// 32 (the filter kernel's blocked layout would put them all in bank j mod 32).
__host__ __device__ inline size_t graph_lut_bytes(uint32_t m, uint32_t ksub) {
    return (sizeof(float) * m * ksub + 15) & ~size_t(15);
}
__host__ __device__ inline size_t graph_smem_bytes(uint32_t m, uint32_t ksub, uint32_t dim_stride, uint64_t smem_heap) {
    const size_t b = (graph_lut_bytes(m, ksub) + sizeof(float) * dim_stride + 7) & ~size_t(7);
    return b + sizeof(unsigned long long) * smem_heap;
}

__device__ __forceinline__ unsigned long long skey(float d, uint32_t id) {
    return (static_cast<unsigned long long>(__float_as_uint(d)) << 32) | id;
}

// Lane 0's binary min-heap (std::priority_queue<ScoredId, ..., greater>), in
// shared or global memory (generic addressing).
struct MinHeap {
    unsigned long long* h;
    uint64_t n, cap;
    __device__ __forceinline__ void sift_down(uint64_t i, unsigned long long x) {
        for (;;) {
            uint64_t c = 2 * i + 1;
            if (c >= n)
                break;
            unsigned long long hc = h[c];
            if (c + 1 < n) {
                const unsigned long long h2 = h[c + 1];
                if (h2 < hc) {
                    hc = h2;
                    ++c;
                }
            }
            if (x <= hc)
                break;
            h[i] = hc;
            i = c;
        }
        h[i] = x;
    }
    // Drop the entries keyed above `bound` (never popped before the search
    // stops) and re-heapify. Returns false if nothing could be dropped.
    __device__ __forceinline__ bool purge(unsigned long long bound) {
        uint64_t w = 0;
        for (uint64_t i = 0; i < n; ++i)
            if (h[i] <= bound)
                h[w++] = h[i];
        if (w == n)
            return false;
        n = w;
        for (uint64_t i = n / 2; i-- > 0;)
            sift_down(i, h[i]);
        return true;
    }
    // Push unless `x` is above `bound`; false when the heap is full.
    __device__ __forceinline__ bool push(unsigned long long x, unsigned long long bound) {
        if (x > bound)
            return true;
        if (n == cap && !purge(bound))
            return false;
        uint64_t i = n++;
        while (i > 0) {
            const uint64_t p = (i - 1) >> 1;
            const unsigned long long hp = h[p];
            if (hp <= x)
                break;
            h[i] = hp;
            i = p;
        }
        h[i] = x;
        return true;
    }
    __device__ __forceinline__ unsigned long long pop() {
        const unsigned long long top = h[0];
        const unsigned long long x = h[--n];
        if (n)
            sift_down(0, x);
        return top;
    }
};

// pq::adc_lookup (pq.hpp:186-192) of one code row in the reference order
// (sequential fp32 sum, j = 0..m-1) over the row-major LUT in shared memory,
// the code bytes fetched 16 at a time (rows are 16-byte aligned), the next 16
// in flight while the current ones are summed.
__device__ __forceinline__ float adc_serial_row(const uint8_t* __restrict__ code, uint32_t m, uint32_t ksub) {
    const uint32_t base = lut_saddr();
    const uint4* c4 = reinterpret_cast<const uint4*>(code);
    float acc = 0.0f;
    uint4 nxt = __ldg(c4);
    for (uint32_t j0 = 0; j0 < m; j0 += 16) {
        const uint4 w = nxt;
        if (j0 + 16 < m)
            nxt = __ldg(c4 + (j0 >> 4) + 1);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
        const uint32_t n = min(16u, m - j0);
#pragma unroll
        for (uint32_t t = 0; t < 16; ++t) {
            if (t < n) {
                const uint32_t c = (ws[t >> 2] >> (8 * (t & 3))) & 0xFFu;
                acc = __fadd_rn(acc, lds_f32(base + 4u * ((j0 + t) * ksub + c)));
            }
        }
    }
    return acc;
}

// The (d, id) lexicographic minimum over the warp (lanes with valid == false
// contribute nothing); result in every lane.
__device__ __forceinline__ void warp_argmin(float& d, uint32_t& id, bool valid) {
    if (!valid) {
        d = __int_as_float(0x7f800000);
        id = kInvalidId;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float od = __shfl_xor_sync(0xffffffffu, d, o);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, id, o);
        if (scored_less(od, oi, d, id)) {
            d = od;
            id = oi;
        }
    }
}

template <int S>
__global__ void __launch_bounds__(kGraphThreads) trim_graph_kernel(GraphDev g, GraphParams p) {
    const DevIndex& ix = g.ix;
    if (blockIdx.x >= p.nq)
        return;
    const uint32_t slot = blockIdx.x;                      // workspace slot
    const uint32_t q = p.qmap ? p.qmap[slot] : slot;       // query (inputs, outputs)
    const uint32_t lane = threadIdx.x;
    float* lut = reinterpret_cast<float*>(trim_dyn_smem); // offset 0 (lut_saddr)
    const size_t lb = graph_lut_bytes(ix.m, ix.ksub);
    float* qv = lut + lb / sizeof(float);
    unsigned long long* sheap = reinterpret_cast<unsigned long long*>(
        trim_dyn_smem + ((lb + sizeof(float) * ix.dim_stride + 7) & ~size_t(7)));
    const float* qg = p.queries + static_cast<size_t>(q) * ix.dim_stride;
    for (uint32_t i = lane; i < ix.dim_stride; i += kWarp)
        qv[i] = qg[i];
    __syncwarp();
    // pq::build_distance_table (search.hpp:204; pq.hpp:158-172): entry (j, c) =
    // euclidean_sq(q_j, C_jc, sub_dim_j) in the reference's arithmetic
    for (uint32_t i = lane; i < ix.m * ix.ksub; i += kWarp) {
        const uint32_t j = i / ix.ksub, c = i - j * ix.ksub;
        const uint32_t sd = __ldg(ix.sub_dims + j), off = __ldg(ix.sub_offsets + j);
        lut[i] = euclid_sq_generic(qv + off, ix.centroids + static_cast<size_t>(ix.ksub) * off + c * sd, sd);
    }
    __syncwarp();

    const uint64_t n = ix.n;
    auto row = [&](uint32_t v) { return ix.vectors + static_cast<size_t>(v) * ix.dim_stride; };
    auto adj = [&](uint32_t lvl, uint32_t v, const uint32_t*& nb) -> uint32_t {
        const uint64_t* o = g.offsets + static_cast<size_t>(lvl) * (n + 1);
        const uint64_t b = __ldg(o + v), e = __ldg(o + v + 1);
        nb = g.nbrs + __ldg(g.nbr_base + lvl) + b;
        return static_cast<uint32_t>(e - b);
    };
    unsigned long long dc = 0, edc = 0, pruned = 0, evaluated = 0, hops = 0;

    // ---- detail_search::descend_to_level0 (search.hpp:37-58). A pass keeps
    // the running lexicographic minimum of (d, id) over the neighbour list,
    // which is the minimum over the list whatever the order.
    uint32_t cur = g.entry;
    float cur_d = euclid_sq_vec4(qv, row(cur), ix.dim, true);
    ++dc;
    ++evaluated;
    for (uint32_t lvl = g.levels - 1; lvl > 0; --lvl) {
        for (bool changed = true; changed;) {
            changed = false;
            const uint32_t* nb;
            const uint32_t deg = adj(lvl, cur, nb);
            float bd = cur_d;
            uint32_t bi = cur;
            for (uint32_t c0 = 0; c0 < deg; c0 += kWarp) {
                const bool valid = c0 + lane < deg;
                uint32_t v = valid ? __ldg(nb + c0 + lane) : 0u;
                float d = valid ? euclid_sq_vec4(qv, row(v), ix.dim, true) : 0.0f;
                warp_argmin(d, v, valid);
                if (scored_less(d, v, bd, bi)) {
                    bd = d;
                    bi = v;
                }
            }
            dc += deg;
            evaluated += deg;
            if (bi != cur) {
                cur = bi;
                cur_d = bd;
                changed = true;
            }
        }
    }

    // ---- the TRIM walk on level 0 (search.hpp:206-262 / 284-333)
    uint32_t* vis = p.visited + static_cast<size_t>(slot) * p.vwords;
    MinHeap sq{p.heap ? p.heap + static_cast<size_t>(slot) * p.heap_cap : sheap, 0, p.heap_cap};
    WarpTopK<S> cand, res;
    cand.init(p.ef);
    res.init(p.range ? 1u : p.k);
    uint32_t cand_n = 0;
    // entries above max_can_dis (C full) are dead: the bound for pushes
    auto live_bound = [&]() -> unsigned long long {
        return cand_n == p.ef ? skey(cand.wd, 0xFFFFFFFFu) : ~0ull;
    };
    const float r2 = p.range ? p.r2[q] : 0.0f;
    unsigned long long nres = 0;
    unsigned long long* pool = p.range ? p.pool + static_cast<size_t>(q) * p.cap : nullptr;
    bool overflow = false;

    if (lane == 0)
        atomicOr(vis + (cur >> 5), 1u << (cur & 31u));
    {
        const float glq = __fsqrt_rn(adc_serial_row(ix.codes + static_cast<size_t>(cur) * ix.code_stride, ix.m, ix.ksub));
        ++edc;
        const float plb = relaxed_lb(glq, __ldg(ix.lx + cur), p.two_gamma);
        if (lane == 0)
            overflow = !sq.push(skey(plb, cur), ~0ull);
        cand.offer(cur_d, cur);
        cand_n = 1;
        if (!p.range) {
            res.offer(cur_d, cur);
        } else if (cur_d <= r2) {
            if (lane == 0)
                pool[0] = skey(cur_d, cur);
            nres = 1;
        }
    }

    for (;;) {
        // search_q.top() / pop (lane 0), then the termination test
        unsigned long long top = 0;
        uint32_t more = 0;
        if (lane == 0 && !overflow && sq.n > 0) {
            top = sq.pop();
            more = 1;
        }
        if (!__shfl_sync(0xffffffffu, more, 0))
            break;
        top = __shfl_sync(0xffffffffu, top, 0);
        const float key = __uint_as_float(static_cast<uint32_t>(top >> 32));
        const uint32_t u = static_cast<uint32_t>(top);
        if (cand_n == p.ef && key > cand.wd) // cand.size() == ef && cur.dist_sq > max_can_dis
            break;
        ++hops;
        const uint32_t* nb;
        const uint32_t deg = adj(0, u, nb);
        for (uint32_t c0 = 0; c0 < deg; c0 += kWarp) {
            const bool valid = c0 + lane < deg;
            const uint32_t v = valid ? __ldg(nb + c0 + lane) : kInvalidId;
            // visited test-and-set in list order: a repeated id in this chunk
            // defers to its first lane; earlier chunks already set their bits
            const uint32_t same = __match_any_sync(0xffffffffu, v);
            bool fresh = false;
            if (valid && (__ffs(same) - 1) == static_cast<int>(lane)) {
                const uint32_t bit = 1u << (v & 31u);
                fresh = !(atomicOr(vis + (v >> 5), bit) & bit);
            }
            float plb = 0.0f, d = 0.0f;
            if (fresh) { // pq::adc_lookup + sqrt + trim::relaxed_lb (search.hpp:229-231)
                const float glq = __fsqrt_rn(adc_serial_row(ix.codes + static_cast<size_t>(v) * ix.code_stride, ix.m, ix.ksub));
                plb = relaxed_lb(glq, __ldg(ix.lx + v), p.two_gamma);
                // exact distance for every neighbour the replay may evaluate:
                // cand only grows and max_dis only falls during the hop
                const bool need = cand_n < p.ef || (p.range ? plb <= r2 : plb < res.wd);
                if (need)
                    d = euclid_sq_vec4(qv, row(v), ix.dim, true);
            }
            uint32_t fm = __ballot_sync(0xffffffffu, fresh);
            evaluated += __popc(fm);
            edc += __popc(fm);
            // Neighbours the replay would only count as pruned: C is full (it
            // stays full) and the bound is at or above both max_dis (or beyond
            // the radius) and max_can_dis now — both only fall during the
            // replay, so at their turn they take the pruned branch without a
            // push (search.hpp:249-259).
            const bool idle = fresh && cand_n == p.ef && (p.range ? plb > r2 : plb >= res.wd) && !(plb < cand.wd);
            const uint32_t im = __ballot_sync(0xffffffffu, idle);
            pruned += __popc(im);
            fm &= ~im;
            while (fm) { // the reference's per-neighbour decisions, in list order
                const uint32_t j = __ffs(fm) - 1;
                fm &= fm - 1;
                const float pj = __shfl_sync(0xffffffffu, plb, j);
                const float dj = __shfl_sync(0xffffffffu, d, j);
                const uint32_t vj = __shfl_sync(0xffffffffu, v, j);
                if (cand_n < p.ef || (p.range ? pj <= r2 : pj < res.wd)) {
                    ++dc;
                    if (p.range && dj <= r2) {
                        if (lane == 0 && nres < p.cap)
                            pool[nres] = skey(dj, vj);
                        ++nres;
                    }
                    if (lane == 0 && !overflow)
                        overflow = !sq.push(skey(pj, vj), live_bound());
                    cand.offer(dj, vj);
                    cand_n = min(cand_n + 1, p.ef);
                    if (!p.range)
                        res.offer(dj, vj);
                } else {
                    ++pruned;
                    if (pj < cand.wd) { // plb < max_can_dis
                        if (lane == 0 && !overflow)
                            overflow = !sq.push(skey(pj, vj), live_bound());
                        cand.offer(pj, vj);
                        cand_n = min(cand_n + 1, p.ef);
                    }
                }
            }
        }
        if (__shfl_sync(0xffffffffu, overflow ? 1u : 0u, 0))
            break;
    }
    if (__shfl_sync(0xffffffffu, overflow ? 1u : 0u, 0)) {
        if (lane == 0)
            p.status[q] |= 1u;
        return;
    }
    if (!p.range)
        res.store_sorted(p.k, p.ids_out + static_cast<size_t>(q) * p.k, p.dist_out + static_cast<size_t>(q) * p.k);
    else if (lane == 0)
        p.counts[q] = nres;
    if (lane == 0) {
        unsigned long long* cc = p.counters + static_cast<size_t>(q) * 6;
        cc[0] = dc;
        cc[1] = edc;
        cc[2] = pruned;
        cc[3] = evaluated;
        cc[4] = hops;
        cc[5] = 0;
    }
}

} // namespace trimgpu
