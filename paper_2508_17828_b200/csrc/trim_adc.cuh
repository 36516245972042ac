// trim_adc.cuh — conflict-free ADC over a shared-memory PQ lookup table.
//
// The reference ADC (pq/pq.hpp:186-192) is a sequential fp32 sum over
// j = 0..m-1 of LUT[j][code_j]. With the natural [j][c] layout, 32 lanes
// reading the same subspace hit banks code % 32 at random (~3.5-way
// conflicts, measured).
//
// Layout here ("blocked"). Subspaces are grouped in blocks of 32 columns; a
// FULL block is 256 rows (= codes) x 32 floats, so an entry's bank is its
// column. The last block may be a HALF block (<= 16 live columns): 256 rows
// x 16 floats — two lanes then share each column (2-way conflicts on those
// lookups) — or, when it is the only block (m <= 16), 16 columns stored
// twice (32 floats per row, conflict-free). Partial blocks are padded with
// zero columns (adding +0.0f to a non-negative sum is exact). m = 48 takes
// 32 KB + 16 KB.
//
// Two schedules:
//   FastCode (fast) — lane l reads column l ^ s at step s, so the 32 lanes
//               read 32 distinct banks; any-order fp32 sum with four partial
//               accumulators, used with a rigorous error interval
//               (est_lower_bound) to decide which candidates can possibly
//               pass the threshold;
//   adc_exact — lane l reads column (l + s) mod 32 and adds the values in
//               exactly the reference order j = 0, 1, ... (two predicated
//               passes), bit-identical to pq::adc_lookup. Used for the
//               candidates the interval cannot decide and for the survivors.
// A lookup is PRMT (code byte) + LOP3 (lane column, with the shared base
// folded in) + IMAD (row) + LDS + FADD.
#pragma once

#include "trim_common.cuh"

// The dynamic shared-memory window of every TRIM kernel; the LUT sits at
// offset 0.
extern __shared__ __align__(16) unsigned char trim_dyn_smem[];

namespace trimgpu {

constexpr uint32_t kFullBytes = 256u * 32u * 4u; // 32 KB

// Block structure of m subspaces.
struct LutShape {
    uint32_t nfull; // 32-column blocks (incl. a zero-padded 17..31 tail)
    uint32_t half;  // 1 if the last block has <= 16 live columns
    uint32_t hdup;  // the HALF block is duplicated (only when it is the only block)
    __host__ __device__ static LutShape of(uint32_t m) {
        LutShape s;
        const uint32_t rem = m & 31u;
        s.nfull = m >> 5;
        s.half = 0;
        if (rem > 16)
            ++s.nfull;
        else if (rem)
            s.half = 1;
        s.hdup = s.half && s.nfull == 0;
        return s;
    }
    __host__ __device__ uint32_t blocks() const { return nfull + half; }
    __host__ __device__ uint32_t half_row_bytes() const { return hdup ? 128u : 64u; }
    __host__ __device__ size_t bytes() const {
        return static_cast<size_t>(nfull) * kFullBytes + (half ? 256u * half_row_bytes() : 0u);
    }
};

__host__ __device__ inline size_t lut_bytes(int /*M_template*/, uint32_t m) { return LutShape::of(m).bytes(); }

// pq::build_distance_table (pq.hpp:158-172) into the blocked layout. Entry
// values are the reference's euclidean_sq, bit for bit.
// Entry (j, c) = euclidean_sq of a 2-, 4- or 8-wide subspace, the reference's
// four-accumulator order collapsed: acc_i = 0 + d_i^2 exactly, unused
// accumulators are +0.0f; at 8, acc_i = d_i^2 + d_{i+4}^2.
template <uint32_t SD>
__device__ __forceinline__ float sub_dist(const float* q, const float* c) {
    if (SD == 2) {
        const float2 v = __ldg(reinterpret_cast<const float2*>(c));
        const float d0 = __fsub_rn(q[0], v.x), d1 = __fsub_rn(q[1], v.y);
        return __fadd_rn(__fmul_rn(d0, d0), __fmul_rn(d1, d1));
    } else if (SD == 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(c));
        const float d0 = __fsub_rn(q[0], v.x), d1 = __fsub_rn(q[1], v.y);
        const float d2 = __fsub_rn(q[2], v.z), d3 = __fsub_rn(q[3], v.w);
        return __fadd_rn(__fadd_rn(__fmul_rn(d0, d0), __fmul_rn(d1, d1)),
                         __fadd_rn(__fmul_rn(d2, d2), __fmul_rn(d3, d3)));
    } else {
        const float4 v = __ldg(reinterpret_cast<const float4*>(c));
        const float4 w = __ldg(reinterpret_cast<const float4*>(c) + 1);
        const float d0 = __fsub_rn(q[0], v.x), d1 = __fsub_rn(q[1], v.y);
        const float d2 = __fsub_rn(q[2], v.z), d3 = __fsub_rn(q[3], v.w);
        const float e0 = __fsub_rn(q[4], w.x), e1 = __fsub_rn(q[5], w.y);
        const float e2 = __fsub_rn(q[6], w.z), e3 = __fsub_rn(q[7], w.w);
        const float a0 = __fadd_rn(__fmul_rn(d0, d0), __fmul_rn(e0, e0));
        const float a1 = __fadd_rn(__fmul_rn(d1, d1), __fmul_rn(e1, e1));
        const float a2 = __fadd_rn(__fmul_rn(d2, d2), __fmul_rn(e2, e2));
        const float a3 = __fadd_rn(__fmul_rn(d3, d3), __fmul_rn(e3, e3));
        return __fadd_rn(__fadd_rn(a0, a1), __fadd_rn(a2, a3));
    }
}

// Store entry (j, c) of the blocked table (bank = column j & 31).
__device__ __forceinline__ void lut_store(float* lut, const LutShape& sh, uint32_t j, uint32_t c, float v) {
    const uint32_t b = j >> 5, t = j & 31u;
    if (b < sh.nfull) {
        lut[b * (kFullBytes / 4) + c * 32 + t] = v;
    } else {
        float* hblk = lut + sh.nfull * (kFullBytes / 4);
        const uint32_t hrow = sh.half_row_bytes() / 4;
        hblk[c * hrow + t] = v;
        if (sh.hdup)
            hblk[c * hrow + t + 16] = v;
    }
}

// Uniform 2-, 4- or 8-wide subspaces. Entry i -> (c = i / m, j = i % m):
// consecutive threads take consecutive subspaces of one code, so a warp reads
// one contiguous run of the code-major centroid copy (ix.centroids_t, 32*SD
// floats) and writes 32 distinct banks of one table row (the j-major order,
// c fastest, put all 32 lanes of a store in one bank). 8 entries in flight
// per thread.
template <uint32_t SD, int M>
__device__ __forceinline__ void build_lut_uniform(const DevIndex& ix, const float* q_smem, float* lut,
                                                  const LutShape& sh, uint32_t t0, uint32_t nt) {
    const uint32_t m = M > 0 ? static_cast<uint32_t>(M) : ix.m, total = m * ix.ksub; // M: constant divisor
    for (uint32_t i0 = t0; i0 < total; i0 += 8 * nt) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t i = i0 + u * nt;
            const uint32_t c = i / m, j = i - c * m;
            v[u] = i < total ? sub_dist<SD>(q_smem + j * SD, ix.centroids_t + static_cast<size_t>(i) * SD) : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t i = i0 + u * nt;
            if (i >= total)
                break;
            const uint32_t c = i / m, j = i - c * m;
            lut_store(lut, sh, j, c, v[u]);
        }
    }
}

// Threads t0 (of nt participating) build the table; defaults: the whole CTA.
// M > 0: the kernel's compile-time code length (= ix.m).
template <int M = 0>
__device__ __forceinline__ void build_lut_blocked(const DevIndex& ix, const float* q_smem, float* lut,
                                                  uint32_t t0 = threadIdx.x, uint32_t nt = blockDim.x) {
    const LutShape sh = LutShape::of(ix.m);
    const uint32_t hrow = sh.half_row_bytes() / 4;          // floats per HALF row
    float* hblk = lut + sh.nfull * (kFullBytes / 4);
    if (ix.sd_uniform == 2)
        build_lut_uniform<2, M>(ix, q_smem, lut, sh, t0, nt);
    else if (ix.sd_uniform == 4)
        build_lut_uniform<4, M>(ix, q_smem, lut, sh, t0, nt);
    else if (ix.sd_uniform == 8)
        build_lut_uniform<8, M>(ix, q_smem, lut, sh, t0, nt);
    else // mixed widths: the same code-major order, widths and offsets per subspace
        for (uint32_t i = t0; i < ix.m * ix.ksub; i += nt) {
            const uint32_t c = i / ix.m, j = i - c * ix.m;
            const uint32_t off = __ldg(ix.sub_offsets + j);
            lut_store(lut, sh, j, c,
                      euclid_sq_generic(q_smem + off, ix.centroids_t + static_cast<size_t>(c) * ix.dim + off,
                                        __ldg(ix.sub_dims + j)));
        }
    // zero every non-live column of the last block: both schedules read all
    // columns, and +0.0f leaves the sum unchanged
    const uint32_t rem = ix.m & 31u;
    if (rem) {
        const uint32_t width = sh.half ? 16u : 32u;
        const uint32_t pad = width - rem;
        for (uint32_t i = t0; i < 256 * pad; i += nt) {
            const uint32_t c = i / pad, t = rem + i % pad;
            if (sh.half) {
                hblk[c * hrow + t] = 0.0f;
                if (sh.hdup)
                    hblk[c * hrow + t + 16] = 0.0f;
            } else {
                lut[(ix.m >> 5) * (kFullBytes / 4) + c * 32 + t] = 0.0f;
            }
        }
    }
}

__device__ __forceinline__ uint32_t sel32(bool p, uint32_t a, uint32_t b) { return p ? a : b; }

// Shared-memory load at a 32-bit .shared window address.
__device__ __forceinline__ float lds_f32(uint32_t saddr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(saddr));
    return v;
}

// .shared window address of the LUT (a multiple of 128: the per-lane column
// bits can be XORed into it).
__device__ __forceinline__ uint32_t lut_saddr() {
    return static_cast<uint32_t>(__cvta_generic_to_shared(trim_dyn_smem));
}

// Per-lane constants of the fast schedule.
struct LaneAdc {
    uint32_t l;      // lane
    uint32_t lf;     // LUT base + 4*l       (FULL blocks: column l ^ s)
    uint32_t lh;     // HALF base + 4*lane'  (lane' = l, or l & 15 without duplication)
    uint32_t sel[4]; // PRMT selectors: output byte 0 = code byte (q ^ (l & 3))
    __device__ __forceinline__ void init(uint32_t lane, const LutShape& sh) {
        l = lane;
        const uint32_t base = lut_saddr();
        lf = base + 4u * lane;
        lh = base + sh.nfull * kFullBytes + 4u * (sh.hdup ? lane : (lane & 15u));
        const uint32_t x = lane & 3u;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            sel[q] = 0x4440u | (static_cast<uint32_t>(q) ^ x);
    }
};

// Code words of one block for the fast schedule. load_block_fast only issues
// the loads (so a prefetch has no dependent instructions); the top bit of the
// word permutation (wl = (l >> 2) & (NW-1)) is applied by the load addresses
// (16-byte halves of a FULL block, 8-byte halves of a HALF block), and
// permute_block applies the rest with selects, leaving word i = original
// word i ^ wl.
template <bool HALF>
__device__ __forceinline__ void load_block_fast(const uint8_t* __restrict__ code, uint32_t b, uint32_t l,
                                                uint32_t w[8]) {
    if (!HALF) {
        const uint32_t top = (l >> 4) & 1u; // bit 2 of wl
        const uint4* p = reinterpret_cast<const uint4*>(code + 32 * b);
        const uint4 a = __ldg(p + top);
        const uint4 c = __ldg(p + (top ^ 1u));
        w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
        w[4] = c.x; w[5] = c.y; w[6] = c.z; w[7] = c.w;
    } else {
        const uint32_t top = (l >> 3) & 1u; // bit 1 of wl
        const uint2* p = reinterpret_cast<const uint2*>(code + 32 * b);
        const uint2 a = __ldg(p + top);
        const uint2 c = __ldg(p + (top ^ 1u));
        w[0] = a.x; w[1] = a.y; w[2] = c.x; w[3] = c.y;
    }
}

template <bool HALF>
__device__ __forceinline__ void permute_block(uint32_t w[8], uint32_t l) {
    const bool b0 = (l >> 2) & 1u;
    if (!HALF) {
        const bool b1 = (l >> 3) & 1u;
        uint32_t t[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
            t[i] = sel32(b0, w[i ^ 1], w[i]);
#pragma unroll
        for (int i = 0; i < 8; ++i)
            w[i] = sel32(b1, t[i ^ 2], t[i]);
    } else {
        const uint32_t a = sel32(b0, w[1], w[0]), b = sel32(b0, w[0], w[1]);
        const uint32_t c = sel32(b0, w[3], w[2]), d = sel32(b0, w[2], w[3]);
        w[0] = a; w[1] = b; w[2] = c; w[3] = d;
    }
}

// Any-order sum of steps [S0, S1) of one block; lane reads column l ^ s at
// step s. ROWB = row bytes; IMM = block byte offset (folds into the LDS
// immediate). Four partial sums keep four independent FADD chains in flight.
template <int S0, int S1, uint32_t ROWB, uint32_t IMM>
__device__ __forceinline__ void block_fast(uint32_t lbase, const uint32_t w[8], const LaneAdc& la,
                                           float part[4]) {
#pragma unroll
    for (int s = S0; s < S1; ++s) {
        const uint32_t c = __byte_perm(w[s >> 2], 0, la.sel[s & 3]);
        const uint32_t col = lbase ^ (static_cast<uint32_t>(s) << 2);
        part[s & 3] = __fadd_rn(part[s & 3], lds_f32(c * ROWB + col + IMM));
    }
}

__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Early-exit test on a PARTIAL any-order ADC sum a_p (a subset of the m
// non-negative LUT terms, so adc_ref >= a_p(1-eps)). est(g) = (g-x)^2 +
// 2*gamma*g*x is increasing for g >= (1-gamma)*x; if g_lo = sqrt(a_p(1-eps))
// is already there, est_ref >= est(g_lo) and the candidate is provably
// pruned when that (rounded down, then shrunk by 4u for the reference's own
// rounding) is >= T. omg_hi = 1 - gamma rounded up.
struct StageCheck {
    static constexpr bool kFine = false; // stages after 8 (first block), 16 and 32 lookups of a block
    static constexpr bool kHalfMid = false, kAt24 = false, kNo8 = false, kNo16 = false, kNo32 = false;
    float glx, two_gamma, omg_hi, eps, T;
    __device__ __forceinline__ bool pruned(float a_p) const {
        const float g_lo = __fmul_rd(sqrt_approx(__fmul_rd(a_p, 1.0f - eps)), 1.0f - 1.0f / 65536.0f);
        if (!(g_lo >= __fmul_ru(omg_hi, glx)))
            return false;
        const float d_lo = __fsub_rd(g_lo, glx), d_hi = __fsub_ru(g_lo, glx);
        const float e = d_lo >= 0.0f ? __fmul_rd(d_lo, d_lo) : (d_hi <= 0.0f ? __fmul_rd(d_hi, d_hi) : 0.0f);
        const float t = __fmul_rd(__fmul_rd(two_gamma, g_lo), glx);
        return __fmul_rd(__fadd_rd(e, t), 1.0f - 4.0f / 16777216.0f) >= T;
    }
};

// The same test as one comparison per stage: the partial sum against a cut
// A computed once per candidate. With x = glx, est(g) = (g - (1-γ)x)^2 +
// γ(2-γ)x^2 is increasing for g >= (1-γ)x, so est(g) >= T' for every
// g >= g* = (1-γ)x + sqrt(max(T' - γ(2-γ)x^2, 0)), where T' = T(1 + 2^-20)
// absorbs the reference's own evaluation error (fl(est) >= est(1 - 4u), u =
// 2^-24). Every operation below is rounded toward a larger G >= g*, and
// A = G^2 kA with kA >= 1 / ((1 - eps)(1 - u)^2) gives: a_p >= A => adc_ref >=
// a_p(1 - eps) => g_ref = fl(sqrt(adc_ref)) >= G => est_ref >= T: the
// reference prunes the candidate (ivf.hpp:275). c1 <= γ(2-γ) and kA come from
// the host (KnnParams.stage_c1 / stage_ka). Cheap enough to test after every
// 8 lookups (kFine).
#ifndef TRIM_STAGE_FINE
#define TRIM_STAGE_FINE 0 // StageCut stages: 0 = after 8 (first block), 16, 32 like StageCheck (measured
                          // best on config 2); 1 = every 8 lookups; 2 = 0 + the middle of the last
                          // half block; 3 = 0 + after 24
#endif
struct StageCut {
    static constexpr bool kFine = TRIM_STAGE_FINE == 1;
    static constexpr bool kHalfMid = TRIM_STAGE_FINE == 1 || TRIM_STAGE_FINE == 2;
    static constexpr bool kAt24 = TRIM_STAGE_FINE == 3;
    static constexpr bool kNo8 = TRIM_STAGE_FINE >= 4, kNo16 = TRIM_STAGE_FINE >= 4; // 4: after 32 only
    static constexpr bool kNo32 = TRIM_STAGE_FINE == 5;                              // 5: no stage at all
    float a_hi;
    __device__ __forceinline__ static StageCut make(float x, float c1, float omg_hi, float kA, float T) {
        const float t_lo = c1 >= 0.0f ? __fmul_rd(c1, __fmul_rd(x, x)) : __fmul_rd(c1, __fmul_ru(x, x));
        const float rad = __fsub_ru(__fmul_ru(T, 1.0f + 1.0f / 1048576.0f), t_lo);
        const float G = fmaxf(__fadd_ru(__fmul_ru(omg_hi, x), __fsqrt_ru(fmaxf(rad, 0.0f))), 0.0f);
        return StageCut{__fmul_ru(__fmul_ru(G, G), kA)};
    }
    __device__ __forceinline__ bool pruned(float a_p) const { return a_p >= a_hi; }
};

// No stage at all: for streams whose candidates are all near the threshold (what the
// list-level bound or the block plan leaves), where a warp's 32 lanes are almost never
// all proven pruned before the last lookup and every stage is overhead (config 2: +14%).
struct StageNone {
    static constexpr bool kFine = false, kHalfMid = false, kAt24 = false, kNo8 = true, kNo16 = true, kNo32 = true;
    __device__ __forceinline__ bool pruned(float) const { return false; }
};

__device__ __forceinline__ float sum4(const float p[4]) {
    return __fadd_rn(__fadd_rn(p[0], p[1]), __fadd_rn(p[2], p[3]));
}

// Fast ADC split into load (global -> registers) and a staged sum, so a
// thread can have the next candidate's loads in flight while it sums the
// current one, and a warp whose candidates are all provably pruned stops
// after the first 16 (or 32, 64, ...) subspaces.
template <int M>
struct FastCode {
    static constexpr uint32_t kMaxB = M > 0 ? (static_cast<uint32_t>(M) + 31) / 32 : 4;
    uint32_t w[kMaxB][8];

    __device__ __forceinline__ void load(const uint8_t* __restrict__ code, uint32_t m, uint32_t l) {
        const LutShape sh = LutShape::of(M > 0 ? static_cast<uint32_t>(M) : m);
#pragma unroll
        for (uint32_t b = 0; b < kMaxB; ++b) {
            if (b < sh.nfull)
                load_block_fast<false>(code, b, l, w[b]);
            else if (b == sh.nfull && sh.half)
                load_block_fast<true>(code, b, l, w[b]);
        }
    }

    // Zero exactly the words load() would write (dead lanes still step through
    // the schedule; unused words must stay dead for the register allocator).
    __device__ __forceinline__ void zero(uint32_t m) {
        const LutShape sh = LutShape::of(M > 0 ? static_cast<uint32_t>(M) : m);
#pragma unroll
        for (uint32_t b = 0; b < kMaxB; ++b) {
            const uint32_t nw = b < sh.nfull ? 8u : (b == sh.nfull && sh.half ? 4u : 0u);
#pragma unroll
            for (uint32_t i = 0; i < 8; ++i)
                if (i < nw)
                    w[b][i] = 0;
        }
    }

    // Apply the lane's word permutation to every block once (for callers that
    // run several LUTs over the same code: sum_staged<false>).
    __device__ __forceinline__ void permute_all(uint32_t m, const LaneAdc& la) {
        const LutShape sh = LutShape::of(M > 0 ? static_cast<uint32_t>(M) : m);
#pragma unroll
        for (uint32_t b = 0; b < kMaxB; ++b) {
            if (b < sh.nfull)
                permute_block<false>(w[b], la.l);
            else if (b == sh.nfull && sh.half)
                permute_block<true>(w[b], la.l);
        }
    }

    // One FULL block B (compile-time), two 16-step stages. Returns true when
    // the whole warp is provably pruned. lofs: byte offset of the LUT used.
    template <uint32_t B, bool PERM, class CK>
    __device__ __forceinline__ bool full_block(const LutShape& sh, const LaneAdc& la, const CK& ck,
                                               float part[4], bool& live, uint32_t lofs) {
        if (B >= sh.nfull)
            return false;
        if (PERM)
            permute_block<false>(w[B], la.l);
        const uint32_t lb = la.lf + lofs;
        if constexpr (CK::kFine) { // a stage every 8 lookups
            block_fast<0, 8, 128u, B * kFullBytes>(lb, w[B], la, part);
            if (live && ck.pruned(sum4(part)))
                live = false;
            if (!__any_sync(0xffffffffu, live))
                return true;
            block_fast<8, 16, 128u, B * kFullBytes>(lb, w[B], la, part);
            if (live && ck.pruned(sum4(part)))
                live = false;
            if (!__any_sync(0xffffffffu, live))
                return true;
            block_fast<16, 24, 128u, B * kFullBytes>(lb, w[B], la, part);
            if (live && ck.pruned(sum4(part)))
                live = false;
            if (!__any_sync(0xffffffffu, live))
                return true;
            block_fast<24, 32, 128u, B * kFullBytes>(lb, w[B], la, part);
            if (B + 1 == sh.nfull && !sh.half)
                return false; // last block: the caller's full check decides
            if (live && ck.pruned(sum4(part)))
                live = false;
            return !__any_sync(0xffffffffu, live);
        }
        if (B == 0 && !CK::kNo8) { // an extra early stage after 8 lookups: ~2/3 of config-2 warps stop here
            block_fast<0, 8, 128u, B * kFullBytes>(lb, w[B], la, part);
            if (live && ck.pruned(sum4(part)))
                live = false;
            if (!__any_sync(0xffffffffu, live))
                return true;
            block_fast<8, 16, 128u, B * kFullBytes>(lb, w[B], la, part);
        } else {
            block_fast<0, 16, 128u, B * kFullBytes>(lb, w[B], la, part);
        }
        if constexpr (!CK::kNo16) {
            if (live && ck.pruned(sum4(part)))
                live = false;
            if (!__any_sync(0xffffffffu, live))
                return true;
        }
        if constexpr (CK::kAt24) {
            block_fast<16, 24, 128u, B * kFullBytes>(lb, w[B], la, part);
            if (live && ck.pruned(sum4(part)))
                live = false;
            if (!__any_sync(0xffffffffu, live))
                return true;
            block_fast<24, 32, 128u, B * kFullBytes>(lb, w[B], la, part);
        } else {
            block_fast<16, 32, 128u, B * kFullBytes>(lb, w[B], la, part);
        }
        if ((B + 1 == sh.nfull && !sh.half) || CK::kNo32)
            return false; // last block: the caller's full check decides
        if (live && ck.pruned(sum4(part)))
            live = false;
        return !__any_sync(0xffffffffu, live);
    }

    // Full any-order sum, or a negative value if a stage proved est >= T for
    // this lane. `alive` = this lane has a candidate; dead lanes still step
    // along (their lookups keep the schedule conflict-free) but never vote.
    // Warp-collective. PERM = false: the words were permuted by permute_all.
    template <bool PERM = true, class CK = StageCheck>
    __device__ __forceinline__ float sum_staged(uint32_t m, const LaneAdc& la, const CK& ck,
                                                bool alive, uint32_t lofs = 0) {
        const LutShape sh = LutShape::of(M > 0 ? static_cast<uint32_t>(M) : m);
        float part[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        bool live = alive;
        if (full_block<0, PERM, CK>(sh, la, ck, part, live, lofs))
            return -1.0f;
        if (kMaxB > 1 && full_block<(kMaxB > 1 ? 1u : 0u), PERM, CK>(sh, la, ck, part, live, lofs))
            return -1.0f;
        if (kMaxB > 2 && full_block<(kMaxB > 2 ? 2u : 0u), PERM, CK>(sh, la, ck, part, live, lofs))
            return -1.0f;
        if (kMaxB > 3 && full_block<(kMaxB > 3 ? 3u : 0u), PERM, CK>(sh, la, ck, part, live, lofs))
            return -1.0f;
        if (sh.half) {
            const uint32_t hb = sh.nfull;
            uint32_t* wh = w[0];
#pragma unroll
            for (uint32_t b = 1; b < kMaxB; ++b)
                if (b == hb)
                    wh = w[b];
            if (PERM)
                permute_block<true>(wh, la.l);
            const uint32_t hl = la.lh + lofs;
            if ((sh.hdup && !CK::kNo8) || CK::kHalfMid) { // (the only block, m <= 16:) an early check after 8 steps
                if (sh.hdup)
                    block_fast<0, 8, 128u, 0u>(hl, wh, la, part);
                else
                    block_fast<0, 8, 64u, 0u>(hl, wh, la, part);
                if (live && ck.pruned(sum4(part)))
                    live = false;
                if (!__any_sync(0xffffffffu, live))
                    return -1.0f;
                if (sh.hdup)
                    block_fast<8, 16, 128u, 0u>(hl, wh, la, part);
                else
                    block_fast<8, 16, 64u, 0u>(hl, wh, la, part);
            } else if (sh.hdup) {
                block_fast<0, 16, 128u, 0u>(hl, wh, la, part);
            } else {
                block_fast<0, 16, 64u, 0u>(hl, wh, la, part);
            }
        }
        return live ? sum4(part) : -1.0f;
    }
};

// ------------------------------------------------------- exact (reference order)
__device__ __forceinline__ void load_block_plain(const uint8_t* __restrict__ code, uint32_t b, bool half,
                                                 uint32_t w[8]) {
    const uint4* p = reinterpret_cast<const uint4*>(code + 32 * b);
    const uint4 a = __ldg(p);
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
    if (!half) {
        const uint4 c = __ldg(p + 1);
        w[4] = c.x; w[5] = c.y; w[6] = c.z; w[7] = c.w;
    } else {
        w[4] = w[5] = w[6] = w[7] = 0;
    }
}

// Rotate the NW words (4*NW bytes) left by r bytes: byte s <- byte (s + r) mod (4*NW).
template <int NW>
__device__ __forceinline__ void rot_bytes(uint32_t w[8], uint32_t r) {
    const uint32_t wr = (r >> 2) & (NW - 1);
#pragma unroll
    for (int k = 1; k < NW; k <<= 1) {
        const bool p = wr & k;
        uint32_t t[8];
#pragma unroll
        for (int i = 0; i < NW; ++i)
            t[i] = sel32(p, w[(i + k) & (NW - 1)], w[i]);
#pragma unroll
        for (int i = 0; i < NW; ++i)
            w[i] = t[i];
    }
    const uint32_t sh = 8 * (r & 3u);
    uint32_t t[8];
#pragma unroll
    for (int i = 0; i < NW; ++i)
        t[i] = __funnelshift_r(w[i], w[(i + 1) & (NW - 1)], sh);
#pragma unroll
    for (int i = 0; i < NW; ++i)
        w[i] = t[i];
}

// Exact sequential block sum: the lane reads column (r + s) mod S at step s
// (r = its rotation), so values arrive in column order r, r+1, ..., S-1,
// 0, ..., r-1; the reference order 0..S-1 is restored by adding the wrapped
// part (s >= S-r) first, then the rest. b0 = address of column r in row 0.
template <int S>
__device__ __forceinline__ float block_exact(uint32_t b0, uint32_t rowb, uint32_t w[8], uint32_t r,
                                             float acc) {
    constexpr int NW = S / 4;
    rot_bytes<NW>(w, r);
    const uint32_t b1 = b0 - 4 * S; // wrapped (s >= S - r)
    float v[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const uint32_t c = (w[s >> 2] >> (8 * (s & 3))) & 0xFFu;
        const bool wrap = static_cast<uint32_t>(s) + r >= S;
        v[s] = lds_f32(c * rowb + (wrap ? b1 : b0) + 4 * s);
    }
#pragma unroll
    for (int s = 0; s < S; ++s)
        if (static_cast<uint32_t>(s) + r >= S)
            acc = __fadd_rn(acc, v[s]);
#pragma unroll
    for (int s = 0; s < S; ++s)
        if (static_cast<uint32_t>(s) + r < S)
            acc = __fadd_rn(acc, v[s]);
    return acc;
}

template <int M>
__device__ __forceinline__ float adc_exact(const uint8_t* __restrict__ code, uint32_t m, uint32_t l) {
    const uint32_t mm = M > 0 ? static_cast<uint32_t>(M) : m;
    const LutShape sh = LutShape::of(mm);
    const uint32_t base = lut_saddr();
    float acc = 0.0f;
    uint32_t w[8];
    constexpr uint32_t kMaxB = M > 0 ? (static_cast<uint32_t>(M) + 31) / 32 : 4;
#pragma unroll
    for (uint32_t b = 0; b < kMaxB; ++b) {
        if (b >= sh.nfull)
            break;
        load_block_plain(code, b, false, w);
        acc = block_exact<32>(base + b * kFullBytes + 4 * l, 128u, w, l, acc);
    }
    if (sh.half) {
        load_block_plain(code, sh.nfull, true, w);
        const uint32_t r = l & 15u;
        const uint32_t hb = base + sh.nfull * kFullBytes + (sh.hdup ? 64u * (l >> 4) : 0u) + 4 * r;
        acc = block_exact<16>(hb, sh.half_row_bytes(), w, r, acc);
    }
    return acc;
}

// --------------------------------------------------------- rigorous interval
// Any two fp32 summations of the same m non-negative terms, each in any
// order or tree (height <= k), differ by at most 2*gamma_k/(1-gamma_k) times
// either result (gamma_k = k*u/(1-k*u), u = 2^-24; Higham, "Accuracy and
// Stability of Numerical Algorithms", eq. 4.4). The fast sum adds +0.0f
// zero-padding terms and at most 6 extra partial-sum combines per block;
// adc_rel_eps(m) uses k = m + 8*blocks and doubles the bound. The same eps
// bounds a partial sum from above by the reference's full sum (the omitted
// terms are non-negative).
__host__ __device__ inline float adc_rel_eps(uint32_t m) {
    const double u = 1.0 / 16777216.0;
    const double k = static_cast<double>(m + 8 * LutShape::of(m).blocks());
    const double g = k * u / (1.0 - k * u);
    return static_cast<float>(2.0 * (2.0 * g / (1.0 - g)));
}

// Lower bound on the reference's est = relaxed_lb(sqrt(adc_ref), glx, gamma)
// (lower_bound.hpp:18-22) given any-order sum a of the same terms:
// adc_ref in [a(1-eps), a(1+eps)], then every reference operation
// (sqrt, sub, square, products, add; each correctly rounded, monotone) is
// bounded with directed rounding. sqrt.approx (rel. error < 2^-21) is
// widened by 2^-16.
__device__ __forceinline__ float est_lower_bound(float a, float glx, float two_gamma, float eps) {
    const float a_lo = __fmul_rd(a, 1.0f - eps);
    const float a_hi = __fmul_ru(a, 1.0f + eps);
    const float g_lo = __fmul_rd(sqrt_approx(a_lo), 1.0f - 1.0f / 65536.0f);
    const float g_hi = __fmul_ru(sqrt_approx(a_hi), 1.0f + 1.0f / 65536.0f);
    const float d_lo = __fsub_rd(g_lo, glx);
    const float d_hi = __fsub_ru(g_hi, glx);
    float e_lo = 0.0f;
    if (d_lo > 0.0f)
        e_lo = __fmul_rd(d_lo, d_lo);
    else if (d_hi < 0.0f)
        e_lo = __fmul_rd(d_hi, d_hi);
    const float t_lo = __fmul_rd(__fmul_rd(two_gamma, g_lo), glx);
    return __fadd_rd(e_lo, t_lo);
}

// Upper bound on the same est (mirror image of est_lower_bound): every
// reference operation is monotone in its inputs, so the largest inputs with
// upward rounding bound each intermediate from above.
__device__ __forceinline__ float est_upper_bound(float a, float glx, float two_gamma, float eps) {
    const float a_lo = __fmul_rd(a, 1.0f - eps);
    const float a_hi = __fmul_ru(a, 1.0f + eps);
    const float g_lo = __fmul_rd(sqrt_approx(a_lo), 1.0f - 1.0f / 65536.0f);
    const float g_hi = __fmul_ru(sqrt_approx(a_hi), 1.0f + 1.0f / 65536.0f);
    const float d_lo = __fsub_rd(g_lo, glx);
    const float d_hi = __fsub_ru(g_hi, glx);
    const float e_hi = fmaxf(__fmul_ru(d_lo, d_lo), __fmul_ru(d_hi, d_hi));
    const float t_hi = __fmul_ru(__fmul_ru(two_gamma, g_hi), glx);
    return __fadd_ru(e_hi, t_hi);
}

// pq::adc_lookup (pq.hpp:186-192) by one thread over the blocked LUT:
// sequential fp32 sum in the reference order j = 0..m-1. For the rare
// candidates whose est interval straddles the live threshold.
template <int M>
__device__ __forceinline__ float adc_serial(const uint8_t* __restrict__ code, uint32_t m, uint32_t lofs = 0) {
    const uint32_t mm = M > 0 ? static_cast<uint32_t>(M) : m;
    const LutShape sh = LutShape::of(mm);
    const uint32_t base = lut_saddr() + lofs;
    const uint32_t hbase = base + sh.nfull * kFullBytes, hrow = sh.half_row_bytes();
    float acc = 0.0f;
    for (uint32_t j = 0; j < mm; ++j) {
        const uint32_t c = __ldg(code + j);
        const uint32_t b = j >> 5, t = j & 31u;
        const uint32_t a = b < sh.nfull ? base + b * kFullBytes + c * 128u + 4u * t : hbase + c * hrow + 4u * t;
        acc = __fadd_rn(acc, lds_f32(a));
    }
    return acc;
}

} // namespace trimgpu
