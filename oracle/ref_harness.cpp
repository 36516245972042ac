// ref_harness.cpp — TEST INFRASTRUCTURE ONLY.
//
// A C-callable shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/trimsearch, included in place by
// oracle/Makefile with -I; no reference source is copied into this repo).
// Built into oracle/_ref/libtrimref.so (git-ignored, travels to the GPU box).
// It is used to (1) generate the golden fixtures in tests/golden/, (2) pin the
// C restatement in oracle/trim_oracle.c, and (3) time the reference CPU path
// for bench.py --impl reference. Compiled -O3 with no -march flag, exactly like
// the reference's Release build (proj/CMakeLists.txt:6-8), so no FMA.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "trimsearch/bench/metrics.hpp"
#include "trimsearch/bench/radius.hpp"
#include "trimsearch/core/distance.hpp"
#include "trimsearch/core/ground_truth.hpp"
#include "trimsearch/core/parallel.hpp"
#include "trimsearch/core/synthetic.hpp"
#include "trimsearch/core/vecs_io.hpp"
#include "trimsearch/graph/hnsw.hpp"
#include "trimsearch/graph/search.hpp"
#include "trimsearch/ivf/ivf.hpp"
#include "trimsearch/pq/pq.hpp"
#include "trimsearch/trim/calibration.hpp"
#include "trimsearch/trim/landmarks.hpp"
#include "trimsearch/trim/lower_bound.hpp"

using namespace trimsearch;

namespace {

thread_local std::string g_err;

enum { REF_OK = 0, REF_EINVAL = 1, REF_EDATA = 2, REF_EOTHER = 3 };

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return REF_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return REF_EINVAL;
    } catch (const DataError& e) {
        g_err = e.what();
        return REF_EDATA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return REF_EOTHER;
    }
}

VectorDataset make_ds(const float* data, std::uint64_t n, std::uint32_t dim) {
    VectorDataset ds(dim, n);
    std::memcpy(ds.data.data(), data, sizeof(float) * n * dim);
    return ds;
}

pq::PqCodebook make_cb(std::uint32_t dim, std::uint32_t m, std::uint32_t c,
                       const std::uint32_t* sub_dims, const float* centroids) {
    pq::PqCodebook cb;
    cb.params.m = m;
    cb.params.c = c;
    cb.dim = dim;
    cb.sub_dims.assign(sub_dims, sub_dims + m);
    cb.sub_offsets.resize(m);
    std::size_t off = 0;
    for (std::uint32_t j = 0; j < m; ++j) {
        cb.sub_offsets[j] = off;
        off += cb.sub_dims[j];
    }
    cb.centroids.resize(m);
    for (std::uint32_t j = 0; j < m; ++j) {
        const float* src = centroids + static_cast<std::size_t>(c) * cb.sub_offsets[j];
        cb.centroids[j].assign(src, src + static_cast<std::size_t>(c) * cb.sub_dims[j]);
    }
    return cb;
}

// Flat CSR view of an IVF index (same layout as oracle/trim_oracle.h).
struct FlatIndex {
    std::uint32_t dim, m, c;
    const std::uint32_t* sub_dims;
    const float* centroids;
    std::uint32_t nlist;
    const float* coarse;
    const std::uint64_t* list_offsets;
    const std::uint32_t* list_ids;
    const std::uint8_t* list_codes;
    std::uint32_t code_stride;
    const float* list_lx;
    std::uint64_t n;
    const float* vectors;
};

ivf::IvfIndex make_ivf(const FlatIndex& f) {
    ivf::IvfIndex ix;
    ix.dim = f.dim;
    ix.nlist = f.nlist;
    ix.codebook = make_cb(f.dim, f.m, f.c, f.sub_dims, f.centroids);
    ix.coarse_centroids.assign(f.coarse, f.coarse + static_cast<std::size_t>(f.nlist) * f.dim);
    ix.lists.resize(f.nlist);
    for (std::uint32_t l = 0; l < f.nlist; ++l) {
        auto& L = ix.lists[l];
        for (std::uint64_t e = f.list_offsets[l]; e < f.list_offsets[l + 1]; ++e) {
            L.ids.push_back(f.list_ids[e]);
            L.codes.insert(L.codes.end(), f.list_codes + e * f.code_stride,
                           f.list_codes + e * f.code_stride + f.m);
            L.lx_dist.push_back(f.list_lx[e]);
        }
    }
    return ix;
}

void put_counters(std::uint64_t* out, const SearchCounters& c, std::uint64_t coarse_dc) {
    out[0] = c.dc;
    out[1] = c.edc;
    out[2] = c.pruned;
    out[3] = c.evaluated;
    out[4] = c.hops;
    out[5] = coarse_dc;
}

// Flat CSR view of an HNSW GraphIndex (graph/hnsw.hpp:22-35): level l's
// adjacency is offsets[l*(n+1) + i .. + i+1) into nbrs + nbr_base[l].
struct FlatGraph {
    std::uint64_t n;
    std::uint32_t M, levels, entry, efc;
    const std::uint64_t* offsets;
    const std::uint64_t* nbr_base;
    const std::uint32_t* nbrs;
};

graph::GraphIndex make_graph(const FlatGraph& f) {
    graph::GraphIndex g;
    g.count = f.n;
    g.M = f.M;
    g.ef_construction = f.efc;
    g.entry = f.entry;
    g.max_level = f.levels - 1;
    g.layers.resize(f.levels);
    for (std::uint32_t l = 0; l < f.levels; ++l) {
        const std::uint64_t* o = f.offsets + static_cast<std::size_t>(l) * (f.n + 1);
        const std::uint32_t* nb = f.nbrs + f.nbr_base[l];
        g.layers[l].resize(f.n);
        for (std::uint64_t i = 0; i < f.n; ++i)
            g.layers[l][i].assign(nb + o[i], nb + o[i + 1]);
    }
    return g;
}

// LandmarkStore (trim/landmarks.hpp:18-28) from flat arrays: codes n*m, lx n.
trim::LandmarkStore make_lm(std::uint32_t dim, std::uint32_t m, std::uint32_t c,
                            const std::uint32_t* sub_dims, const float* centroids,
                            const std::uint8_t* codes, const float* lx, std::uint64_t n) {
    trim::LandmarkStore lm;
    lm.codebook = make_cb(dim, m, c, sub_dims, centroids);
    lm.count = n;
    lm.codes.assign(codes, codes + n * m);
    lm.lx_dist.assign(lx, lx + n);
    return lm;
}

struct GraphSession {
    graph::GraphIndex g;
    trim::LandmarkStore lm;
    VectorDataset ds;
};

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(unsigned t) { thread_cap().store(t); }

// core/synthetic.hpp:11-18
int ref_make_normal(std::uint64_t n, std::uint32_t dim, std::uint64_t seed, float* out) {
    return guarded([&] {
        const auto ds = make_normal_dataset(n, dim, seed);
        std::memcpy(out, ds.data.data(), sizeof(float) * ds.data.size());
    });
}

// core/synthetic.hpp:21-33
int ref_make_blobs(const float* centers, std::uint64_t nc, std::uint32_t dim, std::uint64_t n,
                   float sigma, std::uint64_t seed, float* out) {
    return guarded([&] {
        const auto cs = make_ds(centers, nc, dim);
        const auto ds = make_blob_dataset(cs, n, sigma, seed);
        std::memcpy(out, ds.data.data(), sizeof(float) * ds.data.size());
    });
}

// uniform [0,1) rows as in proj/tests/test_graph.cpp:19-26, then
// VectorDataset::normalize_rows (core/dataset.hpp:44-56) when `normalize`.
int ref_make_uniform(std::uint64_t n, std::uint32_t dim, std::uint64_t seed, int normalize,
                     float* out) {
    return guarded([&] {
        VectorDataset ds(dim, n);
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<float> u(0.0f, 1.0f);
        for (auto& v : ds.data)
            v = u(rng);
        if (normalize)
            ds.normalize_rows();
        std::memcpy(out, ds.data.data(), sizeof(float) * ds.data.size());
    });
}

// pq/pq.hpp:65-113. centroids_out: sum_j c*sub_dims[j] floats.
int ref_pq_train(const float* data, std::uint64_t n, std::uint32_t dim, std::uint32_t m,
                 std::uint32_t c, std::uint32_t iters, std::uint64_t seed,
                 std::uint64_t train_sample, std::uint32_t* sub_dims_out, float* centroids_out,
                 double* mse_out) {
    return guarded([&] {
        const auto ds = make_ds(data, n, dim);
        pq::PqParams p;
        p.m = m;
        p.c = c;
        p.kmeans_iters = iters;
        p.seed = seed;
        p.train_sample = train_sample;
        const auto cb = pq::train(ds, p);
        std::size_t off = 0;
        for (std::uint32_t j = 0; j < m; ++j) {
            sub_dims_out[j] = static_cast<std::uint32_t>(cb.sub_dims[j]);
            std::memcpy(centroids_out + off, cb.centroids[j].data(),
                        sizeof(float) * cb.centroids[j].size());
            off += cb.centroids[j].size();
        }
        if (mse_out)
            *mse_out = cb.training_mse;
    });
}

// trim/landmarks.hpp:57-72. codes_out: n*code_stride bytes (only the first m
// bytes of each row are written).
int ref_build_landmarks(const float* data, std::uint64_t n, std::uint32_t dim, std::uint32_t m,
                        std::uint32_t c, const std::uint32_t* sub_dims, const float* centroids,
                        std::uint8_t* codes_out, std::uint32_t code_stride, float* lx_out) {
    return guarded([&] {
        const auto ds = make_ds(data, n, dim);
        const auto lm = trim::build_landmarks(ds, make_cb(dim, m, c, sub_dims, centroids));
        for (std::uint64_t i = 0; i < n; ++i)
            std::memcpy(codes_out + i * code_stride, lm.code(i), m);
        std::memcpy(lx_out, lm.lx_dist.data(), sizeof(float) * n);
    });
}

// ivf/ivf.hpp:112-154. Outputs: coarse nlist*dim, offsets nlist+1, ids n,
// codes n*code_stride, lx n (lists concatenated in list order).
int ref_build_ivf(const float* data, std::uint64_t n, std::uint32_t dim, std::uint32_t m,
                  std::uint32_t c, const std::uint32_t* sub_dims, const float* centroids,
                  const std::uint8_t* codes, std::uint32_t code_stride, const float* lx,
                  std::uint32_t nlist, std::uint64_t seed, std::uint32_t coarse_iters,
                  float* coarse_out, std::uint64_t* offsets_out, std::uint32_t* ids_out,
                  std::uint8_t* codes_out, float* lx_out) {
    return guarded([&] {
        const auto ds = make_ds(data, n, dim);
        trim::LandmarkStore lm;
        lm.codebook = make_cb(dim, m, c, sub_dims, centroids);
        lm.count = n;
        lm.codes.resize(n * m);
        for (std::uint64_t i = 0; i < n; ++i)
            std::memcpy(lm.codes.data() + i * m, codes + i * code_stride, m);
        lm.lx_dist.assign(lx, lx + n);
        const auto ix = ivf::build_ivf(ds, nlist, lm, seed, coarse_iters);
        std::memcpy(coarse_out, ix.coarse_centroids.data(),
                    sizeof(float) * ix.coarse_centroids.size());
        std::uint64_t off = 0;
        for (std::uint32_t l = 0; l < nlist; ++l) {
            offsets_out[l] = off;
            const auto& L = ix.lists[l];
            for (std::size_t i = 0; i < L.size(); ++i, ++off) {
                ids_out[off] = L.ids[i];
                std::memcpy(codes_out + off * code_stride, L.codes.data() + i * m, m);
                lx_out[off] = L.lx_dist[i];
            }
        }
        offsets_out[nlist] = off;
    });
}

// ivf/ivf.hpp:243-304 over a batch, via bench::detail_sweep's protocol:
// parallel_for over queries (core/parallel.hpp:31-56). counters: 6 per query
// {dc, edc, pruned, evaluated, hops, coarse_dc}.
int ref_search_knn_batch(const FlatIndex* f, const float* qs, std::uint64_t nq, std::uint32_t k,
                         std::uint32_t nprobe, double gamma, std::uint32_t* ids_out,
                         float* dist_out, std::uint64_t* counters_out) {
    return guarded([&] {
        const auto ix = make_ivf(*f);
        VectorDataset ds;
        ds.dim = f->dim;
        ds.count = f->n;
        ds.data.assign(f->vectors, f->vectors + f->n * f->dim);
        const auto prof = trim::PruningProfile::manual(gamma);
        std::vector<std::string> errs(nq);
        parallel_for(nq, [&](std::size_t qi) {
            try {
                const auto r = ivf::search_trim_ivf_knn(ix, ds, prof,
                                                        VectorView(qs + qi * f->dim, f->dim), k,
                                                        nprobe);
                for (std::size_t i = 0; i < r.ids.size(); ++i) {
                    ids_out[qi * k + i] = r.ids[i];
                    dist_out[qi * k + i] = r.dist_sq[i];
                }
                put_counters(counters_out + qi * 6, r.counters, r.coarse_dc);
            } catch (const std::exception& e) {
                errs[qi] = e.what();
            }
        });
        for (const auto& e : errs)
            if (!e.empty())
                throw std::invalid_argument(e);
    });
}

// ivf/ivf.hpp:308-347. Results per query are written at ids_out + qi*cap;
// counts_out[qi] is the true count (may exceed cap: then truncated).
int ref_search_range_batch(const FlatIndex* f, const float* qs, std::uint64_t nq,
                           const float* radius, std::uint32_t nprobe, double gamma,
                           std::uint64_t cap, std::uint32_t* ids_out, float* dist_out,
                           std::uint64_t* counts_out, std::uint64_t* counters_out) {
    return guarded([&] {
        const auto ix = make_ivf(*f);
        VectorDataset ds;
        ds.dim = f->dim;
        ds.count = f->n;
        ds.data.assign(f->vectors, f->vectors + f->n * f->dim);
        const auto prof = trim::PruningProfile::manual(gamma);
        std::vector<std::string> errs(nq);
        parallel_for(nq, [&](std::size_t qi) {
            try {
                const auto r = ivf::search_trim_ivf_range(
                    ix, ds, prof, VectorView(qs + qi * f->dim, f->dim), radius[qi], nprobe);
                counts_out[qi] = r.ids.size();
                for (std::size_t i = 0; i < r.ids.size() && i < cap; ++i) {
                    ids_out[qi * cap + i] = r.ids[i];
                    dist_out[qi * cap + i] = r.dist_sq[i];
                }
                put_counters(counters_out + qi * 6, r.counters, r.coarse_dc);
            } catch (const std::exception& e) {
                errs[qi] = e.what();
            }
        });
        for (const auto& e : errs)
            if (!e.empty())
                throw std::invalid_argument(e);
    });
}

// ivf/ivf.hpp:193-237
int ref_search_baseline_batch(const FlatIndex* f, const float* qs, std::uint64_t nq,
                              std::uint32_t k, std::uint32_t nprobe, std::uint32_t k_prime,
                              std::uint32_t* ids_out, float* dist_out,
                              std::uint64_t* counters_out) {
    return guarded([&] {
        const auto ix = make_ivf(*f);
        VectorDataset ds;
        ds.dim = f->dim;
        ds.count = f->n;
        ds.data.assign(f->vectors, f->vectors + f->n * f->dim);
        std::vector<std::string> errs(nq);
        parallel_for(nq, [&](std::size_t qi) {
            try {
                const auto r = ivf::search_baseline_ivfpq(
                    ix, ds, VectorView(qs + qi * f->dim, f->dim), k, nprobe, k_prime);
                for (std::size_t i = 0; i < r.ids.size(); ++i) {
                    ids_out[qi * k + i] = r.ids[i];
                    dist_out[qi * k + i] = r.dist_sq[i];
                }
                put_counters(counters_out + qi * 6, r.counters, r.coarse_dc);
            } catch (const std::exception& e) {
                errs[qi] = e.what();
            }
        });
        for (const auto& e : errs)
            if (!e.empty())
                throw std::invalid_argument(e);
    });
}

// Prebuilt-index variant for timing: build the reference IvfIndex once, then
// time only the query batch exactly like bench::detail_sweep::run_queries
// (sweep.hpp:121-152, steady_clock around parallel_for).
struct RefSession {
    ivf::IvfIndex ix;
    VectorDataset ds;
};

void* ref_session_create(const FlatIndex* f) {
    RefSession* s = nullptr;
    const int rc = guarded([&] {
        s = new RefSession;
        s->ix = make_ivf(*f);
        s->ds.dim = f->dim;
        s->ds.count = f->n;
        s->ds.data.assign(f->vectors, f->vectors + f->n * f->dim);
    });
    return rc == REF_OK ? s : nullptr;
}

void ref_session_destroy(void* p) { delete static_cast<RefSession*>(p); }

// kind: 0 = trim knn, 1 = trim range (arg = radius), 2 = baseline (arg = k_prime)
int ref_session_run(void* p, int kind, const float* qs, std::uint64_t nq, std::uint32_t k,
                    std::uint32_t nprobe, double gamma, double arg, double* seconds_out,
                    std::uint64_t* counters_sum_out) {
    auto* s = static_cast<RefSession*>(p);
    return guarded([&] {
        const auto prof = trim::PruningProfile::manual(gamma);
        std::vector<SearchCounters> cs(nq);
        const auto t0 = std::chrono::steady_clock::now();
        parallel_for(nq, [&](std::size_t qi) {
            const VectorView q(qs + qi * s->ds.dim, s->ds.dim);
            ivf::IvfResult r;
            if (kind == 0)
                r = ivf::search_trim_ivf_knn(s->ix, s->ds, prof, q, k, nprobe);
            else if (kind == 1)
                r = ivf::search_trim_ivf_range(s->ix, s->ds, prof, q, static_cast<float>(arg),
                                               nprobe);
            else
                r = ivf::search_baseline_ivfpq(s->ix, s->ds, q, k, nprobe,
                                               static_cast<std::size_t>(arg));
            cs[qi] = r.counters;
        });
        *seconds_out =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        SearchCounters tot;
        for (const auto& c : cs)
            tot += c;
        put_counters(counters_sum_out, tot, 0);
    });
}

// Per-query results over a session's index (no per-call copy of a 10M-row
// index): ivf::search_trim_ivf_knn (ivf.hpp:243-304) for every query of the
// batch, parallel_for over queries. ids/dist nq*k; counters 6 per query.
int ref_session_knn(void* p, const float* qs, std::uint64_t nq, std::uint32_t k, std::uint32_t nprobe,
                    double gamma, std::uint32_t* ids_out, float* dist_out, std::uint64_t* counters_out) {
    auto* s = static_cast<RefSession*>(p);
    return guarded([&] {
        const auto prof = trim::PruningProfile::manual(gamma);
        std::vector<std::string> errs(nq);
        parallel_for(nq, [&](std::size_t qi) {
            try {
                const auto r = ivf::search_trim_ivf_knn(s->ix, s->ds, prof,
                                                        VectorView(qs + qi * s->ds.dim, s->ds.dim), k, nprobe);
                for (std::size_t i = 0; i < r.ids.size(); ++i) {
                    ids_out[qi * k + i] = r.ids[i];
                    dist_out[qi * k + i] = r.dist_sq[i];
                }
                put_counters(counters_out + qi * 6, r.counters, r.coarse_dc);
            } catch (const std::exception& e) {
                errs[qi] = e.what();
            }
        });
        for (const auto& e : errs)
            if (!e.empty())
                throw std::invalid_argument(e);
    });
}

// ivf::search_trim_ivf_range (ivf.hpp:308-347) over a session's index: query
// qi's members at ids/dist + qi*cap (truncated to cap), counts_out[qi] = the
// true count.
int ref_session_range(void* p, const float* qs, std::uint64_t nq, const float* radius, std::uint32_t nprobe,
                      double gamma, std::uint64_t cap, std::uint32_t* ids_out, float* dist_out,
                      std::uint64_t* counts_out, std::uint64_t* counters_out) {
    auto* s = static_cast<RefSession*>(p);
    return guarded([&] {
        const auto prof = trim::PruningProfile::manual(gamma);
        std::vector<std::string> errs(nq);
        parallel_for(nq, [&](std::size_t qi) {
            try {
                const auto r = ivf::search_trim_ivf_range(s->ix, s->ds, prof,
                                                          VectorView(qs + qi * s->ds.dim, s->ds.dim), radius[qi],
                                                          nprobe);
                counts_out[qi] = r.ids.size();
                for (std::size_t i = 0; i < r.ids.size() && i < cap; ++i) {
                    ids_out[qi * cap + i] = r.ids[i];
                    dist_out[qi * cap + i] = r.dist_sq[i];
                }
                put_counters(counters_out + qi * 6, r.counters, r.coarse_dc);
            } catch (const std::exception& e) {
                errs[qi] = e.what();
            }
        });
        for (const auto& e : errs)
            if (!e.empty())
                throw std::invalid_argument(e);
    });
}

// ---- on-disk formats (test infrastructure: pins paper_2508_17828_b200/formats.py)
// IvfIndex::save (ivf.hpp:53-76), with the codebook's bookkeeping fields set.
int ref_ivf_save(const FlatIndex* f, double training_mse, std::uint64_t seed, std::uint32_t iters,
                 const char* path) {
    return guarded([&] {
        auto ix = make_ivf(*f);
        ix.codebook.training_mse = training_mse;
        ix.codebook.params.seed = seed;
        ix.codebook.params.kmeans_iters = iters;
        ix.save(path);
    });
}

// IvfIndex::load (ivf.hpp:78-107): sizes, then the arrays (concatenated lists).
int ref_ivf_load_sizes(const char* path, std::uint64_t* dim, std::uint64_t* nlist, std::uint32_t* m,
                       std::uint32_t* c, std::uint64_t* total) {
    return guarded([&] {
        const auto ix = ivf::IvfIndex::load(path);
        *dim = ix.dim;
        *nlist = ix.nlist;
        *m = static_cast<std::uint32_t>(ix.codebook.m());
        *c = static_cast<std::uint32_t>(ix.codebook.c());
        std::uint64_t t = 0;
        for (const auto& l : ix.lists)
            t += l.size();
        *total = t;
    });
}

int ref_ivf_load(const char* path, std::uint32_t* sub_dims, float* centroids, float* coarse,
                 std::uint64_t* offsets, std::uint32_t* ids, std::uint8_t* codes, float* lx,
                 double* training_mse, std::uint64_t* seed, std::uint32_t* iters) {
    return guarded([&] {
        const auto ix = ivf::IvfIndex::load(path);
        const auto& cb = ix.codebook;
        std::size_t co = 0;
        for (std::size_t j = 0; j < cb.m(); ++j) {
            sub_dims[j] = static_cast<std::uint32_t>(cb.sub_dims[j]);
            std::memcpy(centroids + co, cb.centroids[j].data(), sizeof(float) * cb.centroids[j].size());
            co += cb.centroids[j].size();
        }
        std::memcpy(coarse, ix.coarse_centroids.data(), sizeof(float) * ix.coarse_centroids.size());
        std::uint64_t e = 0;
        offsets[0] = 0;
        for (std::size_t l = 0; l < ix.lists.size(); ++l) {
            const auto& L = ix.lists[l];
            for (std::size_t i = 0; i < L.size(); ++i, ++e) {
                ids[e] = L.ids[i];
                std::memcpy(codes + e * cb.m(), L.codes.data() + i * cb.m(), cb.m());
                lx[e] = L.lx_dist[i];
            }
            offsets[l + 1] = e;
        }
        *training_mse = cb.training_mse;
        *seed = cb.params.seed;
        *iters = static_cast<std::uint32_t>(cb.params.kmeans_iters);
    });
}

// LandmarkStore::save / load (trim/landmarks.hpp:29-53).
int ref_landmarks_save(std::uint32_t dim, std::uint32_t m, std::uint32_t c, const std::uint32_t* sub_dims,
                       const float* centroids, std::uint64_t n, const std::uint8_t* codes, const float* lx,
                       const char* path) {
    return guarded([&] {
        trim::LandmarkStore lm;
        lm.codebook = make_cb(dim, m, c, sub_dims, centroids);
        lm.count = n;
        lm.codes.assign(codes, codes + n * m);
        lm.lx_dist.assign(lx, lx + n);
        lm.save(path);
    });
}

int ref_landmarks_load(const char* path, std::uint64_t n_expected, std::uint8_t* codes, float* lx) {
    return guarded([&] {
        const auto lm = trim::LandmarkStore::load(path);
        if (lm.count != n_expected)
            throw DataError("landmark count mismatch");
        std::memcpy(codes, lm.codes.data(), lm.codes.size());
        std::memcpy(lx, lm.lx_dist.data(), sizeof(float) * lm.count);
    });
}

// trim::PruningProfile::save / load (trim/calibration.hpp:234-288).
int ref_profile_save(double p, double gamma, const char* path) {
    return guarded([&] {
        auto prof = trim::PruningProfile::manual(gamma);
        prof.p = p;
        prof.save(path);
    });
}

int ref_profile_load(const char* path, double* p, double* gamma) {
    return guarded([&] {
        const auto prof = trim::PruningProfile::load(path);
        *p = prof.p;
        *gamma = prof.gamma;
    });
}

// core/vecs_io.hpp: write_fvecs / load_vecs.
int ref_write_fvecs(const float* data, std::uint64_t n, std::uint32_t dim, const char* path) {
    return guarded([&] { write_fvecs(path, make_ds(data, n, dim)); });
}

int ref_load_fvecs(const char* path, std::uint64_t n_expected, std::uint32_t dim, float* out) {
    return guarded([&] {
        const auto ds = load_vecs(path, ElementKind::Float32);
        if (ds.count != n_expected || ds.dim != dim)
            throw DataError("fvecs shape mismatch");
        std::memcpy(out, ds.data.data(), sizeof(float) * n_expected * dim);
    });
}

// core/ground_truth.hpp:97-113
int ref_ground_truth_knn(const float* data, std::uint64_t n, std::uint32_t dim, const float* qs,
                         std::uint64_t nq, std::uint32_t k, std::uint32_t* ids_out,
                         float* dist_out) {
    return guarded([&] {
        const auto ds = make_ds(data, n, dim);
        const auto q = make_ds(qs, nq, dim);
        const auto gt = ground_truth_knn(ds, q, k);
        for (std::uint64_t i = 0; i < nq; ++i)
            for (std::uint32_t j = 0; j < k; ++j) {
                ids_out[i * k + j] = gt.ids[i][j];
                dist_out[i * k + j] = gt.dist_sq[i][j];
            }
    });
}

// bench/radius.hpp:19-55
int ref_pick_radius(const float* data, std::uint64_t n, std::uint32_t dim, const float* qs,
                    std::uint64_t nq, double e_fraction, std::uint64_t sample_rows,
                    std::uint64_t sample_queries, std::uint64_t seed, float* radius_out) {
    return guarded([&] {
        const auto ds = make_ds(data, n, dim);
        const auto q = make_ds(qs, nq, dim);
        *radius_out =
            bench::pick_radius_for_fraction(ds, q, e_fraction, sample_rows, sample_queries, seed);
    });
}

// trim/calibration.hpp:101-168 + :294-308 (empirical strategy)
int ref_calibrate_empirical(const float* data, std::uint64_t n, std::uint32_t dim,
                            std::uint32_t m, std::uint32_t c, const std::uint32_t* sub_dims,
                            const float* centroids, const std::uint8_t* codes,
                            std::uint32_t code_stride, const float* lx, const float* cal_qs,
                            std::uint64_t ncal, std::uint64_t sample_x,
                            std::uint64_t queries_per_x, std::uint64_t seed, double p,
                            double* gamma_out) {
    return guarded([&] {
        const auto ds = make_ds(data, n, dim);
        trim::LandmarkStore lm;
        lm.codebook = make_cb(dim, m, c, sub_dims, centroids);
        lm.count = n;
        lm.codes.resize(n * m);
        for (std::uint64_t i = 0; i < n; ++i)
            std::memcpy(lm.codes.data() + i * m, codes + i * code_stride, m);
        lm.lx_dist.assign(lx, lx + n);
        const auto q = make_ds(cal_qs, ncal, dim);
        trim::EmpiricalSampleParams ep;
        ep.sample_x = sample_x;
        ep.queries_per_x = queries_per_x;
        ep.seed = seed;
        *gamma_out =
            trim::calibrate_gamma(trim::sample_one_minus_z_empirical(ds, lm, q, ep), p).gamma;
    });
}

// ---- HNSW graph (graph/hnsw.hpp:165-268) and the TRIM graph searches
// (graph/search.hpp:188-347): test infrastructure for the graph filter path.
void* ref_graph_build(const float* data, std::uint64_t n, std::uint32_t dim, std::uint32_t M,
                      std::uint32_t efc, std::uint64_t seed) {
    auto* s = new GraphSession;
    const int rc = guarded([&] { s->g = graph::build_graph(make_ds(data, n, dim), M, efc, seed); });
    if (rc != REF_OK) {
        delete s;
        return nullptr;
    }
    return s;
}
void ref_graph_free(void* p) { delete static_cast<GraphSession*>(p); }
// levels, entry, and per level the total adjacency size (sizes_out: levels).
int ref_graph_info(void* p, std::uint32_t* levels, std::uint32_t* entry, std::uint64_t* sizes_out) {
    auto* s = static_cast<GraphSession*>(p);
    *levels = static_cast<std::uint32_t>(s->g.max_level + 1);
    *entry = s->g.entry;
    if (sizes_out)
        for (std::size_t l = 0; l <= s->g.max_level; ++l) {
            std::uint64_t t = 0;
            for (const auto& a : s->g.layers[l])
                t += a.size();
            sizes_out[l] = t;
        }
    return REF_OK;
}
int ref_graph_export(void* p, std::uint32_t level, std::uint64_t* offsets_out, std::uint32_t* nbrs_out) {
    auto* s = static_cast<GraphSession*>(p);
    std::uint64_t off = 0;
    for (std::size_t i = 0; i < s->g.count; ++i) {
        offsets_out[i] = off;
        for (std::uint32_t v : s->g.layers[level][i])
            nbrs_out[off++] = v;
    }
    offsets_out[s->g.count] = off;
    return REF_OK;
}
void* ref_graph_load(const char* path) {
    auto* s = new GraphSession;
    const int rc = guarded([&] { s->g = graph::GraphIndex::load(path); });
    if (rc != REF_OK) {
        delete s;
        return nullptr;
    }
    return s;
}
int ref_graph_save(const FlatGraph* f, const char* path) {
    return guarded([&] { make_graph(*f).save(path); });
}

// graph::search_trim_knn (kind 0, k results) / search_trim_range (kind 1,
// arg = radius; results at ids_out + qi*cap, counts_out[qi] = true count) /
// search_baseline_knn (kind 2) over a batch, parallel_for over queries.
int ref_graph_search_batch(const FlatGraph* fg, std::uint32_t dim, std::uint32_t m, std::uint32_t c,
                           const std::uint32_t* sub_dims, const float* centroids,
                           const std::uint8_t* codes, const float* lx, const float* data,
                           const float* qs, std::uint64_t nq, int kind, std::uint32_t k,
                           std::uint32_t ef, double gamma, double arg, std::uint64_t cap,
                           std::uint32_t* ids_out, float* dist_out, std::uint64_t* counts_out,
                           std::uint64_t* counters_out) {
    return guarded([&] {
        const auto g = make_graph(*fg);
        const auto lm = make_lm(dim, m, c, sub_dims, centroids, codes, lx, fg->n);
        const auto ds = make_ds(data, fg->n, dim);
        std::vector<std::string> errs(nq);
        parallel_for(nq, [&](std::size_t qi) {
            try {
                const VectorView q(qs + qi * dim, dim);
                graph::SearchResult r;
                if (kind == 0)
                    r = graph::search_trim_knn(g, ds, lm, trim::PruningProfile::manual(gamma), q, k, ef);
                else if (kind == 1)
                    r = graph::search_trim_range(g, ds, lm, trim::PruningProfile::manual(gamma), q,
                                                 static_cast<float>(arg), ef);
                else
                    r = graph::search_baseline_knn(g, ds, q, k, ef);
                const std::size_t w = kind == 1 ? cap : k;
                for (std::size_t i = 0; i < r.ids.size() && i < w; ++i) {
                    ids_out[qi * w + i] = r.ids[i];
                    dist_out[qi * w + i] = r.dist_sq[i];
                }
                counts_out[qi] = r.ids.size();
                put_counters(counters_out + qi * 6, r.counters, 0);
            } catch (const std::exception& e) {
                errs[qi] = e.what();
            }
        });
        for (const auto& e : errs)
            if (!e.empty())
                throw std::invalid_argument(e);
    });
}

// A resident graph + landmarks + dataset for timing the reference's graph
// searches like bench::detail_sweep::run_queries (sweep.hpp:121-152).
void* ref_graph_session_create(const FlatGraph* fg, std::uint32_t dim, std::uint32_t m, std::uint32_t c,
                               const std::uint32_t* sub_dims, const float* centroids, const std::uint8_t* codes,
                               const float* lx, const float* data) {
    auto* s = new GraphSession;
    const int rc = guarded([&] {
        s->g = make_graph(*fg);
        s->lm = make_lm(dim, m, c, sub_dims, centroids, codes, lx, fg->n);
        s->ds = make_ds(data, fg->n, dim);
    });
    if (rc != REF_OK) {
        delete s;
        return nullptr;
    }
    return s;
}
// kind 0: search_trim_knn (k, ef), 1: search_trim_range (arg = radius, ef).
int ref_graph_session_run(void* p, int kind, const float* qs, std::uint64_t nq, std::uint32_t k,
                          std::uint32_t ef, double gamma, double arg, double* seconds_out,
                          std::uint64_t* counters_sum_out) {
    auto* s = static_cast<GraphSession*>(p);
    return guarded([&] {
        const auto prof = trim::PruningProfile::manual(gamma);
        std::vector<SearchCounters> cs(nq);
        const auto t0 = std::chrono::steady_clock::now();
        parallel_for(nq, [&](std::size_t qi) {
            const VectorView q(qs + qi * s->ds.dim, s->ds.dim);
            cs[qi] = kind == 0 ? graph::search_trim_knn(s->g, s->ds, s->lm, prof, q, k, ef).counters
                               : graph::search_trim_range(s->g, s->ds, s->lm, prof, q, static_cast<float>(arg), ef)
                                     .counters;
        });
        *seconds_out = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        SearchCounters tot;
        for (const auto& c : cs)
            tot += c;
        put_counters(counters_sum_out, tot, 0);
    });
}

// Scalar kernels, for the known-answer tests (test_trim.cpp:18-39,
// test_core.cpp:32-44, test_pq.cpp:181-231).
float ref_euclidean_sq(const float* a, const float* b, std::uint64_t dim) {
    return euclidean_sq(a, b, dim);
}
int ref_strict_lb(float a, float b, float* out) {
    return guarded([&] { *out = trim::strict_lb(a, b); });
}
int ref_relaxed_lb(float a, float b, float g, float* out) {
    return guarded([&] { *out = trim::relaxed_lb(a, b, g); });
}
int ref_build_table(std::uint32_t dim, std::uint32_t m, std::uint32_t c,
                    const std::uint32_t* sub_dims, const float* centroids, const float* q,
                    float* table_out) {
    return guarded([&] {
        const auto cb = make_cb(dim, m, c, sub_dims, centroids);
        const auto t = pq::build_distance_table(cb, VectorView(q, dim));
        std::memcpy(table_out, t.entries.data(), sizeof(float) * t.entries.size());
    });
}
float ref_adc_lookup(const float* table, std::uint32_t m, std::uint32_t c,
                     const std::uint8_t* code) {
    pq::DistanceTable t;
    t.m = m;
    t.c = c;
    t.entries.assign(table, table + static_cast<std::size_t>(m) * c);
    return pq::adc_lookup(t, code);
}

} // extern "C"
