// trim_b200/graph.hpp — C++ façade over the graph filter of the C ABI
// (include/trim_gpu.h, trim_graph_*) with the reference's graph-search
// signatures and exceptions (proj/include/trimsearch/graph/search.hpp):
//
//   reference                                              here
//   graph::search_trim_knn(g, ds, lm, prof, q, k, ef)       trim_b200::graph::search_trim_knn(gg, prof, q, k, ef)
//   graph::search_trim_range(g, ds, lm, prof, q, r, ef)     trim_b200::graph::search_trim_range(gg, prof, q, r, ef)
//   graph::SearchResult {ids, dist_sq, counters}           trim_b200::graph::SearchResult
//
// from_reference() reads GraphIndex (graph/hnsw.hpp:22-35: count, entry,
// max_level, layers), LandmarkStore (trim/landmarks.hpp:18-28: codebook,
// codes, lx_dist) and VectorDataset (core/dataset.hpp:18-27) by member name.
#pragma once

#include "ivf.hpp"

namespace trim_b200 {
namespace graph {

// graph::SearchResult (graph/search.hpp:22-26)
struct SearchResult {
    std::vector<std::uint32_t> ids;
    std::vector<float> dist_sq;
    SearchCounters counters;
};

// RAII owner of a device-resident graph + landmark store (trim_graph_create).
class GpuGraph {
  public:
    explicit GpuGraph(const trim_graph_desc& d) : dim_(d.dim) { check(trim_graph_create(&d, &h_)); }
    GpuGraph(const GpuGraph&) = delete;
    GpuGraph& operator=(const GpuGraph&) = delete;
    GpuGraph(GpuGraph&& o) noexcept : h_(o.h_), dim_(o.dim_) { o.h_ = nullptr; }
    ~GpuGraph() {
        if (h_)
            trim_graph_destroy(h_);
    }
    trim_graph_t handle() const { return h_; }
    std::uint32_t dim() const { return dim_; }

  private:
    trim_graph_t h_ = nullptr;
    std::uint32_t dim_ = 0;
};

// search.hpp:198-199: the landmark store must cover the dataset.
template <class RefGraph, class RefLandmarks, class RefDataset>
GpuGraph from_reference(const RefGraph& g, const RefLandmarks& lm, const RefDataset& ds, int device = 0) {
    if (lm.count != ds.count || g.count != ds.count)
        throw std::invalid_argument("search_trim_knn: landmark store size mismatch");
    const std::uint32_t m = static_cast<std::uint32_t>(lm.codebook.params.m);
    std::vector<std::uint32_t> sub(m);
    std::vector<float> cent;
    for (std::uint32_t j = 0; j < m; ++j) {
        sub[j] = static_cast<std::uint32_t>(lm.codebook.sub_dims[j]);
        cent.insert(cent.end(), lm.codebook.centroids[j].begin(), lm.codebook.centroids[j].end());
    }
    const std::size_t n = g.count, levels = g.max_level + 1;
    std::vector<std::uint64_t> offs, base;
    std::vector<std::uint32_t> nbrs;
    for (std::size_t l = 0; l < levels; ++l) {
        base.push_back(nbrs.size());
        std::uint64_t off = 0;
        for (std::size_t i = 0; i < n; ++i) {
            offs.push_back(off);
            const auto& a = g.layers[l][i];
            nbrs.insert(nbrs.end(), a.begin(), a.end());
            off += a.size();
        }
        offs.push_back(off);
    }
    trim_graph_desc d{};
    d.n = n;
    d.dim = static_cast<std::uint32_t>(ds.dim);
    d.m = m;
    d.ksub = static_cast<std::uint32_t>(lm.codebook.params.c);
    d.sub_dims = sub.data();
    d.centroids = cent.data();
    d.codes = lm.codes.data();
    d.code_stride = m;
    d.lx = lm.lx_dist.data();
    d.vectors = ds.data.data();
    d.levels = static_cast<std::uint32_t>(levels);
    d.entry = g.entry;
    d.offsets = offs.data();
    d.nbr_base = base.data();
    d.nbrs = nbrs.data();
    d.total_nbrs = nbrs.size();
    d.device = device;
    d.memory = TRIM_MEM_HOST;
    return GpuGraph(d);
}

// The production path: one launch per batch (queries nq x dim).
template <class Profile>
ivf::BatchResult search_trim_knn_batch(const GpuGraph& g, const Profile& prof, const float* queries, std::size_t nq,
                                       std::size_t k, std::size_t ef) {
    ivf::BatchResult r;
    r.ids.resize(nq * k);
    r.dist_sq.resize(nq * k);
    r.counters.resize(nq);
    check(trim_graph_search_knn(g.handle(), queries, nq, static_cast<std::uint32_t>(k),
                                static_cast<std::uint32_t>(ef), gamma_of(prof), r.ids.data(), r.dist_sq.data(),
                                r.counters.data()));
    return r;
}

template <class Profile>
ivf::BatchResult search_trim_range_batch(const GpuGraph& g, const Profile& prof, const float* queries,
                                         std::size_t nq, const float* radius, std::size_t ef) {
    ivf::BatchResult r;
    r.offsets.resize(nq + 1);
    r.counters.resize(nq);
    std::uint32_t* ids = nullptr;
    float* dist = nullptr;
    check(trim_graph_search_range(g.handle(), queries, nq, radius, static_cast<std::uint32_t>(ef), gamma_of(prof),
                                  r.offsets.data(), &ids, &dist, r.counters.data()));
    const std::size_t tot = r.offsets[nq];
    r.ids.assign(ids, ids + tot);
    r.dist_sq.assign(dist, dist + tot);
    trim_free(ids);
    trim_free(dist);
    return r;
}

namespace detail {
inline SearchResult one(const ivf::BatchResult& b, std::size_t begin, std::size_t end) {
    SearchResult r;
    for (std::size_t i = begin; i < end; ++i) {
        if (b.ids[i] == 0xFFFFFFFFu) // fewer than k results: padding
            break;
        r.ids.push_back(b.ids[i]);
        r.dist_sq.push_back(b.dist_sq[i]);
    }
    const trim_counters& c = b.counters[0];
    r.counters.dc = c.dc;
    r.counters.edc = c.edc;
    r.counters.pruned = c.pruned;
    r.counters.evaluated = c.evaluated;
    r.counters.hops = c.hops;
    return r;
}
} // namespace detail

// graph::search_trim_knn (graph/search.hpp:188-264)
template <class Profile, class View>
SearchResult search_trim_knn(const GpuGraph& g, const Profile& prof, const View& q, std::size_t k, std::size_t ef) {
    const auto b = search_trim_knn_batch(g, prof, ivf::detail::data_of(q, g.dim()), 1, k, ef);
    return detail::one(b, 0, k);
}

// graph::search_trim_range (graph/search.hpp:267-347)
template <class Profile, class View>
SearchResult search_trim_range(const GpuGraph& g, const Profile& prof, const View& q, float radius, std::size_t ef) {
    const auto b = search_trim_range_batch(g, prof, ivf::detail::data_of(q, g.dim()), 1, &radius, ef);
    return detail::one(b, 0, b.offsets[1]);
}

} // namespace graph
} // namespace trim_b200
