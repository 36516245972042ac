// trim_b200/ivf.hpp — C++ façade over the C ABI (include/trim_gpu.h) with the
// reference's query-path signatures and exceptions.
//
// A caller of the reference (proj/include/trimsearch/ivf/ivf.hpp) switches by
// building a GpuIvfIndex once from its existing IvfIndex + VectorDataset and
// calling the same-named functions:
//
//   reference                                     here
//   ivf::search_trim_ivf_knn(ix, ds, prof, q,k,np) trim_b200::ivf::search_trim_ivf_knn(g, prof, q, k, np)
//   ivf::search_trim_ivf_range(ix, ds, prof, q,r,np) trim_b200::ivf::search_trim_ivf_range(g, prof, q, r, np)
//   ivf::search_baseline_ivfpq(ix, ds, q,k,np,k')  trim_b200::ivf::search_baseline_ivfpq(g, q, k, np, k')
//   std::invalid_argument / DataError              std::invalid_argument / trim_b200::DataError
//
// from_reference() reads the reference types by their public member names
// (duck-typed templates: nothing from the reference is included here). The
// `*_batch` functions are the production path: one launch per batch.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../trim_gpu.h"

namespace trim_b200 {

// trimsearch::DataError (core/io_util.hpp:13-16)
struct DataError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
// CUDA failure or no device: there is no CPU fallback.
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int rc) {
    if (rc == TRIM_OK)
        return;
    const std::string msg = trim_last_error();
    switch (rc) {
    case TRIM_EINVAL:
        throw std::invalid_argument(msg);
    case TRIM_EDATA:
        throw DataError(msg);
    case TRIM_ENOMEM:
        throw std::bad_alloc();
    default:
        throw CudaError(msg);
    }
}

// trimsearch::SearchCounters (core/counters.hpp:10-30)
struct SearchCounters {
    std::uint64_t dc = 0, edc = 0, pruned = 0, evaluated = 0, hops = 0;
    double pruning_ratio() const {
        const std::uint64_t d = pruned + dc;
        return d == 0 ? 0.0 : static_cast<double>(pruned) / static_cast<double>(d);
    }
};

// ivf::IvfResult (ivf.hpp:164-169)
struct IvfResult {
    std::vector<std::uint32_t> ids;
    std::vector<float> dist_sq;
    SearchCounters counters;
    std::uint64_t coarse_dc = 0;
};

// trim::PruningProfile, the part the search reads (calibration.hpp:215-232)
struct PruningProfile {
    double p = -1.0;
    double gamma = -1.0;
    bool calibrated() const { return gamma >= 0.0; }
    static PruningProfile manual(double g) {
        if (g < 0.0)
            throw std::invalid_argument("PruningProfile::manual: gamma must be nonnegative");
        PruningProfile pr;
        pr.gamma = g;
        return pr;
    }
};

// Any profile type with calibrated() and gamma -> the float the kernels use
// (ivf.hpp:246-250: uncalibrated -> invalid_argument, float(profile.gamma)).
template <class Profile>
float gamma_of(const Profile& prof) {
    return prof.calibrated() ? static_cast<float>(prof.gamma) : -1.0f;
}

// RAII owner of a device-resident index (trim_index_create / _destroy).
class GpuIvfIndex {
  public:
    explicit GpuIvfIndex(const trim_index_desc& d) {
        check(trim_index_create(&d, &h_));
        dim_ = d.dim;
        nlist_ = d.nlist;
    }
    GpuIvfIndex(const GpuIvfIndex&) = delete;
    GpuIvfIndex& operator=(const GpuIvfIndex&) = delete;
    GpuIvfIndex(GpuIvfIndex&& o) noexcept : h_(o.h_), dim_(o.dim_), nlist_(o.nlist_) { o.h_ = nullptr; }
    ~GpuIvfIndex() {
        if (h_)
            trim_index_destroy(h_);
    }
    trim_index_t handle() const { return h_; }
    std::uint32_t dim() const { return dim_; }
    std::uint32_t nlist() const { return nlist_; }
    trim_index_info info() const {
        trim_index_info i{};
        check(trim_index_get_info(h_, &i));
        return i;
    }

  private:
    trim_index_t h_ = nullptr;
    std::uint32_t dim_ = 0, nlist_ = 0;
};

// Build from the reference's own IvfIndex (ivf.hpp:37-51) and VectorDataset
// (dataset.hpp:18-27): reads ix.dim, ix.nlist, ix.codebook.{params.m, params.c,
// sub_dims, centroids}, ix.coarse_centroids, ix.lists[l].{ids, codes, lx_dist},
// ds.{count, data}.
// devices + mode (TRIM_SHARD_ID / TRIM_SHARD_REPLICAS): one index over several
// GPUs of the box (include/trim_gpu.h trim_shard_mode); searches return the
// merged answer. An empty `devices` means one device, `device`.
template <class RefIvfIndex, class RefDataset>
GpuIvfIndex from_reference(const RefIvfIndex& ix, const RefDataset& ds, int device,
                           const std::vector<int>& devices, trim_shard_mode mode) {
    const std::uint32_t m = static_cast<std::uint32_t>(ix.codebook.params.m);
    const std::uint32_t c = static_cast<std::uint32_t>(ix.codebook.params.c);
    std::vector<std::uint32_t> sub(m);
    std::vector<float> cent;
    for (std::uint32_t j = 0; j < m; ++j) {
        sub[j] = static_cast<std::uint32_t>(ix.codebook.sub_dims[j]);
        cent.insert(cent.end(), ix.codebook.centroids[j].begin(), ix.codebook.centroids[j].end());
    }
    std::vector<std::uint64_t> offs(1, 0);
    std::vector<std::uint32_t> ids;
    std::vector<std::uint8_t> codes;
    std::vector<float> lx;
    for (const auto& l : ix.lists) {
        ids.insert(ids.end(), l.ids.begin(), l.ids.end());
        codes.insert(codes.end(), l.codes.begin(), l.codes.end());
        lx.insert(lx.end(), l.lx_dist.begin(), l.lx_dist.end());
        offs.push_back(ids.size());
    }
    trim_index_desc d{};
    d.dim = static_cast<std::uint32_t>(ix.dim);
    d.m = m;
    d.ksub = c;
    d.sub_dims = sub.data();
    d.centroids = cent.data();
    d.nlist = static_cast<std::uint32_t>(ix.nlist);
    d.coarse = ix.coarse_centroids.data();
    d.list_offsets = offs.data();
    d.list_ids = ids.data();
    d.list_codes = codes.data();
    d.code_stride = m;
    d.list_lx = lx.data();
    d.n = ds.count;
    d.vectors = ds.data.data();
    d.id_base = 0;
    d.device = device;
    d.memory = TRIM_MEM_HOST;
    if (!devices.empty() && mode != TRIM_SHARD_SINGLE) {
        d.devices = devices.data();
        d.ndevices = static_cast<std::uint32_t>(devices.size());
        d.shard_mode = mode;
    }
    return GpuIvfIndex(d);
}

template <class RefIvfIndex, class RefDataset>
GpuIvfIndex from_reference(const RefIvfIndex& ix, const RefDataset& ds, int device = 0) {
    return from_reference(ix, ds, device, std::vector<int>{}, TRIM_SHARD_SINGLE);
}

namespace ivf {

struct BatchResult {
    std::vector<std::uint32_t> ids; // nq*k, or concatenated (range)
    std::vector<float> dist_sq;
    std::vector<std::uint64_t> offsets; // range: nq+1
    std::vector<trim_counters> counters; // nq
};

template <class Profile>
BatchResult search_trim_ivf_knn_batch(const GpuIvfIndex& ix, const Profile& prof, const float* queries,
                                      std::size_t nq, std::size_t k, std::size_t nprobe) {
    BatchResult r;
    r.ids.resize(nq * k);
    r.dist_sq.resize(nq * k);
    r.counters.resize(nq);
    check(trim_search_knn(ix.handle(), queries, nq, static_cast<std::uint32_t>(k),
                          static_cast<std::uint32_t>(nprobe), gamma_of(prof), r.ids.data(), r.dist_sq.data(),
                          r.counters.data()));
    return r;
}

template <class Profile>
BatchResult search_trim_ivf_range_batch(const GpuIvfIndex& ix, const Profile& prof, const float* queries,
                                        std::size_t nq, const float* radius, std::size_t nprobe) {
    BatchResult r;
    r.offsets.resize(nq + 1);
    r.counters.resize(nq);
    std::uint32_t* ids = nullptr;
    float* dist = nullptr;
    check(trim_search_range(ix.handle(), queries, nq, radius, static_cast<std::uint32_t>(nprobe),
                            gamma_of(prof), r.offsets.data(), &ids, &dist, r.counters.data()));
    const std::size_t tot = r.offsets[nq];
    r.ids.assign(ids, ids + tot);
    r.dist_sq.assign(dist, dist + tot);
    trim_free(ids);
    trim_free(dist);
    return r;
}

inline BatchResult search_baseline_ivfpq_batch(const GpuIvfIndex& ix, const float* queries, std::size_t nq,
                                               std::size_t k, std::size_t nprobe, std::size_t k_prime) {
    BatchResult r;
    r.ids.resize(nq * k);
    r.dist_sq.resize(nq * k);
    r.counters.resize(nq);
    check(trim_search_baseline_ivfpq(ix.handle(), queries, nq, static_cast<std::uint32_t>(k),
                                     static_cast<std::uint32_t>(nprobe), static_cast<std::uint32_t>(k_prime),
                                     r.ids.data(), r.dist_sq.data(), r.counters.data()));
    return r;
}

namespace detail {
inline IvfResult one(const BatchResult& b, std::size_t begin, std::size_t end) {
    IvfResult r;
    r.ids.assign(b.ids.begin() + static_cast<std::ptrdiff_t>(begin), b.ids.begin() + static_cast<std::ptrdiff_t>(end));
    r.dist_sq.assign(b.dist_sq.begin() + static_cast<std::ptrdiff_t>(begin),
                     b.dist_sq.begin() + static_cast<std::ptrdiff_t>(end));
    const trim_counters& c = b.counters[0];
    r.counters.dc = c.dc;
    r.counters.edc = c.edc;
    r.counters.pruned = c.pruned;
    r.counters.evaluated = c.evaluated;
    r.counters.hops = c.hops;
    r.coarse_dc = c.coarse_dc;
    return r;
}
template <class View>
const float* data_of(const View& q, std::uint32_t dim) {
    if (static_cast<std::size_t>(q.size()) != dim)
        throw std::invalid_argument("query dimension mismatch");
    return q.data();
}
} // namespace detail

// ivf::search_trim_ivf_knn (ivf.hpp:243-304); View = std::span<const float>,
// std::vector<float>, trimsearch::VectorView, ...
template <class Profile, class View>
IvfResult search_trim_ivf_knn(const GpuIvfIndex& ix, const Profile& prof, const View& q, std::size_t k,
                              std::size_t nprobe) {
    const auto b = search_trim_ivf_knn_batch(ix, prof, detail::data_of(q, ix.dim()), 1, k, nprobe);
    return detail::one(b, 0, k);
}

// ivf::search_trim_ivf_range (ivf.hpp:308-347)
template <class Profile, class View>
IvfResult search_trim_ivf_range(const GpuIvfIndex& ix, const Profile& prof, const View& q, float radius,
                                std::size_t nprobe) {
    const auto b = search_trim_ivf_range_batch(ix, prof, detail::data_of(q, ix.dim()), 1, &radius, nprobe);
    return detail::one(b, 0, b.offsets[1]);
}

// ivf::search_baseline_ivfpq (ivf.hpp:193-237)
template <class View>
IvfResult search_baseline_ivfpq(const GpuIvfIndex& ix, const View& q, std::size_t k, std::size_t nprobe,
                                std::size_t k_prime) {
    const auto b = search_baseline_ivfpq_batch(ix, detail::data_of(q, ix.dim()), 1, k, nprobe, k_prime);
    return detail::one(b, 0, k);
}

} // namespace ivf
} // namespace trim_b200
