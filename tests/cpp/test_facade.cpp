// Exercises include/trim_b200/ivf.hpp (the reference-shaped C++ façade) on a
// GPU: the assertions restate proj/tests/test_ivf.cpp (exactness at gamma=0
// with full probing :171-200, accounting identity :202-224, error cases
// :246-251/:286-290) against types that carry the reference's member names.
// Built and run by tests/test_cpp_facade.py.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <span>
#include <stdexcept>
#include <vector>

#include "trim_b200/ivf.hpp"

namespace {

int failures = 0;
#define CHECK(cond)                                                                  \
    do {                                                                             \
        if (!(cond)) {                                                               \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                              \
        }                                                                            \
    } while (0)
template <class E, class F>
void check_throws(F&& f, const char* what) {
    try {
        f();
    } catch (const E&) {
        return;
    } catch (...) {
    }
    std::fprintf(stderr, "expected exception not thrown: %s\n", what);
    ++failures;
}

// The reference's member names (ivf.hpp:29-51, pq.hpp:40-54, dataset.hpp:18-27)
struct Params { std::size_t m, c; };
struct Codebook { Params params; std::vector<std::size_t> sub_dims; std::vector<std::vector<float>> centroids; };
struct List { std::vector<std::uint32_t> ids; std::vector<std::uint8_t> codes; std::vector<float> lx_dist; };
struct Ivf { std::size_t dim, nlist; Codebook codebook; std::vector<float> coarse_centroids; std::vector<List> lists; };
struct Dataset { std::size_t dim, count; std::vector<float> data; };

float euclid(const float* a, const float* b, std::size_t d) { // distance.hpp:11-29
    float a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    std::size_t i = 0;
    for (; i + 4 <= d; i += 4) {
        const float x0 = a[i] - b[i], x1 = a[i + 1] - b[i + 1], x2 = a[i + 2] - b[i + 2], x3 = a[i + 3] - b[i + 3];
        a0 += x0 * x0; a1 += x1 * x1; a2 += x2 * x2; a3 += x3 * x3;
    }
    for (; i < d; ++i) { const float x = a[i] - b[i]; a0 += x * x; }
    return (a0 + a1) + (a2 + a3);
}

} // namespace

int main() {
    const std::size_t n = 3000, dim = 16, m = 4, c = 32, nlist = 12;
    std::mt19937_64 rng(7);
    std::normal_distribution<float> nd(0.0f, 1.0f);
    Dataset ds{dim, n, std::vector<float>(n * dim)};
    for (auto& v : ds.data) v = nd(rng);
    Ivf ix;
    ix.dim = dim;
    ix.nlist = nlist;
    ix.codebook.params = {m, c};
    ix.codebook.sub_dims.assign(m, dim / m);
    for (std::size_t j = 0; j < m; ++j) { // any codebook will do: rows of the data
        std::vector<float> cj(c * (dim / m));
        for (std::size_t i = 0; i < c; ++i)
            for (std::size_t t = 0; t < dim / m; ++t)
                cj[i * (dim / m) + t] = ds.data[(i * 13) * dim + j * (dim / m) + t];
        ix.codebook.centroids.push_back(cj);
    }
    for (std::size_t l = 0; l < nlist; ++l)
        for (std::size_t t = 0; t < dim; ++t)
            ix.coarse_centroids.push_back(ds.data[(l * 101) * dim + t]);
    ix.lists.resize(nlist);
    for (std::uint32_t i = 0; i < n; ++i) { // nearest coarse centroid, ascending ids
        std::size_t best = 0;
        float bd = 3.4e38f;
        for (std::size_t l = 0; l < nlist; ++l) {
            const float d = euclid(&ds.data[i * dim], &ix.coarse_centroids[l * dim], dim);
            if (d < bd) { bd = d; best = l; }
        }
        List& L = ix.lists[best];
        L.ids.push_back(i);
        std::vector<float> lm(dim);
        for (std::size_t j = 0; j < m; ++j) {
            std::size_t bc = 0;
            float bcd = 3.4e38f;
            for (std::size_t k = 0; k < c; ++k) {
                const float d = euclid(&ds.data[i * dim + j * 4], &ix.codebook.centroids[j][k * 4], 4);
                if (d < bcd) { bcd = d; bc = k; }
            }
            L.codes.push_back(static_cast<std::uint8_t>(bc));
            std::copy_n(&ix.codebook.centroids[j][bc * 4], 4, &lm[j * 4]);
        }
        L.lx_dist.push_back(std::sqrt(euclid(&ds.data[i * dim], lm.data(), dim)));
    }

    auto g = trim_b200::from_reference(ix, ds);
    CHECK(g.info().total_entries == n);
    std::vector<float> qs(20 * dim);
    for (auto& v : qs) v = nd(rng);
    const auto zero = trim_b200::PruningProfile::manual(0.0);

    // test_ivf.cpp:171-185 — gamma = 0 with full probing is exact kNN
    for (std::size_t k : {1u, 10u}) {
        for (std::size_t qi = 0; qi < 20; ++qi) {
            const std::span<const float> q(&qs[qi * dim], dim);
            const auto r = trim_b200::ivf::search_trim_ivf_knn(g, zero, q, k, nlist);
            std::vector<std::pair<float, std::uint32_t>> bf;
            for (std::uint32_t i = 0; i < n; ++i)
                bf.push_back({euclid(q.data(), &ds.data[i * dim], dim), i});
            std::sort(bf.begin(), bf.end());
            CHECK(r.ids.size() == k);
            for (std::size_t i = 0; i < k; ++i) {
                CHECK(r.ids[i] == bf[i].second);
                CHECK(r.dist_sq[i] == bf[i].first);
            }
            // test_ivf.cpp:209 — accounting identity
            CHECK(r.counters.dc + r.counters.pruned == r.counters.evaluated);
            CHECK(r.counters.evaluated == n);
            CHECK(r.coarse_dc == nlist);
        }
    }
    // test_ivf.cpp:187-200 — range at gamma = 0, full probe, equals brute force
    for (std::size_t qi = 0; qi < 20; ++qi) {
        const std::span<const float> q(&qs[qi * dim], dim);
        const float radius = 4.0f;
        const auto r = trim_b200::ivf::search_trim_ivf_range(g, zero, q, radius, nlist);
        std::size_t want = 0;
        for (std::uint32_t i = 0; i < n; ++i)
            want += euclid(q.data(), &ds.data[i * dim], dim) <= radius * radius;
        CHECK(r.ids.size() == want);
        for (std::size_t i = 0; i < r.ids.size(); ++i)
            CHECK(r.dist_sq[i] == euclid(q.data(), &ds.data[r.ids[i] * dim], dim));
    }
    // batch == per query
    const auto prof = trim_b200::PruningProfile::manual(0.5);
    const auto b = trim_b200::ivf::search_trim_ivf_knn_batch(g, prof, qs.data(), 20, 5, 4);
    for (std::size_t qi = 0; qi < 20; ++qi) {
        const std::span<const float> q(&qs[qi * dim], dim);
        const auto r = trim_b200::ivf::search_trim_ivf_knn(g, prof, q, 5, 4);
        for (std::size_t i = 0; i < 5; ++i)
            CHECK(r.ids[i] == b.ids[qi * 5 + i]);
    }
    // baseline IVFPQ with k' = n and full probing is exact (test_ivf.cpp:121-135)
    {
        const std::span<const float> q(&qs[0], dim);
        const auto r = trim_b200::ivf::search_baseline_ivfpq(g, q, 10, nlist, n);
        CHECK(r.counters.dc == n);
    }
    // error semantics (ivf.hpp:195-198, 246-249, 289-290, 311-314)
    const std::span<const float> q0(&qs[0], dim);
    check_throws<std::invalid_argument>([&] { trim_b200::ivf::search_trim_ivf_knn(g, prof, q0, 0, 2); }, "k=0");
    check_throws<std::invalid_argument>(
        [&] { trim_b200::ivf::search_trim_ivf_knn(g, trim_b200::PruningProfile{}, q0, 5, 2); }, "uncalibrated");
    check_throws<std::invalid_argument>([&] { trim_b200::ivf::search_trim_ivf_knn(g, prof, q0, n + 1, nlist); },
                                        "k exceeds probed");
    check_throws<std::invalid_argument>([&] { trim_b200::ivf::search_trim_ivf_range(g, prof, q0, -1.0f, 2); },
                                        "negative radius");
    check_throws<std::invalid_argument>([&] { trim_b200::ivf::search_baseline_ivfpq(g, q0, 10, 4, 5); }, "k > k'");
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
