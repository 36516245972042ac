// trim_host.h — host plumbing shared by the C-ABI translation units
// (trim_capi.cu: single-device indexes; trim_multi.cu: multi-device layouts).
// Internal: not part of the ABI (include/trim_gpu.h is).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/trim_gpu.h"
#include "trim_common.cuh"

namespace trimhost {
using trimgpu::DevIndex;

inline thread_local std::string g_err;
// Perf probe (profiles/knn_timeline.py): device buffer of nq*kTimeline u64 that the next kNN
// launches on this thread fill with per-CTA phase timestamps; null disables.
inline thread_local unsigned long long* g_timeline = nullptr;

inline int set_err(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

struct CudaError {
    int code;
};

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t _e = (call);                                                          \
        if (_e != cudaSuccess) {                                                          \
            ::trimhost::set_err(TRIM_ECUDA, "CUDA error %s (%s) at %s:%d",                 \
                                cudaGetErrorName(_e), cudaGetErrorString(_e), __FILE__, __LINE__); \
            throw ::trimhost::CudaError{TRIM_ECUDA};                                      \
        }                                                                                 \
    } while (0)

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        return fn();
    } catch (const CudaError& e) {
        return e.code;
    } catch (const std::bad_alloc&) {
        return set_err(TRIM_ENOMEM, "host allocation failed");
    } catch (const std::runtime_error& e) { // a nested trim_* call failed (message kept)
        return set_err(TRIM_ECUDA, "%s", e.what());
    }
}

inline uint32_t round_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

inline uint32_t pow2_at_least(uint32_t x) {
    uint32_t p = 1;
    while (p < x)
        p <<= 1;
    return p;
}

// Per-host-thread resources of the host API: one non-blocking stream per
// device and a pinned status word. Released when the thread exits (client
// thread pools that come and go do not accumulate streams or pinned pages).
struct ThreadRes {
    std::vector<cudaStream_t> streams;
    uint32_t* word = nullptr;
    ~ThreadRes() {
        int prev = 0;
        const bool have = cudaGetDevice(&prev) == cudaSuccess;
        for (size_t d = 0; d < streams.size(); ++d)
            if (streams[d]) {
                cudaSetDevice(static_cast<int>(d));
                cudaStreamDestroy(streams[d]);
            }
        if (word)
            cudaFreeHost(word);
        if (have)
            cudaSetDevice(prev);
    }
};
inline ThreadRes& thread_res() {
    thread_local ThreadRes r;
    return r;
}

inline cudaStream_t thread_stream(int device) {
    auto& streams = thread_res().streams;
    if (static_cast<int>(streams.size()) <= device)
        streams.resize(device + 1, nullptr);
    if (!streams[device])
        CK(cudaStreamCreateWithFlags(&streams[device], cudaStreamNonBlocking));
    return streams[device];
}

// A pinned host word per thread (status readbacks without a pageable copy).
inline uint32_t* pinned_word() {
    uint32_t*& w = thread_res().word;
    if (!w)
        CK(cudaMallocHost(&w, sizeof(uint32_t)));
    return w;
}

// RAII stream-ordered device buffer on the device current at construction
// (freed on that device, whatever is current when it goes out of scope).
struct DevBuf {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    int dev = 0;
    DevBuf() = default;
    DevBuf(size_t bytes, cudaStream_t st) : s(st) {
        CK(cudaGetDevice(&dev));
        if (bytes)
            CK(cudaMallocAsync(&p, bytes, st));
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), s(o.s), dev(o.dev) { o.p = nullptr; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        std::swap(p, o.p);
        std::swap(s, o.s);
        std::swap(dev, o.dev);
        return *this;
    }
    ~DevBuf() {
        if (!p)
            return;
        int cur = dev;
        cudaGetDevice(&cur);
        if (cur != dev)
            cudaSetDevice(dev);
        cudaFreeAsync(p, s);
        if (cur != dev)
            cudaSetDevice(cur);
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int d) {
        CK(cudaGetDevice(&prev));
        if (prev != d)
            CK(cudaSetDevice(d));
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

} // namespace trimhost

struct NcclGroup; // trim_multi.cu
struct trim_index;
namespace trimhost {
void group_destroy(trim_index* ix);
}

struct trim_index {
    int device = 0;
    trimgpu::DevIndex dev{};
    uint32_t code_stride_host = 0;
    uint64_t total = 0;
    std::vector<uint64_t> list_offsets;  // host copy
    std::vector<uint64_t> top_prefix;    // prefix sums of list sizes sorted descending
    uint64_t max_list = 0;
    uint32_t max_sub_dim = 0;
    unsigned long long* d_skipped = nullptr; // trim_index_skip_stats
    // tensor-core probe (trim_probe_mma.cuh): pre-tiled centroids and norms
    float4* coarse_t = nullptr;
    float* cn2 = nullptr;
    float* cn = nullptr;
    // flat kNN distance bounds (trim_flat_mma.cuh): pre-tiled rows + norms, built on first use
    std::mutex flat_mu;
    float4* flat_tiles = nullptr;
    float* xn = nullptr;
    float* xn2 = nullptr;
    // flat range search: a block partition of the rows (build_flat_partition), built on first use
    std::mutex part_mu;
    bool part_tried = false;
    uint32_t part_nb = 0;
    trimgpu::DevIndex part{};
    float4* part_tiles = nullptr;
    float* part_cn2 = nullptr;
    float* part_cn = nullptr;
    uint32_t* part_assign = nullptr; // block of every row
    // flat kNN: rows n0.. regrouped by (segment of seg_len consecutive ids, block) for the
    // segmented block scan (ensure_flat_segments), built on first use
    std::mutex seg_mu;
    bool seg_tried = false, seg_ok = false;
    std::vector<uint64_t> seg_bounds; // segment g = rows [seg_bounds[g], seg_bounds[g + 1]); [0] = n0
    uint32_t seg_nseg = 0;
    uint64_t* seg_off = nullptr;  // nseg * part_nb + 1
    trimgpu::DevIndex seg{};      // dev with the regrouped codes / lx / ids
    trimgpu::DevIndex seg_head{}; // dev restricted to rows [0, n0)
    uint64_t bytes = 0;
    std::vector<void*> allocs;
    // multi-device layouts (trim_index_desc.ndevices > 0, trim_multi.cu): this
    // object is then a group over `parts` (one single-device index per entry of
    // `devices`, in order); `device` is the home device (devices[0])
    uint32_t shard_mode = TRIM_SHARD_SINGLE;
    std::vector<trim_index*> parts;
    std::vector<uint64_t> part_lo; // id_shard: part p holds ids [part_lo[p], part_lo[p+1])
    NcclGroup* nccl = nullptr;     // id_shard over distinct devices

    bool is_group() const { return !parts.empty(); }

    ~trim_index() {
        if (is_group())
            trimhost::group_destroy(this);
        if (!allocs.empty()) {
            int prev = 0;
            cudaGetDevice(&prev);
            cudaSetDevice(device);
            for (void* p : allocs)
                cudaFree(p);
            cudaSetDevice(prev);
        }
    }

    template <typename T>
    T* alloc(size_t count) {
        void* p = nullptr;
        const size_t b = std::max<size_t>(sizeof(T) * count, 16);
        CK(cudaMalloc(&p, b));
        allocs.push_back(p);
        bytes += b;
        return static_cast<T*>(p);
    }

    // Upper bound on a query's stream length at `np` probes.
    uint64_t stream_bound(uint32_t np) const {
        np = std::min<uint32_t>(np, dev.nlist);
        return top_prefix[np];
    }
};

namespace trimhost {
// trim_capi.cu
int check_device_present();
int validate_knn(uint32_t k, float gamma);
DevBuf upload_queries(const trim_index* ix, const float* q, uint64_t nq, cudaMemcpyKind kind, cudaStream_t st);
uint32_t run_probe(const trim_index* ix, const float* d_q, uint64_t nq, uint32_t nprobe, DevBuf& d_probe,
                   cudaStream_t st);
int knn_device(const trim_index* ix, const float* d_q, uint64_t nq, uint32_t k, uint32_t nprobe, float gamma,
               uint32_t* d_ids, float* d_dist, unsigned long long* d_ct, uint32_t* d_status, cudaStream_t st);
void range_launch(const trim_index* ix, const float* d_q, uint64_t nq, const float* d_r2, uint32_t np,
                  const uint32_t* d_probe, float gamma, uint32_t cap, unsigned long long* d_keys, unsigned int* d_cnt,
                  unsigned long long* d_dc, unsigned long long* d_eval, cudaStream_t st);
int baseline_device(const trim_index* ix, const float* d_q, uint64_t nq, uint32_t k, uint32_t np,
                    const uint32_t* d_probe, uint32_t kp, uint32_t* ids_out, float* dist_out,
                    trim_counters* counters_out, cudaStream_t st);
int create_single(const trim_index_desc* d, trim_index** out);
// trim_multi.cu: multi-device layouts (trim_index_desc.ndevices > 0)
int group_create(const trim_index_desc* d, trim_index** out);
void group_destroy(trim_index* ix);
int group_search_knn(trim_index* ix, const float* queries, uint64_t nq, uint32_t k, uint32_t nprobe, float gamma,
                     uint32_t* ids_out, float* dist_out, trim_counters* counters_out);
int group_search_knn_device(trim_index* ix, const float* d_queries, uint64_t nq, uint32_t k, uint32_t nprobe,
                            float gamma, uint32_t* d_ids, float* d_dist, trim_counters* d_counters,
                            uint32_t* d_status, void* stream);
int group_search_range(trim_index* ix, const float* queries, uint64_t nq, const float* radius, uint32_t nprobe,
                       float gamma, uint64_t* offsets_out, uint32_t** ids_out, float** dist_out,
                       trim_counters* counters_out);
int group_search_baseline(trim_index* ix, const float* queries, uint64_t nq, uint32_t k, uint32_t nprobe,
                          uint32_t k_prime, uint32_t* ids_out, float* dist_out, trim_counters* counters_out);
} // namespace trimhost
