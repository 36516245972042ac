// trim_multi.cu — multi-device index layouts behind the C ABI
// (include/trim_gpu.h: trim_index_desc.devices / ndevices / shard_mode).
//
// SURVEY.md §8e. The reference has one caller, bench::run_sweep, which fans
// queries out over host threads (sweep.hpp:121-152, 237-246); here one process
// drives every GPU of the box through one index handle:
//
//   TRIM_SHARD_ID        part p (on devices[p]) holds ids [p*n/W, (p+1)*n/W):
//                        for every inverted list the sub-range of its entries
//                        with those ids (entries ascend by id inside a list,
//                        ivf.hpp:147-152, so each is one contiguous run) and
//                        those vector rows; codebook and coarse quantizer are
//                        replicated, so every part computes the same probe
//                        order. A search broadcasts the query batch from the
//                        home device (devices[0]), runs every part's fused
//                        filter on its sub-stream of each query — its result
//                        and counters equal the reference run over that
//                        shard's candidate subsequence — all-gathers the
//                        per-part top-k (dist, id) and counters (the only data
//                        exchange: k*8 + 48 bytes per query per part), merges
//                        on the home device by (dist, id) (ScoredId order,
//                        ground_truth.hpp:39-50) and sums the counters. With
//                        distinct devices the broadcast / all-gather are NCCL
//                        collectives over NVLink (libnccl.so.2, loaded at first
//                        use); when devices[] repeats an entry (several shards
//                        on one GPU, e.g. for tests) they are device-to-device
//                        copies. Result parity with the unsharded run is exact
//                        at gamma = 0 (a sound bound); for gamma > 0 the prune
//                        decisions are per shard.
//   TRIM_SHARD_REPLICAS  every device holds the whole index; a batch is split
//                        into contiguous query slices, one per device; results
//                        equal the single-device run; no collective.
#include <cub/device/device_segmented_sort.cuh>
#include <dlfcn.h>
#include <nccl.h> // types and prototypes only: the library is dlopen()ed

#include <cstdlib>
#include <thread>

#include "trim_host.h"

using namespace trimhost;

// ------------------------------------------------------------------ NCCL
namespace {

struct NcclApi {
    decltype(&ncclCommInitAll) comm_init_all = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    std::string err;
    bool ok = false;
};

NcclApi load_nccl() {
    NcclApi a;
    // the process may already hold torch's libnccl.so.2: dlopen returns it
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h)
        h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        const char* e = dlerror();
        a.err = e ? e : "dlopen(libnccl.so.2) failed";
        return a;
    }
#define TRIM_NCCL_SYM(field, name)                                                                 \
    a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));                                 \
    if (!a.field) {                                                                                \
        a.err = std::string("libnccl.so.2 lacks ") + name;                                         \
        return a;                                                                                  \
    }
    TRIM_NCCL_SYM(comm_init_all, "ncclCommInitAll")
    TRIM_NCCL_SYM(comm_destroy, "ncclCommDestroy")
    TRIM_NCCL_SYM(group_start, "ncclGroupStart")
    TRIM_NCCL_SYM(group_end, "ncclGroupEnd")
    TRIM_NCCL_SYM(all_gather, "ncclAllGather")
    TRIM_NCCL_SYM(broadcast, "ncclBroadcast")
    TRIM_NCCL_SYM(error_string, "ncclGetErrorString")
#undef TRIM_NCCL_SYM
    a.ok = true;
    return a;
}

const NcclApi& nccl() {
    static const NcclApi a = load_nccl();
    return a;
}

struct NcclError {};

#define NK(call)                                                                                   \
    do {                                                                                           \
        const ncclResult_t _r = (call);                                                            \
        if (_r != ncclSuccess) {                                                                   \
            set_err(TRIM_ENCCL, "NCCL error %d (%s) at %s:%d", static_cast<int>(_r),               \
                    nccl().error_string ? nccl().error_string(_r) : "?", __FILE__, __LINE__);      \
            throw CudaError{TRIM_ENCCL};                                                           \
        }                                                                                          \
    } while (0)

// TRIM_NCCL=0 replaces the collectives by device-to-device copies (A/B; the
// results are identical).
bool nccl_wanted() {
    const char* e = std::getenv("TRIM_NCCL");
    return !(e && e[0] == '0');
}

} // namespace

struct NcclGroup {
    std::vector<ncclComm_t> comms; // one per part, rank p = part p
    // Every collective is enqueued on all W communicators inside one
    // ncclGroupStart/End; concurrent host calls on the index take this lock
    // around each such group, so every communicator sees the same sequence of
    // collectives (two threads interleaving per-communicator enqueues could
    // order them differently on two devices and deadlock).
    std::mutex mu;
    ~NcclGroup() {
        for (ncclComm_t c : comms)
            if (c)
                nccl().comm_destroy(c);
    }
};

// ------------------------------------------------------------------ kernels
namespace {

// Per-query counters summed over W parts ([W][nq][6] -> [nq][6]); coarse_dc
// is one part's (every part runs the same probe, ivf.hpp:173-187). Bit 0 of
// *status: some query's total stream (over all parts) is shorter than k —
// the reference's "k exceeds probed vectors" (ivf.hpp:289-290).
__global__ void group_counters_kernel(const unsigned long long* __restrict__ ct, uint32_t W, uint64_t nq, uint32_t k,
                                      unsigned long long* __restrict__ out, uint32_t* __restrict__ status) {
    const uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= nq)
        return;
    unsigned long long s[5] = {0, 0, 0, 0, 0};
    for (uint32_t p = 0; p < W; ++p)
        for (int i = 0; i < 5; ++i)
            s[i] += ct[(static_cast<uint64_t>(p) * nq + q) * 6 + i];
    if (out) {
        for (int i = 0; i < 5; ++i)
            out[q * 6 + i] = s[i];
        out[q * 6 + 5] = ct[q * 6 + 5];
    }
    if (status && s[3] < k)
        atomicOr(status, 1u);
}

// Range results of W parts: part p's unsorted (d, id) keys of query q are
// keys[p][q][0 .. min(cnt[p][q], cap)); compact them into query q's segment
// [q*W*cap, q*W*cap + sum_p cnt[p][q]) for the per-query sort (ivf.hpp:341).
__global__ void group_range_compact_kernel(const unsigned long long* __restrict__ keys,
                                           const unsigned int* __restrict__ cnt, uint32_t W, uint64_t nq, uint32_t cap,
                                           unsigned long long* __restrict__ out, uint64_t* __restrict__ beg,
                                           uint64_t* __restrict__ end) {
    const uint64_t q = blockIdx.x;
    if (q >= nq)
        return;
    const uint64_t seg = q * W * cap;
    uint64_t o = seg;
    for (uint32_t p = 0; p < W; ++p) {
        const uint32_t c = min(cnt[static_cast<uint64_t>(p) * nq + q], cap);
        const unsigned long long* src = keys + (static_cast<uint64_t>(p) * nq + q) * cap;
        for (uint32_t i = threadIdx.x; i < c; i += blockDim.x)
            out[o + i] = src[i];
        o += c;
    }
    if (threadIdx.x == 0) {
        beg[q] = seg;
        end[q] = o;
    }
}

__global__ void group_range_unpack_kernel(const unsigned long long* __restrict__ sorted, uint32_t W, uint32_t cap,
                                          const uint64_t* __restrict__ offs, uint64_t nq, uint32_t* __restrict__ ids,
                                          float* __restrict__ dist) {
    const uint64_t q = blockIdx.x;
    if (q >= nq)
        return;
    const uint64_t o = offs[q], n = offs[q + 1] - o, seg = q * W * cap;
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const unsigned long long key = sorted[seg + i];
        ids[o + i] = static_cast<uint32_t>(key & 0xffffffffu);
        dist[o + i] = __uint_as_float(static_cast<uint32_t>(key >> 32));
    }
}

__global__ void group_status_or_kernel(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst) {
    if (*src)
        atomicOr(dst, *src);
}

// r^2 = r * r in fp32 (ivf.hpp:315)
__global__ void group_r2_kernel(const float* __restrict__ r, uint64_t nq, float* __restrict__ r2) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < nq)
        r2[i] = __fmul_rn(r[i], r[i]);
}

// ------------------------------------------------------------------ helpers
uint32_t parts_of(const trim_index* ix) { return static_cast<uint32_t>(ix->parts.size()); }

// Contiguous query slice of part p (replicas).
void slice_of(uint64_t nq, uint32_t p, uint32_t W, uint64_t& lo, uint64_t& n) {
    lo = nq * p / W;
    n = nq * (p + 1) / W - lo;
}

struct Ev {
    cudaEvent_t e = nullptr;
    int dev = 0;
    explicit Ev(int d) : dev(d) {
        DeviceGuard g(d);
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    Ev(const Ev&) = delete;
    Ev& operator=(const Ev&) = delete;
    ~Ev() {
        if (e) {
            int cur = dev;
            cudaGetDevice(&cur);
            cudaSetDevice(dev);
            cudaEventDestroy(e);
            cudaSetDevice(cur);
        }
    }
};

// b waits for everything enqueued on a so far (a on device da).
void order_after(cudaStream_t a, int da, cudaStream_t b, int db) {
    Ev ev(da);
    {
        DeviceGuard g(da);
        CK(cudaEventRecord(ev.e, a));
    }
    DeviceGuard g(db);
    CK(cudaStreamWaitEvent(b, ev.e, 0));
}

// host-memory copy of `count` elements of a descriptor array (host or device)
template <typename T>
std::vector<T> host_copy(const T* src, size_t count, bool host) {
    std::vector<T> v(count);
    if (!count)
        return v;
    if (host)
        std::memcpy(v.data(), src, sizeof(T) * count);
    else
        CK(cudaMemcpy(v.data(), src, sizeof(T) * count, cudaMemcpyDeviceToHost));
    return v;
}

} // namespace

// ------------------------------------------------------------------ create
int trimhost::group_create(const trim_index_desc* d, trim_index** out) {
    *out = nullptr;
    const uint32_t W = d->ndevices;
    std::vector<int> devs(d->devices, d->devices + W);
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    for (int v : devs)
        if (v < 0 || v >= ndev)
            return set_err(TRIM_EINVAL, "trim_index_create: device %d out of range (%d devices)", v, ndev);
    if (d->id_base != 0)
        return set_err(TRIM_EINVAL, "trim_index_create: a multi-device descriptor holds the whole index (id_base 0)");
    auto* g = new trim_index;
    g->shard_mode = d->shard_mode;
    g->device = devs[0];
    try {
        const bool host = d->memory == TRIM_MEM_HOST;
        if (d->shard_mode == TRIM_SHARD_REPLICAS) {
            for (uint32_t p = 0; p < W; ++p) {
                trim_index_desc pd = *d;
                pd.ndevices = 0;
                pd.devices = nullptr;
                pd.shard_mode = TRIM_SHARD_SINGLE;
                pd.device = devs[p];
                trim_index* part = nullptr;
                if (int rc = create_single(&pd, &part)) {
                    delete g;
                    return rc;
                }
                g->parts.push_back(part);
            }
        } else {
            // id shards: split every list at the part boundaries (host staging)
            const uint32_t nlist = d->nlist, m = d->m, cs = d->code_stride, dim = d->dim;
            const uint64_t n = d->n;
            const std::vector<uint64_t> offs = host_copy(d->list_offsets, nlist + 1, host);
            const uint64_t total = offs[nlist];
            const std::vector<uint32_t> ids = host_copy(d->list_ids, total, host);
            std::vector<uint8_t> codes_h;
            std::vector<float> lx_h, vec_h;
            const uint8_t* codes = d->list_codes;
            const float* lx = d->list_lx;
            const float* vec = d->vectors;
            if (!host) {
                codes_h = host_copy(d->list_codes, total * cs, false);
                lx_h = host_copy(d->list_lx, total, false);
                vec_h = host_copy(d->vectors, n * dim, false);
                codes = codes_h.data();
                lx = lx_h.data();
                vec = vec_h.data();
            }
            for (uint32_t l = 0; l < nlist; ++l)
                for (uint64_t e = offs[l] + 1; e < offs[l + 1]; ++e)
                    if (ids[e] <= ids[e - 1]) {
                        delete g;
                        return set_err(TRIM_EDATA, "id sharding needs ascending ids inside every list "
                                                   "(ivf.hpp:147-152); list %u is not", l);
                    }
            std::vector<uint32_t> sub = host_copy(d->sub_dims, m, host);
            std::vector<float> cent = host_copy(d->centroids, static_cast<size_t>(d->ksub) * dim, host);
            std::vector<float> coarse = host_copy(d->coarse, static_cast<size_t>(nlist) * dim, host);
            for (uint32_t p = 0; p <= W; ++p)
                g->part_lo.push_back(n * p / W);
            for (uint32_t p = 0; p < W; ++p) {
                const uint64_t lo = g->part_lo[p], hi = g->part_lo[p + 1];
                std::vector<uint64_t> po(nlist + 1, 0);
                std::vector<uint32_t> pid;
                std::vector<uint8_t> pcode;
                std::vector<float> plx;
                for (uint32_t l = 0; l < nlist; ++l) {
                    const uint32_t* b = ids.data() + offs[l];
                    const uint32_t* e = ids.data() + offs[l + 1];
                    const uint64_t s0 = offs[l] + (std::lower_bound(b, e, lo) - b);
                    const uint64_t s1 = offs[l] + (std::lower_bound(b, e, hi) - b);
                    pid.insert(pid.end(), ids.begin() + s0, ids.begin() + s1);
                    pcode.insert(pcode.end(), codes + s0 * cs, codes + s1 * cs);
                    plx.insert(plx.end(), lx + s0, lx + s1);
                    po[l + 1] = po[l] + (s1 - s0);
                }
                trim_index_desc pd = *d;
                pd.ndevices = 0;
                pd.devices = nullptr;
                pd.shard_mode = TRIM_SHARD_SINGLE;
                pd.device = devs[p];
                pd.memory = TRIM_MEM_HOST;
                pd.sub_dims = sub.data();
                pd.centroids = cent.data();
                pd.coarse = coarse.data();
                pd.list_offsets = po.data();
                pd.list_ids = pid.data();
                pd.list_codes = pcode.data();
                pd.list_lx = plx.data();
                pd.n = hi - lo;
                pd.vectors = vec + lo * dim;
                pd.id_base = lo;
                trim_index* part = nullptr;
                if (int rc = create_single(&pd, &part)) {
                    delete g;
                    return rc;
                }
                g->parts.push_back(part);
            }
            bool distinct = true;
            for (uint32_t a = 0; a < W; ++a)
                for (uint32_t b = a + 1; b < W; ++b)
                    distinct &= devs[a] != devs[b];
            if (distinct && nccl_wanted()) {
                if (!nccl().ok) {
                    delete g;
                    return set_err(TRIM_ENCCL, "id_shard index over %u devices needs NCCL: %s", W, nccl().err.c_str());
                }
                auto* ng = new NcclGroup;
                ng->comms.assign(W, nullptr);
                const ncclResult_t r = nccl().comm_init_all(ng->comms.data(), static_cast<int>(W), devs.data());
                if (r != ncclSuccess) {
                    ng->comms.assign(W, nullptr);
                    delete ng;
                    delete g;
                    return set_err(TRIM_ENCCL, "ncclCommInitAll over %u devices: %s", W, nccl().error_string(r));
                }
                g->nccl = ng;
            }
        }
    } catch (...) {
        delete g;
        throw;
    }
    // the group's own descriptor fields (trim_index_get_info)
    const trim_index* p0 = g->parts[0];
    g->dev = p0->dev;
    g->dev.n = d->n;
    g->dev.id_base = 0;
    g->max_list = 0;
    g->total = 0;
    for (const trim_index* pt : g->parts) {
        g->total += pt->total;
        g->max_list = std::max(g->max_list, pt->max_list);
    }
    if (d->shard_mode == TRIM_SHARD_REPLICAS)
        g->total = p0->total;
    *out = g;
    return TRIM_OK;
}

void trimhost::group_destroy(trim_index* ix) {
    delete ix->nccl;
    ix->nccl = nullptr;
    for (trim_index* p : ix->parts)
        delete p;
    ix->parts.clear();
}

// ------------------------------------------------------------------ kNN
// Queries and outputs on the home device, ordered on the caller's `stream`.
int trimhost::group_search_knn_device(trim_index* ix, const float* d_queries, uint64_t nq, uint32_t k,
                                      uint32_t nprobe, float gamma, uint32_t* d_ids, float* d_dist,
                                      trim_counters* d_counters, uint32_t* d_status, void* stream) {
    const uint32_t W = parts_of(ix);
    const int home = ix->device;
    const uint32_t dim = ix->dev.dim, ds = ix->dev.dim_stride;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    DeviceGuard gh(home);
    // padded query rows on the home device (dim_stride floats)
    DevBuf qpad;
    const float* q = d_queries;
    if (ds != dim) {
        qpad = upload_queries(ix->parts[0], d_queries, nq, cudaMemcpyDeviceToDevice, st);
        q = qpad.as<float>();
    }
    if (ix->shard_mode == TRIM_SHARD_REPLICAS) {
        // slice p searched on devices[p]; part 0 (home) on the caller's stream
        std::vector<DevBuf> bq(W), bi(W), bd(W), bc(W), bs(W);
        std::vector<cudaStream_t> sts(W, st);
        for (uint32_t p = 1; p < W; ++p) {
            const int dv = ix->parts[p]->device;
            sts[p] = thread_stream(dv);
            order_after(st, home, sts[p], dv);
        }
        for (uint32_t p = 0; p < W; ++p) {
            uint64_t lo, n;
            slice_of(nq, p, W, lo, n);
            if (!n)
                continue;
            const int dv = ix->parts[p]->device;
            DeviceGuard g(dv);
            unsigned long long* ct = d_counters ? reinterpret_cast<unsigned long long*>(d_counters + lo) : nullptr;
            if (p == 0) {
                if (int rc = knn_device(ix->parts[0], q, n, k, nprobe, gamma, d_ids, d_dist, ct, d_status, st))
                    return rc;
                continue;
            }
            cudaStream_t s = sts[p];
            bq[p] = DevBuf(sizeof(float) * n * ds, s);
            CK(cudaMemcpyPeerAsync(bq[p].p, dv, q + lo * ds, home, sizeof(float) * n * ds, s));
            bi[p] = DevBuf(sizeof(uint32_t) * n * k, s);
            bd[p] = DevBuf(sizeof(float) * n * k, s);
            bc[p] = DevBuf(sizeof(unsigned long long) * n * 6, s);
            bs[p] = DevBuf(sizeof(uint32_t), s);
            CK(cudaMemsetAsync(bs[p].p, 0, sizeof(uint32_t), s));
            if (int rc = knn_device(ix->parts[p], bq[p].as<float>(), n, k, nprobe, gamma, bi[p].as<uint32_t>(),
                                    bd[p].as<float>(), bc[p].as<unsigned long long>(), bs[p].as<uint32_t>(), s))
                return rc;
            CK(cudaMemcpyPeerAsync(d_ids + lo * k, home, bi[p].p, dv, sizeof(uint32_t) * n * k, s));
            CK(cudaMemcpyPeerAsync(d_dist + lo * k, home, bd[p].p, dv, sizeof(float) * n * k, s));
            if (ct)
                CK(cudaMemcpyPeerAsync(ct, home, bc[p].p, dv, sizeof(unsigned long long) * n * 6, s));
        }
        for (uint32_t p = 1; p < W; ++p)
            order_after(sts[p], ix->parts[p]->device, st, home);
        if (d_status) { // fold every other part's status word into *d_status (home)
            std::vector<DevBuf> tmp(W);
            for (uint32_t p = 1; p < W; ++p) {
                if (!bs[p].p)
                    continue;
                tmp[p] = DevBuf(sizeof(uint32_t), st);
                CK(cudaMemcpyPeerAsync(tmp[p].p, home, bs[p].p, ix->parts[p]->device, sizeof(uint32_t), st));
                group_status_or_kernel<<<1, 1, 0, st>>>(tmp[p].as<uint32_t>(), d_status);
                CK(cudaGetLastError());
            }
        }
        for (uint32_t p = 1; p < W; ++p) // part buffers are freed on their streams after the copies
            order_after(st, home, sts[p], ix->parts[p]->device);
        return TRIM_OK;
    }
    // ---- id shards
    const uint64_t nres = nq * k;
    // gathered per-part results on every part's device ([W][nq][k], [W][nq][6]);
    // only the home device's copy is merged
    std::vector<DevBuf> bq(W), bi(W), bd(W), bc(W), gi(W), gd(W), gc(W);
    std::vector<cudaStream_t> sts(W);
    for (uint32_t p = 0; p < W; ++p) {
        const int dv = ix->parts[p]->device;
        sts[p] = thread_stream(dv);
        order_after(st, home, sts[p], dv); // the queries (and output buffers) are ready on `stream`
    }
    for (uint32_t p = 0; p < W; ++p) {
        DeviceGuard g(ix->parts[p]->device);
        cudaStream_t s = sts[p];
        bq[p] = DevBuf(sizeof(float) * nq * ds, s);
        bi[p] = DevBuf(sizeof(uint32_t) * nres, s);
        bd[p] = DevBuf(sizeof(float) * nres, s);
        bc[p] = DevBuf(sizeof(unsigned long long) * nq * 6, s);
        if (ix->nccl || p == 0) {
            gi[p] = DevBuf(sizeof(uint32_t) * nres * W, s);
            gd[p] = DevBuf(sizeof(float) * nres * W, s);
            gc[p] = DevBuf(sizeof(unsigned long long) * nq * 6 * W, s);
        }
    }
    // 1. the query batch to every part: NCCL broadcast from the home rank, or copies
    if (ix->nccl) {
        std::lock_guard<std::mutex> lk(ix->nccl->mu);
        NK(nccl().group_start());
        for (uint32_t p = 0; p < W; ++p)
            NK(nccl().broadcast(p == 0 ? q : nullptr, bq[p].p, nq * ds, ncclFloat32, 0, ix->nccl->comms[p], sts[p]));
        NK(nccl().group_end());
    } else {
        for (uint32_t p = 0; p < W; ++p) {
            DeviceGuard g(ix->parts[p]->device);
            CK(cudaMemcpyPeerAsync(bq[p].p, ix->parts[p]->device, q, home, sizeof(float) * nq * ds, sts[p]));
        }
    }
    // 2. every part's filter over its sub-stream of each query
    for (uint32_t p = 0; p < W; ++p) {
        DeviceGuard g(ix->parts[p]->device);
        if (int rc = knn_device(ix->parts[p], bq[p].as<float>(), nq, k, nprobe, gamma, bi[p].as<uint32_t>(),
                                bd[p].as<float>(), bc[p].as<unsigned long long>(), nullptr, sts[p]))
            return rc;
    }
    // 3. the exchange: all-gather of the per-part top-k and counters
    if (ix->nccl) {
        std::lock_guard<std::mutex> lk(ix->nccl->mu);
        NK(nccl().group_start());
        for (uint32_t p = 0; p < W; ++p) {
            NK(nccl().all_gather(bi[p].p, gi[p].p, nres, ncclUint32, ix->nccl->comms[p], sts[p]));
            NK(nccl().all_gather(bd[p].p, gd[p].p, nres, ncclFloat32, ix->nccl->comms[p], sts[p]));
            NK(nccl().all_gather(bc[p].p, gc[p].p, nq * 6, ncclUint64, ix->nccl->comms[p], sts[p]));
        }
        NK(nccl().group_end());
    } else {
        for (uint32_t p = 0; p < W; ++p) {
            const int dv = ix->parts[p]->device;
            DeviceGuard g(dv);
            CK(cudaMemcpyPeerAsync(gi[0].as<uint32_t>() + p * nres, home, bi[p].p, dv, sizeof(uint32_t) * nres, sts[p]));
            CK(cudaMemcpyPeerAsync(gd[0].as<float>() + p * nres, home, bd[p].p, dv, sizeof(float) * nres, sts[p]));
            CK(cudaMemcpyPeerAsync(gc[0].as<unsigned long long>() + p * nq * 6, home, bc[p].p, dv,
                                   sizeof(unsigned long long) * nq * 6, sts[p]));
        }
    }
    // 4. merge on the home device, ordered on the caller's stream
    for (uint32_t p = 0; p < W; ++p)
        order_after(sts[p], ix->parts[p]->device, st, home);
    if (int rc = trim_merge_topk_device(gd[0].as<float>(), gi[0].as<uint32_t>(), W, nq, k, d_dist, d_ids, home, st))
        return rc;
    group_counters_kernel<<<static_cast<unsigned>((nq + 255) / 256), 256, 0, st>>>(
        gc[0].as<unsigned long long>(), W, nq, k, reinterpret_cast<unsigned long long*>(d_counters), d_status);
    CK(cudaGetLastError());
    // the per-part buffers are freed on their streams after the exchange; the
    // home gather buffers must outlive the merge on `stream`
    for (uint32_t p = 0; p < W; ++p)
        order_after(st, home, sts[p], ix->parts[p]->device);
    return TRIM_OK;
}

namespace {

// Replicas, host API: part p searches its contiguous query slice on its own
// device (its own H2D / D2H, concurrently: one host thread per extra part).
template <typename Fn>
int run_slices(const trim_index* ix, uint64_t nq, Fn&& fn) {
    const uint32_t W = parts_of(ix);
    std::vector<int> rc(W, TRIM_OK);
    std::vector<std::string> err(W);
    std::vector<std::thread> th;
    for (uint32_t p = 1; p < W; ++p)
        th.emplace_back([&, p] {
            uint64_t lo, n;
            slice_of(nq, p, W, lo, n);
            rc[p] = n ? fn(ix->parts[p], lo, n) : TRIM_OK;
            if (rc[p])
                err[p] = trim_last_error();
        });
    uint64_t lo, n;
    slice_of(nq, 0, W, lo, n);
    rc[0] = n ? fn(ix->parts[0], lo, n) : TRIM_OK;
    if (rc[0])
        err[0] = trim_last_error();
    for (auto& t : th)
        t.join();
    for (uint32_t p = 0; p < W; ++p)
        if (rc[p])
            return set_err(rc[p], "%s", err[p].c_str());
    return TRIM_OK;
}

} // namespace

int trimhost::group_search_knn(trim_index* ix, const float* queries, uint64_t nq, uint32_t k, uint32_t nprobe,
                               float gamma, uint32_t* ids_out, float* dist_out, trim_counters* counters_out) {
    const uint32_t dim = ix->dev.dim;
    if (ix->shard_mode == TRIM_SHARD_REPLICAS)
        return run_slices(ix, nq, [&](trim_index* part, uint64_t lo, uint64_t n) {
            return trim_search_knn(part, queries + lo * dim, n, k, nprobe, gamma, ids_out + lo * k, dist_out + lo * k,
                                   counters_out ? counters_out + lo : nullptr);
        });
    // id shards: the batch goes to the home device; the device path broadcasts,
    // filters on every part, all-gathers and merges
    const int home = ix->device;
    DeviceGuard g(home);
    cudaStream_t st = thread_stream(home);
    DevBuf d_q(sizeof(float) * nq * dim, st);
    CK(cudaMemcpyAsync(d_q.p, queries, sizeof(float) * nq * dim, cudaMemcpyHostToDevice, st));
    DevBuf d_ids(sizeof(uint32_t) * nq * k, st), d_dist(sizeof(float) * nq * k, st),
        d_ct(sizeof(trim_counters) * nq, st), d_status(sizeof(uint32_t), st);
    CK(cudaMemsetAsync(d_status.p, 0, sizeof(uint32_t), st));
    if (int rc = group_search_knn_device(ix, d_q.as<float>(), nq, k, nprobe, gamma, d_ids.as<uint32_t>(),
                                         d_dist.as<float>(), d_ct.as<trim_counters>(), d_status.as<uint32_t>(), st))
        return rc;
    uint32_t* status_h = pinned_word();
    CK(cudaMemcpyAsync(ids_out, d_ids.p, sizeof(uint32_t) * nq * k, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(dist_out, d_dist.p, sizeof(float) * nq * k, cudaMemcpyDeviceToHost, st));
    if (counters_out)
        CK(cudaMemcpyAsync(counters_out, d_ct.p, sizeof(trim_counters) * nq, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(status_h, d_status.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (*status_h & 1u)
        return set_err(TRIM_EINVAL, "search_trim_ivf_knn: k exceeds probed vectors");
    return TRIM_OK;
}

// ------------------------------------------------------------------ range
int trimhost::group_search_range(trim_index* ix, const float* queries, uint64_t nq, const float* radius,
                                 uint32_t nprobe, float gamma, uint64_t* offsets_out, uint32_t** ids_out,
                                 float** dist_out, trim_counters* counters_out) {
    const uint32_t W = parts_of(ix), dim = ix->dev.dim;
    if (ix->shard_mode == TRIM_SHARD_REPLICAS) {
        // every slice through the single-device host call, then concatenated
        std::vector<std::vector<uint64_t>> offs(W);
        std::vector<uint32_t*> pid(W, nullptr);
        std::vector<float*> pd(W, nullptr);
        auto release = [&] {
            for (uint32_t p = 0; p < W; ++p) {
                std::free(pid[p]);
                std::free(pd[p]);
            }
        };
        for (uint32_t p = 0; p < W; ++p) {
            uint64_t lo, n;
            slice_of(nq, p, W, lo, n);
            offs[p].assign(n + 1, 0);
        }
        const int rc = run_slices(ix, nq, [&](trim_index* part, uint64_t lo, uint64_t n) {
            uint32_t p = 0;
            while (ix->parts[p] != part)
                ++p;
            return trim_search_range(part, queries + lo * dim, n, radius + lo, nprobe, gamma, offs[p].data(), &pid[p],
                                     &pd[p], counters_out ? counters_out + lo : nullptr);
        });
        if (rc) {
            release();
            return rc;
        }
        uint64_t tot = 0;
        for (uint32_t p = 0; p < W; ++p)
            tot += offs[p].back();
        auto* hid = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * std::max<uint64_t>(tot, 1)));
        auto* hd = static_cast<float*>(std::malloc(sizeof(float) * std::max<uint64_t>(tot, 1)));
        if (!hid || !hd) {
            std::free(hid);
            std::free(hd);
            release();
            return set_err(TRIM_ENOMEM, "search_trim_ivf_range: result allocation failed");
        }
        uint64_t base = 0;
        for (uint32_t p = 0; p < W; ++p) {
            uint64_t lo, n;
            slice_of(nq, p, W, lo, n);
            for (uint64_t i = 0; i < n; ++i)
                offsets_out[lo + i] = base + offs[p][i];
            const uint64_t c = offs[p].back();
            if (c) {
                std::memcpy(hid + base, pid[p], sizeof(uint32_t) * c);
                std::memcpy(hd + base, pd[p], sizeof(float) * c);
            }
            base += c;
        }
        offsets_out[nq] = base;
        release();
        *ids_out = hid;
        *dist_out = hd;
        return TRIM_OK;
    }
    // ---- id shards: the union of the parts' member sets is the single run's
    // (the range filter has no running state, ivf.hpp:323-340)
    const int home = ix->device;
    std::vector<float> r2(nq);
    for (uint64_t i = 0; i < nq; ++i)
        r2[i] = radius[i] * radius[i]; // ivf.hpp:315, fp32
    std::vector<cudaStream_t> sts(W);
    std::vector<DevBuf> bq(W), br(W), bprobe(W), bk(W), bc(W), bdc(W), bev(W);
    std::vector<uint32_t> npv(W, 0);
    for (uint32_t p = 0; p < W; ++p) {
        const trim_index* pt = ix->parts[p];
        DeviceGuard g(pt->device);
        sts[p] = thread_stream(pt->device);
        bq[p] = upload_queries(pt, queries, nq, cudaMemcpyHostToDevice, sts[p]);
        br[p] = DevBuf(sizeof(float) * nq, sts[p]);
        CK(cudaMemcpyAsync(br[p].p, r2.data(), sizeof(float) * nq, cudaMemcpyHostToDevice, sts[p]));
        npv[p] = run_probe(pt, bq[p].as<float>(), nq, nprobe, bprobe[p], sts[p]);
        bc[p] = DevBuf(sizeof(unsigned int) * nq, sts[p]);
        bdc[p] = DevBuf(sizeof(unsigned long long) * nq, sts[p]);
        bev[p] = DevBuf(sizeof(unsigned long long) * nq, sts[p]);
    }
    uint32_t cap = 1024;
    std::vector<std::vector<unsigned int>> cnt(W, std::vector<unsigned int>(nq));
    for (int attempt = 0; attempt < 2; ++attempt) {
        for (uint32_t p = 0; p < W; ++p) {
            const trim_index* pt = ix->parts[p];
            DeviceGuard g(pt->device);
            cudaStream_t s = sts[p];
            bk[p] = DevBuf(sizeof(unsigned long long) * nq * cap, s);
            CK(cudaMemsetAsync(bc[p].p, 0, sizeof(unsigned int) * nq, s));
            CK(cudaMemsetAsync(bdc[p].p, 0, sizeof(unsigned long long) * nq, s));
            CK(cudaMemsetAsync(bev[p].p, 0, sizeof(unsigned long long) * nq, s));
            range_launch(pt, bq[p].as<float>(), nq, br[p].as<float>(), npv[p],
                         bprobe[p].p ? bprobe[p].as<uint32_t>() : nullptr, gamma, cap,
                         bk[p].as<unsigned long long>(), bc[p].as<unsigned int>(), bdc[p].as<unsigned long long>(),
                         bev[p].as<unsigned long long>(), s);
            CK(cudaMemcpyAsync(cnt[p].data(), bc[p].p, sizeof(unsigned int) * nq, cudaMemcpyDeviceToHost, s));
        }
        unsigned int mx = 0;
        for (uint32_t p = 0; p < W; ++p) {
            DeviceGuard g(ix->parts[p]->device);
            CK(cudaStreamSynchronize(sts[p]));
            for (unsigned int c : cnt[p])
                mx = std::max(mx, c);
        }
        if (mx <= cap)
            break;
        cap = mx; // the exact size: the second run cannot overflow
    }
    // counters: per-query sums over the parts (read back; the host API syncs anyway)
    std::vector<unsigned long long> dc(nq, 0), ev(nq, 0), tmp(nq);
    for (uint32_t p = 0; p < W; ++p) {
        DeviceGuard g(ix->parts[p]->device);
        CK(cudaMemcpy(tmp.data(), bdc[p].p, sizeof(unsigned long long) * nq, cudaMemcpyDeviceToHost));
        for (uint64_t i = 0; i < nq; ++i)
            dc[i] += tmp[i];
        CK(cudaMemcpy(tmp.data(), bev[p].p, sizeof(unsigned long long) * nq, cudaMemcpyDeviceToHost));
        for (uint64_t i = 0; i < nq; ++i)
            ev[i] += tmp[i];
    }
    // the exchange: every part's member keys and counts to the home device
    DeviceGuard gh(home);
    cudaStream_t st = sts[0];
    const uint64_t per = nq * cap;
    std::vector<DevBuf> gk(W), gc(W);
    for (uint32_t p = 0; p < W; ++p) {
        if (!ix->nccl && p)
            continue;
        DeviceGuard g(ix->parts[p]->device);
        gk[p] = DevBuf(sizeof(unsigned long long) * per * W, sts[p]);
        gc[p] = DevBuf(sizeof(unsigned int) * nq * W, sts[p]);
    }
    if (ix->nccl) {
        std::lock_guard<std::mutex> lk(ix->nccl->mu);
        NK(nccl().group_start());
        for (uint32_t p = 0; p < W; ++p) {
            NK(nccl().all_gather(bk[p].p, gk[p].p, per, ncclUint64, ix->nccl->comms[p], sts[p]));
            NK(nccl().all_gather(bc[p].p, gc[p].p, nq, ncclUint32, ix->nccl->comms[p], sts[p]));
        }
        NK(nccl().group_end());
    } else {
        for (uint32_t p = 0; p < W; ++p) {
            const int dv = ix->parts[p]->device;
            DeviceGuard g(dv);
            CK(cudaMemcpyPeerAsync(gk[0].as<unsigned long long>() + p * per, home, bk[p].p, dv,
                                   sizeof(unsigned long long) * per, sts[p]));
            CK(cudaMemcpyPeerAsync(gc[0].as<unsigned int>() + p * nq, home, bc[p].p, dv, sizeof(unsigned int) * nq,
                                   sts[p]));
        }
    }
    for (uint32_t p = 1; p < W; ++p)
        order_after(sts[p], ix->parts[p]->device, st, home);
    // per-query sort by (dist, id) of the union (ivf.hpp:341), on the home device
    uint64_t tot = 0;
    offsets_out[0] = 0;
    for (uint64_t i = 0; i < nq; ++i) {
        uint64_t c = 0;
        for (uint32_t p = 0; p < W; ++p)
            c += cnt[p][i];
        offsets_out[i] = tot;
        tot += c;
    }
    offsets_out[nq] = tot;
    DevBuf d_cat(sizeof(unsigned long long) * per * W, st), d_sorted(sizeof(unsigned long long) * per * W, st),
        d_beg(sizeof(uint64_t) * nq, st), d_end(sizeof(uint64_t) * nq, st), d_offs(sizeof(uint64_t) * (nq + 1), st);
    group_range_compact_kernel<<<static_cast<unsigned>(nq), 128, 0, st>>>(
        gk[0].as<unsigned long long>(), gc[0].as<unsigned int>(), W, nq, cap, d_cat.as<unsigned long long>(),
        d_beg.as<uint64_t>(), d_end.as<uint64_t>());
    CK(cudaGetLastError());
    size_t tmp_bytes = 0;
    CK(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp_bytes, d_cat.as<unsigned long long>(),
                                          d_sorted.as<unsigned long long>(), static_cast<int64_t>(per * W),
                                          static_cast<int64_t>(nq), d_beg.as<uint64_t>(), d_end.as<uint64_t>(), st));
    DevBuf d_tmp(tmp_bytes, st);
    CK(cub::DeviceSegmentedSort::SortKeys(d_tmp.p, tmp_bytes, d_cat.as<unsigned long long>(),
                                          d_sorted.as<unsigned long long>(), static_cast<int64_t>(per * W),
                                          static_cast<int64_t>(nq), d_beg.as<uint64_t>(), d_end.as<uint64_t>(), st));
    CK(cudaMemcpyAsync(d_offs.p, offsets_out, sizeof(uint64_t) * (nq + 1), cudaMemcpyHostToDevice, st));
    DevBuf d_ids(sizeof(uint32_t) * std::max<uint64_t>(tot, 1), st), d_dist(sizeof(float) * std::max<uint64_t>(tot, 1), st);
    group_range_unpack_kernel<<<static_cast<unsigned>(nq), 128, 0, st>>>(
        d_sorted.as<unsigned long long>(), W, cap, d_offs.as<uint64_t>(), nq, d_ids.as<uint32_t>(), d_dist.as<float>());
    CK(cudaGetLastError());
    auto* hid = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * std::max<uint64_t>(tot, 1)));
    auto* hd = static_cast<float*>(std::malloc(sizeof(float) * std::max<uint64_t>(tot, 1)));
    if (!hid || !hd) {
        std::free(hid);
        std::free(hd);
        return set_err(TRIM_ENOMEM, "search_trim_ivf_range: result allocation failed");
    }
    cudaError_t e1 = cudaMemcpyAsync(hid, d_ids.p, sizeof(uint32_t) * tot, cudaMemcpyDeviceToHost, st);
    cudaError_t e2 = cudaMemcpyAsync(hd, d_dist.p, sizeof(float) * tot, cudaMemcpyDeviceToHost, st);
    cudaError_t e3 = cudaStreamSynchronize(st);
    if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
        std::free(hid);
        std::free(hd);
        CK(e1 != cudaSuccess ? e1 : (e2 != cudaSuccess ? e2 : e3));
    }
    for (uint32_t p = 1; p < W; ++p) // part buffers are released after the exchange
        order_after(st, home, sts[p], ix->parts[p]->device);
    if (counters_out)
        for (uint64_t i = 0; i < nq; ++i) {
            trim_counters& c = counters_out[i];
            c.evaluated = ev[i];
            c.edc = ev[i];
            c.dc = dc[i];
            c.pruned = ev[i] - dc[i];
            c.hops = 0;
            c.coarse_dc = ix->dev.nlist;
        }
    *ids_out = hid;
    *dist_out = hd;
    return TRIM_OK;
}

// ------------------------------------------------------------------ IVFPQ baseline
int trimhost::group_search_baseline(trim_index* ix, const float* queries, uint64_t nq, uint32_t k, uint32_t nprobe,
                                    uint32_t k_prime, uint32_t* ids_out, float* dist_out,
                                    trim_counters* counters_out) {
    if (ix->shard_mode != TRIM_SHARD_REPLICAS)
        return set_err(TRIM_EINVAL, "search_baseline_ivfpq: the refine pool (k' smallest ADC estimates over the "
                                    "whole probed stream, ivf.hpp:205-215) needs a single or replicas index");
    const uint32_t dim = ix->dev.dim;
    return run_slices(ix, nq, [&](trim_index* part, uint64_t lo, uint64_t n) {
        return trim_search_baseline_ivfpq(part, queries + lo * dim, n, k, nprobe, k_prime, ids_out + lo * k,
                                          dist_out + lo * k, counters_out ? counters_out + lo : nullptr);
    });
}
