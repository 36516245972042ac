/*
 * trim_gpu.h — C ABI of the B200-native TRIM candidate filter.
 *
 * This is the drop-in boundary for the reference's query path. The reference
 * has no FFI; its boundary is the header-level C++ API in
 * proj/include/trimsearch/ivf/ivf.hpp. Each entry point below names the
 * reference function it replaces (file:line relative to
 * /root/reference/proj/include/trimsearch). The reference functions take
 * one query; these take a batch, because a GPU launch per query is too small.
 * The C++ header include/trim_b200/ivf.hpp re-exposes the reference's
 * per-query signatures and exceptions on top of this ABI.
 *
 * There is no CPU fallback. If no CUDA device is present, or the library was
 * built without sm_100a code, every search returns TRIM_ECUDA.
 *
 * Threading: an index is immutable after trim_index_create. Concurrent
 * searches on one index from several host threads are safe: every call uses
 * its own stream and its own stream-ordered workspace.
 *
 * Errors: functions return trim_status. The message of the last failure on
 * the calling thread is available from trim_last_error(). The codes map 1:1
 * to the reference exceptions:
 *   TRIM_EINVAL -> std::invalid_argument
 *   TRIM_EDATA  -> trimsearch::DataError (core/io_util.hpp:13-16)
 */
#ifndef TRIM_GPU_H
#define TRIM_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TRIM_ABI_VERSION 3

typedef enum {
    TRIM_OK = 0,
    TRIM_EINVAL = 1, /* std::invalid_argument in the reference */
    TRIM_EDATA = 2,  /* trimsearch::DataError */
    TRIM_ECUDA = 3,  /* CUDA runtime / launch failure, or no device */
    TRIM_ENCCL = 4,  /* NCCL failure in a multi-device (id_shard) index */
    TRIM_ENOMEM = 5
} trim_status;

/* trimsearch::SearchCounters (core/counters.hpp:10-16), followed by
 * IvfResult::coarse_dc (ivf/ivf.hpp:164-169). */
typedef struct {
    uint64_t dc;
    uint64_t edc;
    uint64_t pruned;
    uint64_t evaluated;
    uint64_t hops;
    uint64_t coarse_dc;
} trim_counters;

typedef enum {
    TRIM_MEM_HOST = 0,  /* descriptor arrays are host pointers */
    TRIM_MEM_DEVICE = 1 /* descriptor arrays are device pointers on `device` */
} trim_memory;

/* Multi-device layouts. */
typedef enum {
    TRIM_SHARD_SINGLE = 0,   /* one device: `device` */
    TRIM_SHARD_ID = 1,       /* the rows split by id over devices[]: device p holds ids
                                [p*n/W, (p+1)*n/W) (per list, that sub-range of the list);
                                codebook + coarse quantizer replicated. A search runs every
                                shard's filter on its sub-stream of each query, then the
                                per-shard top-k (dist, id) are all-gathered (ncclAllGather over
                                NVLink; device-to-device copies when entries of devices[]
                                repeat, e.g. W shards on one GPU) and merged by (dist, id). */
    TRIM_SHARD_REPLICAS = 2  /* the whole index on every device; a batch's queries split into
                                contiguous slices, one per device; no collective */
} trim_shard_mode;

/*
 * Index descriptor: trimsearch::ivf::IvfIndex (ivf/ivf.hpp:37-51) flattened to
 * CSR, plus the VectorDataset (core/dataset.hpp:18-27) the survivors are read
 * from. trim_index_create copies everything; the caller keeps ownership.
 *
 *   centroids    PqCodebook::centroids, subspace j at float ksub*sub_off[j],
 *                where sub_off is the prefix sum of sub_dims (pq/pq.hpp:40-54)
 *   coarse       IvfIndex::coarse_centroids, nlist*dim
 *   list_*       InvertedList arrays (ivf/ivf.hpp:29-35) concatenated in list
 *                order; list l is [list_offsets[l], list_offsets[l+1]);
 *                entries within a list in ascending id order (ivf.hpp:147-152)
 *   vectors      rows for ids [id_base, id_base + n); an id-shard of the
 *                dataset when id_base != 0 (multi-GPU)
 */
typedef struct {
    uint32_t dim;
    uint32_t m;
    uint32_t ksub; /* centroids per subspace, <= 256 (byte codes, pq.hpp:27-29) */
    const uint32_t* sub_dims;
    const float* centroids;
    uint32_t nlist;
    const float* coarse;
    const uint64_t* list_offsets;
    const uint32_t* list_ids;
    const uint8_t* list_codes;
    uint32_t code_stride; /* bytes between consecutive codes, >= m */
    const float* list_lx; /* plain (non-squared) Γ(l,x) */
    uint64_t n;
    const float* vectors;
    uint64_t id_base;
    int device;
    trim_memory memory;
    /* ABI 3: multi-device layout. ndevices == 0 (or shard_mode SINGLE): one
     * device, `device`. Otherwise devices[0..ndevices) (entries may repeat) and
     * `device` is ignored; the descriptor holds the WHOLE index (id_base 0, host
     * memory, or device memory on devices[0]); results are returned as for one
     * index. Per-query counters of an id_shard search are the shards' sums
     * (coarse_dc: nlist, the probe runs once per query as in the reference). */
    const int* devices;
    uint32_t ndevices;
    trim_shard_mode shard_mode;
} trim_index_desc;

typedef struct trim_index* trim_index_t;

typedef struct {
    uint32_t dim, m, ksub, nlist;
    uint64_t n, total_entries, id_base;
    uint64_t max_list_size;
    uint64_t device_bytes;     /* summed over the devices of a multi-device index */
    int device;                /* the (home) device */
    uint32_t range_query_tile; /* queries sharing one code stream in the flat range scan */
    uint32_t ndevices;         /* 1 for a single-device index */
    uint32_t shard_mode;       /* trim_shard_mode */
    uint32_t nccl;             /* 1: the id_shard exchange runs over NCCL */
} trim_index_info;

const char* trim_last_error(void);
int trim_abi_version(void);

/* IvfIndex construction from prebuilt arrays (the reference builds on host:
 * ivf/ivf.hpp:112-154; its artefact format is ivf.hpp:53-107). */
int trim_index_create(const trim_index_desc* desc, trim_index_t* out);
int trim_index_destroy(trim_index_t index);
int trim_index_get_info(trim_index_t index, trim_index_info* info);
/* Diagnostic (no reference equivalent): stream positions the kNN kernel pruned
 * as whole lists by the list-level bound (and, for flat range search, rows
 * pruned as whole blocks of the block partition) since creation or the last reset
 * (they are counted as pruned in trim_counters, exactly as the reference
 * prunes them one by one). Synchronises the index's device. */
int trim_index_skip_stats(trim_index_t index, uint64_t* skipped_positions, int reset);
/* Kernels trim_probe / trim_probe_device launch per call at this nprobe
 * (2 on the tensor-core path: distance bounds + select; 1 otherwise; 0 when
 * nlist == 1). For launch accounting. */
int trim_probe_launches(trim_index_t index, uint32_t nprobe, uint32_t* launches);

/*
 * ivf::search_trim_ivf_knn (ivf/ivf.hpp:243-304), for nq queries.
 * queries: nq*dim (host). ids_out/dist_out: nq*k (host), each row ascending by
 * (dist_sq, id). counters_out: nq (host, may be NULL).
 * gamma is float(profile.gamma) (ivf.hpp:250); gamma < 0 is an uncalibrated
 * profile (ivf.hpp:246-247). k > probed vectors of any query -> TRIM_EINVAL
 * (ivf.hpp:289-290). k <= 4096 (k > 256: a shared-memory top-k in the
 * runtime-(m, ksub) kernel).
 */
int trim_search_knn(trim_index_t index, const float* queries, uint64_t nq, uint32_t k,
                    uint32_t nprobe, float gamma, uint32_t* ids_out, float* dist_out,
                    trim_counters* counters_out);

/*
 * ivf::search_trim_ivf_range (ivf/ivf.hpp:308-347). radius: nq plain radii.
 * offsets_out: nq+1 (host). *ids_out / *dist_out are allocated by the library
 * (release with trim_free) and hold the concatenated per-query results, each
 * query ascending by (dist_sq, id). Negative radius -> TRIM_EINVAL.
 */
int trim_search_range(trim_index_t index, const float* queries, uint64_t nq,
                      const float* radius, uint32_t nprobe, float gamma, uint64_t* offsets_out,
                      uint32_t** ids_out, float** dist_out, trim_counters* counters_out);

/*
 * ivf::search_baseline_ivfpq (ivf/ivf.hpp:193-237): two-phase IVFPQ with a
 * refine pool of k_prime. ids_out/dist_out: nq*k. Requires 1 <= k <= k_prime,
 * nprobe >= 1; k > probed -> TRIM_EINVAL.
 */
int trim_search_baseline_ivfpq(trim_index_t index, const float* queries, uint64_t nq,
                               uint32_t k, uint32_t nprobe, uint32_t k_prime, uint32_t* ids_out,
                               float* dist_out, trim_counters* counters_out);

/*
 * Device-resident variants (inputs already in HBM; used by the serving loop
 * and bench.py's device-timed leg). All pointers are device pointers on the
 * index's device; the call is asynchronous on `stream` (a cudaStream_t, NULL =
 * per-thread default). A query whose probed stream is shorter than k sets bit
 * 0 of *status_out (device u32, may be NULL); its row holds the partial top-k
 * (every entry of the stream, ascending (dist, id)) padded with
 * (+inf, 0xFFFFFFFF). For a multi-device index the pointers are on its home
 * device (devices[0]) and `stream` is a home-device stream: the library moves
 * the queries to the other devices and the results back itself (id_shard:
 * NCCL broadcast / all-gather), ordered after / before the work on `stream`.
 */
int trim_search_knn_device(trim_index_t index, const float* d_queries, uint64_t nq, uint32_t k,
                           uint32_t nprobe, float gamma, uint32_t* d_ids, float* d_dist,
                           trim_counters* d_counters, uint32_t* d_status, void* stream);

/* The two stages of trim_search_knn_device, separately (device pointers, async):
 * probe_order into d_lists (nq*min(nprobe,nlist)), then the fused filter over
 * those lists (like FAISS's search_preassigned). dim must be a multiple of 4. */
int trim_probe_device(trim_index_t index, const float* d_queries, uint64_t nq, uint32_t nprobe,
                      uint32_t* d_lists, void* stream);
int trim_search_knn_preassigned_device(trim_index_t index, const float* d_queries, uint64_t nq,
                                       uint32_t k, const uint32_t* d_lists, uint32_t np,
                                       float gamma, uint32_t* d_ids, float* d_dist,
                                       trim_counters* d_counters, uint32_t* d_status,
                                       void* stream);

/* ivf::search_trim_ivf_range (ivf/ivf.hpp:308-347), device-resident. d_queries
 * nq*dim, d_radius nq (device). Query i's members, sorted by (dist_sq, id) like
 * ivf.hpp:341, are d_ids/d_dist[i*cap .. i*cap + min(count, cap)); d_counts[i]
 * = the true member count. Bit 0 of *d_status: some query had more than cap
 * members (its slots then hold an arbitrary sorted subset of cap of them: call
 * again with cap >= max count); bit 1: some
 * radius was negative (the host API's TRIM_EINVAL; that query returns nothing).
 * dim must be a multiple of 4. */
int trim_search_range_device(trim_index_t index, const float* d_queries, uint64_t nq,
                             const float* d_radius, uint32_t nprobe, float gamma, uint32_t cap,
                             uint32_t* d_counts, uint32_t* d_ids, float* d_dist,
                             trim_counters* d_counters, uint32_t* d_status, void* stream);

/* core/ground_truth.hpp ground_truth_knn (:97-113, brute_force_knn :53-74): the
 * exact k nearest rows of every query over the index's vectors, ascending by
 * (dist_sq, id), bit-identical to the reference (fp32 4-accumulator distances).
 * queries nq*dim (host); ids_out/dist_out nq*k (host). 1 <= k <= min(n, 4096). */
int trim_ground_truth_knn(trim_index_t index, const float* queries, uint64_t nq, uint32_t k,
                          uint32_t* ids_out, float* dist_out);

/* pq::build_distance_table (pq/pq.hpp:158-172) for nq queries: lut_out is
 * nq*m*ksub floats (host), j-major like DistanceTable::entries. */
int trim_build_lut(trim_index_t index, const float* queries, uint64_t nq, float* lut_out);

/* detail_ivf::probe_order (ivf/ivf.hpp:173-187): lists_out nq*min(nprobe,nlist). */
int trim_probe(trim_index_t index, const float* queries, uint64_t nq, uint32_t nprobe,
               uint32_t* lists_out);

/*
 * Merge of per-shard top-k lists (multi-GPU id-sharding, after the NCCL
 * all-gather). d_dist/d_ids: [nshards][nq][k] device arrays; the merged row
 * is the k smallest (dist_sq, id) — the same order ScoredId defines
 * (core/ground_truth.hpp:39-50). Entries with id 0xFFFFFFFF are ignored.
 */
int trim_merge_topk_device(const float* d_dist, const uint32_t* d_ids, uint32_t nshards,
                           uint64_t nq, uint32_t k, float* d_dist_out, uint32_t* d_ids_out,
                           int device, void* stream);

void trim_free(void* p);

/* ------------------------------------------------------------------------
 * Device-side index build. The reference builds on host
 * threads; these are its B200 equivalents. All d_* pointers are device
 * memory on `device`; `stream` is a cudaStream_t (NULL = default).
 * ------------------------------------------------------------------------ */

/* Seeded N(0,1) rows (the role of make_normal_dataset, core/synthetic.hpp:11-18;
 * Philox4x32-10 + Box-Muller, not libstdc++'s generator). */
int trim_synth_normal_device(uint64_t n, uint32_t dim, uint64_t seed, float* d_out, int device,
                             void* stream);
/* Gaussian blobs, row i around center i % nc (make_blob_dataset,
 * core/synthetic.hpp:21-33). */
int trim_synth_blobs_device(const float* d_centers, uint64_t nc, uint32_t dim, uint64_t n,
                            float sigma, uint64_t seed, float* d_out, int device, void* stream);
/* Uniform [0,1) rows, optionally L2-normalised (dataset.hpp:44-56). */
int trim_synth_uniform_device(uint64_t n, uint32_t dim, uint64_t seed, int normalize,
                              float* d_out, int device, void* stream);
/* The reference's seeded row sampler (pq/pq.hpp:72-80, ivf/ivf.hpp:121-126);
 * host only. The caller xors the reference's seed constant in. */
int trim_sample_rows(uint64_t n, uint64_t sample_n, uint64_t seed, uint64_t* rows_out);
/* detail::nearest_centroid for n rows (pq/kmeans.hpp:27-41): exact fp32
 * arithmetic, ties to the lowest index. d_dist may be NULL. */
int trim_assign_device(const float* d_x, uint64_t n, uint32_t dim, const float* d_cent,
                       uint32_t k, uint32_t* d_assign, float* d_dist, int device, void* stream);
/* k-means (pq/kmeans.hpp:89-158 structure: k-means++ seeding, Lloyd steps,
 * empty-cluster repair). Synchronous. */
int trim_kmeans_device(const float* d_x, uint64_t n, uint32_t dim, uint32_t k, uint32_t iters,
                       uint64_t seed, float* d_centroids, int device);
/* pq::train (pq/pq.hpp:65-113). sub_dims_out: host, m entries.
 * d_centroids_out: ksub*dim floats in the trim_index_desc layout. */
int trim_pq_train_device(const float* d_x, uint64_t n, uint32_t dim, uint32_t m, uint32_t ksub,
                         uint32_t iters, uint64_t seed, uint64_t train_sample,
                         uint32_t* sub_dims_out, float* d_centroids_out, int device);
/* pq::encode for every row + Γ(l,x) (trim/landmarks.hpp:57-72), bit-exact.
 * sub_dims: host. d_lx may be NULL. Synchronous. */
int trim_pq_encode_device(const float* d_x, uint64_t n, uint32_t dim, uint32_t m, uint32_t ksub,
                          const uint32_t* sub_dims, const float* d_centroids, uint8_t* d_codes,
                          uint32_t code_stride, float* d_lx, int device, void* stream);
/* Inverted lists from list assignments (ivf/ivf.hpp:145-152): d_ids holds
 * the row ids grouped by list, ascending within a list; d_offsets nlist+1. */
int trim_ivf_lists_device(const uint32_t* d_assign, uint64_t n, uint32_t nlist,
                          uint64_t* d_offsets, uint32_t* d_ids, int device, void* stream);

/* ------------------------------------------------------------------------
 * TRIM filter over an HNSW graph: the per-hop
 * neighbour filter of graph::search_trim_knn / search_trim_range
 * (graph/search.hpp:188-347), batched over queries (one warp per query).
 * ------------------------------------------------------------------------ */

/*
 * graph::GraphIndex (graph/hnsw.hpp:22-35) as per-level CSR, with the
 * trim::LandmarkStore (trim/landmarks.hpp:18-28) and VectorDataset it is
 * searched with. trim_graph_create copies everything (host or device arrays
 * per `memory`); the caller keeps ownership.
 *   offsets   levels x (n+1): node i's level-l list is
 *             nbrs[nbr_base[l] + offsets[l*(n+1)+i] .. + offsets[l*(n+1)+i+1])
 *   codes     n x code_stride landmark codes (LandmarkStore::codes, by node id)
 *   lx        n plain Γ(l,x) (LandmarkStore::lx_dist)
 *   centroids the codebook, trim_index_desc layout
 * lm.count != ds.count (search.hpp:198-199) cannot arise: both are n.
 */
typedef struct {
    uint64_t n;
    uint32_t dim;
    uint32_t m;
    uint32_t ksub;
    const uint32_t* sub_dims;
    const float* centroids;
    const uint8_t* codes;
    uint32_t code_stride;
    const float* lx;
    const float* vectors;
    uint32_t levels; /* GraphIndex::max_level + 1 */
    uint32_t entry;  /* GraphIndex::entry */
    const uint64_t* offsets;
    const uint64_t* nbr_base;
    const uint32_t* nbrs;
    uint64_t total_nbrs;
    int device;
    trim_memory memory;
} trim_graph_desc;

typedef struct trim_graph* trim_graph_t;

int trim_graph_create(const trim_graph_desc* desc, trim_graph_t* out);
int trim_graph_destroy(trim_graph_t graph);

/*
 * graph::search_trim_knn (graph/search.hpp:188-264) for nq queries (host
 * arrays). ids_out/dist_out: nq*k, each row ascending by (dist_sq, id); a
 * query with fewer than k results pads with id 0xFFFFFFFF / +inf.
 * counters_out: nq (hops = expanded nodes, coarse_dc = 0), may be NULL.
 * k == 0 or k > ef -> TRIM_EINVAL (search.hpp:193-194); gamma < 0 ->
 * TRIM_EINVAL (uncalibrated profile, search.hpp:195-196); ef <= 1024.
 */
int trim_graph_search_knn(trim_graph_t graph, const float* queries, uint64_t nq, uint32_t k,
                          uint32_t ef, float gamma, uint32_t* ids_out, float* dist_out,
                          trim_counters* counters_out);
/* Device-resident trim_graph_search_knn: device pointers on the graph's device
 * (queries nq*dim, ids/dist nq*k, counters nq*6 u64 in trim_counters order),
 * asynchronous on `stream` (cudaStream_t). */
int trim_graph_search_knn_device(trim_graph_t graph, const float* d_queries, uint64_t nq, uint32_t k,
                                 uint32_t ef, float gamma, uint32_t* d_ids, float* d_dist,
                                 unsigned long long* d_counters, void* stream);
/*
 * graph::search_trim_range (graph/search.hpp:267-347). radius: nq plain radii
 * (negative -> TRIM_EINVAL). Results as trim_search_range: offsets_out nq+1,
 * library-allocated *ids_out / *dist_out (trim_free), ascending (dist_sq, id).
 * 1 <= ef <= 1024.
 */
int trim_graph_search_range(trim_graph_t graph, const float* queries, uint64_t nq,
                            const float* radius, uint32_t ef, float gamma, uint64_t* offsets_out,
                            uint32_t** ids_out, float** dist_out, trim_counters* counters_out);

#ifdef __cplusplus
}
#endif

#endif /* TRIM_GPU_H */
