/*
 * qmsort_gpu.h -- C-ABI of the B200-native QuickMergesort replacement.
 *
 * Drop-in boundary for the reference entry point
 *     template <class It, class Less = std::less<>>
 *     Metrics qmsort::sort(It first, It last, const SortConfig& cfg = {},
 *                          Less less = {}, SortObserver* obs = nullptr);
 *   (/root/reference/proj/core/include/qmsort/sort.hpp:215-226)
 * and its counted twin sort_range_counted (sort.hpp:207-211).  The reference is
 * a header-only C++ template library; a foreign caller (ctypes, a C++ shim,
 * JNI ...) binds the plain-C functions below.  No torch or CUDA types appear in
 * the signatures: device buffers and streams are passed as void*.
 *
 * Every entry point returns QMSORT_OK (0) or a QMSORT_E* code and never
 * throws; qmsort_gpu_last_error() describes the last failure of the calling
 * thread.  There is no CPU fallback: without a usable sm_100 device every
 * compute call fails with QMSORT_ECUDA.
 */
#ifndef QMSORT_GPU_H
#define QMSORT_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (SURVEY.md 8(b) "Errors") ---------------------------- */
#define QMSORT_OK 0
#define QMSORT_EINVAL 1    /* bad dtype / comparator / n / config          */
#define QMSORT_ENOWS 2     /* caller workspace smaller than required       */
#define QMSORT_ECUDA 3     /* CUDA runtime error (see last_error)          */
#define QMSORT_ENCCL 4     /* collective failure (sharded path)            */
#define QMSORT_EINTERNAL 5 /* internal capacity overflow                   */

/* ---- element types: the five BASELINE.json configs plus int64 ---------- */
typedef enum {
    QMSORT_DT_I32 = 0,   /* int32_t                                        */
    QMSORT_DT_U32 = 1,   /* uint32_t                                       */
    QMSORT_DT_U64 = 2,   /* uint64_t                                       */
    QMSORT_DT_F64 = 3,   /* double, NaN-free, no -0.0                       */
    QMSORT_DT_REC32 = 4, /* 4 x uint64_t, lexicographic over w0..w3         */
    QMSORT_DT_I64 = 5    /* int64_t: the reference profile's key type
                            (element.hpp:16, Vec in test_sort.cpp:22)        */
} qmsort_dtype;

/* ---- comparator: the reference's Less template argument ---------------- */
typedef enum {
    QMSORT_LESS = 0,    /* std::less<>    (ascending)                      */
    QMSORT_GREATER = 1  /* std::greater<> (descending, test_sort.cpp:356)  */
} qmsort_cmp;

/* ---- SortConfig as C scalars (sort.hpp:17-34, merge.hpp:14-31) --------- */
typedef struct {
    int variant;                     /* Variant: 0 qms 1 qmqs 2 momqms 3 hqms       */
    int pivot;                       /* PivotStrategy: 0 median_of_3 and
                                        1 median_of_sqrt_n -> seeded random sample;
                                        2 mom_of_thirds -> strided triple-median
                                        sample at every level; 3 hybrid -> random,
                                        triple medians for buckets outside the
                                        delta band                                 */
    int base_case_kind;              /* BaseCase: 0 insertion 1 hardcoded_small
                                        2 clever_quicksort                         */
    uint64_t base_case_size_threshold; /* BaseCasePolicy::size_threshold (10)     */
    int base_case_use_levels;        /* BaseCasePolicy::use_levels                 */
    double beta;                     /* 0.5; with base_case_use_levels the largest
                                        bucket the block sorter takes is n^beta
                                        (clamped to its size classes), the GPU
                                        form of "X on blocks of ~n^beta"
                                        (sort.hpp:91-96)                             */
    double delta;                    /* 1/16; hybrid: a bucket larger than
                                        (parent / buckets) / delta is re-split with
                                        the triple-median sample next level         */
    int side;                        /* MergesortSide: 0 smaller_always,
                                        1 larger_when_feasible (ignored on GPU)     */
    int three_way;                   /* always on for equal splitters on the GPU    */
    uint64_t block;                  /* partition block hint (kDefaultBlock 128)    */
    /* GPU knobs (GpuSortOptions): not in the reference SortConfig */
    int algorithm;                   /* 0 samplesort (default), 1 mergesort          */
    uint64_t seed;                   /* sampling seed                                */
    int max_levels;                  /* partition levels before the merge fallback   */
    int profile;                     /* 1: time every launch (phase_ns in metrics)   */
} qmsort_gpu_config;

/* Kernel families of the per-phase ledger: 0 transform, 1 sample (K1),
 * 2 count (K2), 3 plan (K3), 4 scatter (K4), 5 block sort (K5), 6 merge pass
 * (K6/K7), 7 equal-bucket fill (K8). */
#define QMSORT_NUM_PHASES 8

/* ---- Metrics (metrics.hpp:14-24) plus GPU pass ledger ------------------- */
typedef struct {
    uint64_t comparisons; /* not instrumented on the GPU: 0                 */
    uint64_t moves;       /* not instrumented on the GPU: 0                 */
    uint64_t max_depth;   /* partition levels used                          */
    uint64_t elapsed_ns;  /* device time of the sort (CUDA events)          */
    uint64_t alg_bytes;   /* B_alg: key bytes credited per executed pass     */
    uint32_t levels;      /* samplesort partition levels                    */
    uint32_t merge_passes;/* merge-path passes (fallback / mergesort)       */
    uint32_t kernel_launches; /* kernels launched by this call              */
    uint32_t host_syncs;  /* host synchronisations inside the sort          */
    uint64_t phase_bytes[QMSORT_NUM_PHASES];   /* algorithmic bytes per family */
    uint64_t phase_ns[QMSORT_NUM_PHASES];      /* device ns (profile = 1 only)  */
    uint32_t phase_launches[QMSORT_NUM_PHASES];
    uint32_t resplits;    /* hybrid pivot: buckets outside the delta band that
                             were re-sampled with triple medians (sort.hpp:114-118) */
    uint64_t sample_keys; /* splitter-sample keys drawn over all levels (median_of_3:
                             32 K per segment; median_of_sqrt_n: 2 floor(sqrt(len)/2)+1,
                             the reference's s, partition.hpp:240-241) */
    uint32_t table_buckets; /* integer-key buckets sent to the comparison-free table / cell
                               sorts (tablesort.cuh) instead of the network */
    uint32_t reserved;
} qmsort_gpu_metrics;

/* Presets qms() / qmqs() / momqms() / hqms() (sort.hpp:37-66). */
void qmsort_gpu_config_init(qmsort_gpu_config* cfg, int variant);

/* Bytes of device workspace qmsort_gpu_sort needs for n elements. */
size_t qmsort_gpu_workspace_bytes(int dtype, size_t n, const qmsort_gpu_config* cfg);

/* Sort d_data[0..n) in place on the device.  Replaces qmsort::sort
 * (sort.hpp:215-226) for device-resident ranges.  d_ws may be NULL (the
 * library allocates and frees it); otherwise ws_bytes must be at least
 * qmsort_gpu_workspace_bytes().  `stream` is a cudaStream_t (NULL = legacy
 * default stream).  The call returns after the sort completed. */
int qmsort_gpu_sort(int dtype, int cmp, void* d_data, size_t n, const qmsort_gpu_config* cfg,
                    void* d_ws, size_t ws_bytes, qmsort_gpu_metrics* metrics, void* stream);

/* Host-array drop-in: copies h_data[0..n) to the device, sorts, copies back.
 * Same contract as qmsort::sort(v.begin(), v.end(), cfg, less) on a
 * contiguous host range.  Device buffers are cached per thread. */
int qmsort_gpu_sort_host(int dtype, int cmp, void* h_data, size_t n, const qmsort_gpu_config* cfg,
                         qmsort_gpu_metrics* metrics);

/* A stream of independent host arrays (e.g. the trials of a harness, or
 * request batches of a service): the same contract as qmsort_gpu_sort_host for
 * every h_arrays[i] of ns[i] elements, pipelined through a ring of three
 * device arenas: array i+1 is copied in while array i sorts and array i-1 is
 * copied back, so both PCIe directions stay busy.  Pinned host memory gives
 * the overlap.  metrics
 * (optional) holds the sums (elapsed_ns: device sort time of all arrays). */
int qmsort_gpu_sort_host_batch(int dtype, int cmp, void* const* h_arrays, const size_t* ns,
                               size_t count, const qmsort_gpu_config* cfg,
                               qmsort_gpu_metrics* metrics);

/* ---- key + payload elements --------------------- */
/* Replaces qmsort::sort over Element<PayloadBytes> (element.hpp:13-20:
 * ordering on the key alone, payload moved with it; test_sort.cpp:328-339).
 * Sorts n elements of elem_bytes bytes (a multiple of 4, <= 4096) by the key of
 * key_dtype (I32/U32/U64/F64/I64) stored at byte offset key_offset, naturally
 * aligned.  Equal keys keep their input order (stable), which is one of the
 * arrangements the reference's unstable sort may produce; the key sequence is
 * the reference's exactly. */
size_t qmsort_gpu_elements_workspace_bytes(size_t n, size_t elem_bytes);
int qmsort_gpu_sort_elements(int key_dtype, int cmp, void* d_data, size_t n, size_t elem_bytes,
                             size_t key_offset, const qmsort_gpu_config* cfg, void* d_ws,
                             size_t ws_bytes, qmsort_gpu_metrics* metrics, void* stream);
int qmsort_gpu_sort_elements_host(int key_dtype, int cmp, void* h_data, size_t n,
                                  size_t elem_bytes, size_t key_offset,
                                  const qmsort_gpu_config* cfg, qmsort_gpu_metrics* metrics);

/* ---- selection ---------------------------------- */
/* Replaces select_nth(first, last, k, cmp, m) (selection.hpp:207-212): k is
 * 1-based; on return *pos = k-1 holds the k-th smallest element under cmp,
 * every element left of it is <= it and every element right of it >= it
 * (selection.hpp:124-126).  EINVAL unless 1 <= k <= n. */
size_t qmsort_gpu_select_workspace_bytes(int dtype, size_t n);
int qmsort_gpu_select_nth(int dtype, int cmp, void* d_data, size_t n, size_t k, size_t* pos,
                          const qmsort_gpu_config* cfg, void* d_ws, size_t ws_bytes,
                          qmsort_gpu_metrics* metrics, void* stream);
int qmsort_gpu_select_nth_host(int dtype, int cmp, void* h_data, size_t n, size_t k, size_t* pos,
                               const qmsort_gpu_config* cfg, qmsort_gpu_metrics* metrics);

/* Description of the last failure on the calling thread ("" if none). */
const char* qmsort_gpu_last_error(void);

/* Size in bytes of one element of dtype (0 for an unknown dtype). */
size_t qmsort_gpu_dtype_size(int dtype);

/* ---- sharded samplesort building blocks ---------------- */
/* In-place order-preserving transform into / out of the unsigned key domain
 * (inverse = 0 forward, 1 back).  After the forward transform, (I32,*) data is
 * sorted as (U32, LESS), (F64,*) as (U64, LESS), (*, GREATER) as LESS. */
int qmsort_gpu_transform(int dtype, int cmp, void* d_data, size_t n, int inverse, void* stream);

/* Core key dtype for a caller dtype: I32->U32, F64->U64, others unchanged. */
int qmsort_gpu_core_dtype(int dtype);

/* Gather s seeded random keys of d_data[0..n) (core dtype) into d_out. */
int qmsort_gpu_sample(int core_dtype, const void* d_data, size_t n, size_t s, uint64_t seed,
                      void* d_out, void* stream);

/* One partition level with caller-given sorted splitters (core dtype):
 * bucket b = #{splitters < key} (b in [0, nsplit]); writes d_in permuted so
 * that buckets are contiguous and ascending into d_out and the bucket sizes
 * into d_counts[0..nsplit] (uint64).  nsplit <= 511 (255 for REC32).  Uses
 * d_ws (see qmsort_gpu_partition_workspace_bytes) or allocates if NULL. */
size_t qmsort_gpu_partition_workspace_bytes(int core_dtype, size_t n);
int qmsort_gpu_partition(int core_dtype, const void* d_in, size_t n, const void* d_splitters,
                         uint32_t nsplit, void* d_out, uint64_t* d_counts, void* d_ws,
                         size_t ws_bytes, void* stream);

/* ---- PartitionResult (partition_result.hpp:12-17) ----------------------- */
/* Three-way partition of d_data[0..n) around the pivot value *h_pivot (caller
 * dtype, host memory) under cmp, in place: on return [0, c0) < pivot,
 * [c0, c0 + c1) == pivot, [c0 + c1, n) > pivot, with h_counts3 = {c0, c1, c2}
 * -- PartitionResult{lt_end = c0, gt_begin = c0 + c1, left_size = c0,
 * right_size = c2} (the three-way contract of three_way_partition,
 * partition.hpp:196-230).  The arrangement inside each part is unspecified. */
size_t qmsort_gpu_partition3_workspace_bytes(int dtype, size_t n);
int qmsort_gpu_partition3(int dtype, int cmp, void* d_data, size_t n, const void* h_pivot, uint64_t* h_counts3,
                          const qmsort_gpu_config* cfg, void* d_ws, size_t ws_bytes, qmsort_gpu_metrics* metrics,
                          void* stream);
int qmsort_gpu_partition3_host(int dtype, int cmp, void* h_data, size_t n, const void* h_pivot,
                               uint64_t* h_counts3, const qmsort_gpu_config* cfg, qmsort_gpu_metrics* metrics);

/* ---- the distributed samplesort ------------------------ */
/* Single-process entry over P <= 8 devices (one host thread drives them all):
 * rank r holds d_in[r][0..n_in[r]) (caller dtype, on device devices[r];
 * read only).  The call sorts the union of all ranks' keys under cmp and
 * leaves the r-th slice of the global order in d_out[r] (capacity out_cap[r]
 * elements, on devices[r]), its length in out_n[r]: concatenating the slices
 * in rank order gives the sorted array.  Global splitters from a seeded
 * sample, one exchange fused into the partition's scatter (each rank's kernel
 * stores straight into the peers' receive buffers over NVLink; peer access is
 * enabled between distinct devices), then local sorts.  A device may be listed
 * more than once (P ranks on one GPU run the same kernels and exchange).
 * QMSORT_ENOWS if some out_cap[r] < out_n[r] (out_n holds the sizes needed).
 * metrics: elapsed_ns = host wall time of the call, launches and pass bytes
 * summed over the ranks.  Replaces, for a sharded array, the reference entry
 * qmsort::sort (sort.hpp:215-226), which has no distributed form. */
int qmsort_gpu_sort_sharded(int dtype, int cmp, uint32_t P, const int* devices,
                            const void* const* d_in, const size_t* n_in, void* const* d_out,
                            const size_t* out_cap, size_t* out_n, const qmsort_gpu_config* cfg,
                            qmsort_gpu_metrics* metrics);

/* The same algorithm as steps a rank runs (one process per GPU; the caller
 * carries the small host collectives -- samples, the count matrix -- and the
 * receive-buffer handles, e.g. over torch.distributed):
 *   1. shard_sample: s seeded keys of the rank's caller-dtype data, mapped
 *      into the core key domain (seed: cfg.seed ^ 0x9E3779B97F4A7C15 * (r+1));
 *   2. (all ranks' samples gathered and sorted as core keys, e.g. with
 *      qmsort_gpu_sort) shard_splitters: nbuckets - 1 quantile splitters,
 *      merged into nuniq distinct values with multiplicities (host only);
 *      nbuckets = P * shard_subbuckets(dtype, P, n_total) for the folded
 *      exchange (n_total: the keys of all ranks), P
 *      for the plain one;
 *   3. shard_count: three-way counts, 2 nuniq + 1 bins (bin 2j: keys between
 *      splitters j-1 and j; 2j+1: keys equal to splitter j), or -- three_way
 *      = 0, for distinct splitters (every multiplicity 1) -- two-way counts,
 *      nuniq + 1 bins (bin j: keys above splitter j-1 up to splitter j; read
 *      them as the open bins 2j of the plan, equal bins 0); the plan stays in
 *      d_ws (shard_workspace_bytes); shard_scatter takes the same flag;
 *   4. the plan (host only, identical on every rank) from the P x (2 nuniq
 *      + 1) count matrix (row = sender):
 *      - folded (shard_plan_folded): every rank's slice as a three-way bin
 *        list of its own -- loc_m[r] local distinct splitters (indices into
 *        the global ones, P x (K0+1)), 2 loc_m[r] + 1 bin counts (P x
 *        (2K0+3)) -- the level 0 of its local sort; out_n[r] keys in all;
 *      - plain (shard_plan): receive sizes and lower / upper fills;
 *      both give bin -> rank (-1: equal keys, filled by the receivers) and
 *      per-sender offsets in the receivers' buffers;
 *   5. shard_scatter: the rank's bins straight into rank_dest[] (its row of
 *      bin_off; recv_n[r] keys in rank r's buffer), peer memory or local;
 *      raw = 0 ships core keys (folded), 1 the caller's (plain);
 *   6. folded: shard_finish_presplit sorts rank r's keys -- core keys already
 *      at their level-0 offsets in the B half (offset 0) of the workspace d_ws
 *      that served as its receive buffer (>= workspace_bytes(dtype, n)) --
 *      into d_out, fills included; plain: shard_finish writes [lo fill |
 *      sorted received keys | hi fill] into d_out (d_recv is only read). */
size_t qmsort_gpu_shard_workspace_bytes(int dtype, size_t n);
uint32_t qmsort_gpu_shard_subbuckets(int dtype, uint32_t P, uint64_t n_total);
int qmsort_gpu_shard_sample(int dtype, int cmp, const void* d_in, size_t n, size_t s, uint64_t seed,
                            void* d_out_core, void* stream);
int qmsort_gpu_shard_splitters(int core_dtype, const void* h_sorted_sample, size_t m, uint32_t nbuckets,
                               void* h_uniq, uint32_t* h_mult, uint32_t* nuniq);
int qmsort_gpu_shard_count(int dtype, int cmp, const void* d_in, size_t n, const void* d_uniq,
                           uint32_t nuniq, int three_way, uint64_t* d_counts, void* d_ws, size_t ws_bytes,
                           void* stream);
int qmsort_gpu_shard_plan(uint32_t P, uint32_t nuniq, const uint32_t* h_mult, const uint64_t* h_counts,
                          int32_t* h_bin_rank, uint64_t* h_bin_off, uint64_t* h_recv_n,
                          uint64_t* h_lo_fill, uint64_t* h_hi_fill, int32_t* h_lo_val, int32_t* h_hi_val);
int qmsort_gpu_shard_plan_folded(uint32_t P, uint32_t K0, uint32_t nuniq, const uint32_t* h_mult,
                                 const uint64_t* h_counts, int32_t* h_bin_rank, uint64_t* h_bin_off,
                                 uint64_t* h_out_n, uint32_t* h_loc_m, int32_t* h_loc_uniq,
                                 uint64_t* h_loc_counts);
int qmsort_gpu_shard_scatter(int dtype, int cmp, const void* d_in, size_t n, uint32_t nuniq, int three_way,
                             const int32_t* h_bin_rank, const uint64_t* h_bin_off, void* const* rank_dest,
                             const uint64_t* h_recv_n, uint32_t P, int raw, void* d_ws, size_t ws_bytes,
                             void* stream);
int qmsort_gpu_shard_finish_presplit(int dtype, int cmp, void* d_out, size_t n, const void* d_local_uniq,
                                     uint32_t local_m, const uint64_t* h_local_counts,
                                     const qmsort_gpu_config* cfg, void* d_ws, size_t ws_bytes,
                                     qmsort_gpu_metrics* metrics, void* stream);
int qmsort_gpu_shard_finish(int dtype, int cmp, const void* d_recv, size_t n_recv, const void* d_uniq,
                            int32_t lo_val, uint64_t lo_fill, int32_t hi_val, uint64_t hi_fill, void* d_out,
                            const qmsort_gpu_config* cfg, void* d_ws, size_t ws_bytes,
                            qmsort_gpu_metrics* metrics, void* stream);

/* CUDA IPC for the receive buffers of the fused exchange (one process per
 * GPU): export the allocation holding d_ptr (handle + d_ptr's byte offset in
 * it), open a peer's (d_ptr for the kernels, d_base for the close; peer access
 * over NVLink enabled lazily), close it. */
#define QMSORT_IPC_HANDLE_BYTES 64
int qmsort_gpu_ipc_handle(void* d_ptr, void* handle_out, uint64_t* offset_out);
int qmsort_gpu_ipc_open(const void* handle, uint64_t offset, void** d_ptr, void** d_base);
int qmsort_gpu_ipc_close(void* d_base);

/* ---- harness (K9 generators, verification) ----------------------------- */
/* kind: 0 u32 uniform, 1 u64 uniform, 2 rec32, 10..14 f64 sorted / reverse /
 * 16-distinct / gaussian / organ-pipe.  Element i is global element start+i
 * of an array of `total` elements (SURVEY.md 8(d) recipes). */
int qmsort_gpu_generate(int kind, void* d_out, size_t n, uint64_t seed, uint64_t start,
                        uint64_t total, void* stream);

/* out3[0] = adjacent order violations under (dtype, cmp) (if check_order),
 * out3[1] = sum, out3[2] = xor of a per-element fingerprint (multiset hash).
 * Synchronises the stream. */
int qmsort_gpu_check(int dtype, int cmp, const void* d_data, size_t n, int check_order,
                     uint64_t* out3, void* stream);

/* Library build identification (e.g. "qmsort-b200 sm_100a"). */
const char* qmsort_gpu_version(void);

/* Layout check for foreign binders: sizeof(qmsort_gpu_config) and
 * sizeof(qmsort_gpu_metrics) as compiled into the library. */
void qmsort_gpu_abi_sizes(size_t* config_bytes, size_t* metrics_bytes);

#ifdef __cplusplus
}
#endif

#endif /* QMSORT_GPU_H */
