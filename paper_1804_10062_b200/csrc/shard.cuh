// shard.cuh -- the distributed samplesort across GPUs.
//
// Included by qmsort_gpu.cu inside namespace qmsort_b200 (it uses the
// partition, sort and transform helpers defined there).  One global sort of
// the keys held by P ranks:
//   1. every rank draws a seeded sample of its keys through the comparator's
//      transform f (shard_sample_kernel);
//   2. the P samples are sorted together and P-1 evenly spaced quantiles are
//      the global splitters; equal splitters are merged into distinct values
//      u_j with a multiplicity c_j (shard_splitters, host);
//   3. every rank classifies its keys three-way against the u_j -- bin 2j =
//      keys between u_{j-1} and u_j, bin 2j+1 = keys equal to u_j -- and
//      counts them (partition_given, eq mode);
//   4. from the P x (2m+1) count matrix every rank computes the same plan
//      (shard_plan, host): open bins go to the rank #{splitters below}; the
//      keys equal to a splitter value repeated c_j >= 2 times are NOT sent --
//      their global count is split evenly over the c_j + 1 ranks the repeated
//      splitter spans and each of those ranks writes its share as a fill
//      (duplicate-heavy input stays balanced: no rank receives every copy of a
//      frequent key);
//   5. the scatter kernel stores every bin straight into its rank's receive
//      buffer (peer memory over NVLink: P2P pointers in one process, CUDA IPC
//      mappings across processes) -- the exchange IS the partition's scatter;
//   6. each rank sorts its received keys into its output (out of place,
//      transform fused) between its lower and upper fill.
// Folded form (the default of both drivers): step 2 picks P * K0 - 1
// splitters, K0 per rank, and the exchange scatter of step 5 IS level 0 of
// every rank's local sort -- each receive buffer is the B half of that rank's
// sort workspace, holding its K0 sub-buckets at their final offsets (core
// keys), and every equal-key run is a fill -- so the local sort starts at
// level 1 (shard_plan_folded_host, shard_finish_presplit): 8 n w of HBM per
// rank instead of 11 n w.
// Rank r's output is the r-th slice of the global order.  The reference has
// no distributed sort (single-threaded); the algorithm is the
// north star's "global splitter selection, one all-to-all, local sorts".
#pragma once

// out[i] = f(src[position i]): seeded positions (counter-based SplitMix64,
// uniform via a 64x64 high multiply), the same draw as gather_sample_kernel.
template <class K>
__global__ void shard_sample_kernel(const K* __restrict__ src, uint64_t n, uint64_t s, uint64_t seed,
                                    K* __restrict__ out, Xf xf) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t h = sm_mix(seed + (i + 1) * kGamma);
        out[i] = xf_fwd(src[__umul64hi(h, n)], xf);
    }
}

// dst[0, len) = f^-1(values[idx]) -- a rank's share of an equal-key run.
template <class K>
__global__ void shard_fill_kernel(K* __restrict__ dst, uint64_t len, const K* __restrict__ values,
                                  uint32_t idx, Xf xf) {
    const K v = xf_inv(values[idx], xf);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len;
         i += (uint64_t)gridDim.x * blockDim.x)
        dst[i] = v;
}

static int dispatch_sample(int dt, int cmp, const void* d, size_t n, size_t s, uint64_t seed, void* out,
                           cudaStream_t st) {
    if (n == 0 || s == 0) return QMSORT_OK;
    const Xf xf = make_xf(dt, cmp);
    const unsigned grid = (unsigned)std::min<size_t>((s + 255) / 256, 1184);
    switch (core_dtype(dt)) {
        case QMSORT_DT_U32:
            shard_sample_kernel<uint32_t><<<grid, 256, 0, st>>>((const uint32_t*)d, n, s, seed, (uint32_t*)out, xf);
            break;
        case QMSORT_DT_U64:
            shard_sample_kernel<uint64_t><<<grid, 256, 0, st>>>((const uint64_t*)d, n, s, seed, (uint64_t*)out, xf);
            break;
        case QMSORT_DT_REC32:
            shard_sample_kernel<Rec32><<<grid, 256, 0, st>>>((const Rec32*)d, n, s, seed, (Rec32*)out, xf);
            break;
    }
    QCK(cudaGetLastError());
    return QMSORT_OK;
}

// The local sort of a folded sharded exchange: the n keys (core keys,
// grouped into the three-way bins of uniq / counts) sit in the B half of the
// workspace ws (offset 0 of make_layout); the sorted caller-dtype keys land in
// d, fills included.
static int sort_presplit_device(int dt, int cmp, void* d, size_t n, const void* d_uniq, uint32_t m,
                                const uint64_t* counts, const qmsort_gpu_config* cfgp, void* wsp, size_t ws_bytes,
                                qmsort_gpu_metrics* mt, cudaStream_t st) {
    QTRY(validate(dt, cmp, n, d));
    if (m && !d_uniq) return fail(QMSORT_EINVAL, "null splitters");
    qmsort_gpu_config tmp;
    const qmsort_gpu_config& cfg = cfg_or_default(cfgp, tmp);
    const size_t nn = std::max<size_t>(n, 2);
    CallFrame f(st);
    if (!wsp || ws_bytes < ws_bytes_for(dt, nn)) return fail(QMSORT_ENOWS, "presplit: workspace too small");
    QTRY(f.begin(cfg, wsp, ws_bytes, ws_bytes_for(dt, nn)));
    unsigned char* w = static_cast<unsigned char*>(f.ws);
    const Xf xf = make_xf(dt, cmp);
    int rc = QMSORT_OK;
    if (n > 0) {
        switch (core_dtype(dt)) {
#define QPRE(K)                                                                                             \
    {                                                                                                       \
        const WsLayout L = make_layout<K>(nn);                                                              \
        const Presplit<K> pre{static_cast<const K*>(d_uniq), m, counts};                                    \
        rc = samplesort<K>(static_cast<K*>(d), reinterpret_cast<K*>(w + L.b_off), n, cfg, w, L, st, f.led,  \
                           xf, nullptr, &pre);                                                              \
        break;                                                                                              \
    }
            case QMSORT_DT_U32: QPRE(uint32_t)
            case QMSORT_DT_U64: QPRE(uint64_t)
            case QMSORT_DT_REC32: QPRE(Rec32)
#undef QPRE
        }
    }
    return f.end(rc, mt);
}

// Sample seed of rank r (the same on every path).
static uint64_t shard_seed(uint64_t seed, uint32_t r) { return seed ^ (0x9E3779B97F4A7C15ull * (uint64_t)(r + 1)); }

// Host: the splitters at sample ranks ((i+1) m) / nbuckets of the sorted
// sample, merged into distinct values (byte equality of core keys = key
// equality) with their multiplicities.
// nbuckets - 1 splitters (P for the plain exchange, P * K0 folded).
static int shard_splitters_host(int core, const void* sorted, size_t m, uint32_t nbuckets, void* uniq,
                                uint32_t* mult, uint32_t* nuniq) {
    const size_t w = dtype_size(core);
    if (w == 0 || core != core_dtype(core)) return fail(QMSORT_EINVAL, "splitters expect a core dtype");
    if (nbuckets < 1 || nbuckets > (uint32_t)(kMaxPeerBins / 2)) return fail(QMSORT_EINVAL, "1 <= buckets <= 512");
    if (m < nbuckets) return fail(QMSORT_EINVAL, "sample smaller than the bucket count");
    const unsigned char* s = static_cast<const unsigned char*>(sorted);
    unsigned char* u = static_cast<unsigned char*>(uniq);
    uint32_t k = 0;
    for (uint32_t i = 0; i + 1 < nbuckets; ++i) {
        const unsigned char* v = s + ((uint64_t)(i + 1) * m / nbuckets) * w;
        if (k > 0 && std::memcmp(u + (k - 1) * w, v, w) == 0) {
            ++mult[k - 1];
        } else {
            std::memcpy(u + k * w, v, w);
            mult[k++] = 1;
        }
    }
    *nuniq = k;
    return QMSORT_OK;
}

// Host: the exchange plan from the P x (2m+1) count matrix (row = sender).
// Every rank computes the same plan from the same matrix.
static int shard_plan_host(uint32_t P, uint32_t m, const uint32_t* mult, const uint64_t* counts,
                           int32_t* bin_rank, uint64_t* bin_off, uint64_t* recv_n, uint64_t* lo_fill,
                           uint64_t* hi_fill, int32_t* lo_val, int32_t* hi_val) {
    if (P < 1 || P > (uint32_t)kMaxPeers) return fail(QMSORT_EINVAL, "1 <= P <= 8 ranks");
    const uint32_t nb = 2 * m + 1;
    if (nb > (uint32_t)kMaxPeerBins) return fail(QMSORT_EINVAL, "too many splitters");
    uint64_t tot_mult = 0;
    for (uint32_t j = 0; j < m; ++j) {
        if (mult[j] == 0) return fail(QMSORT_EINVAL, "splitter multiplicity 0");
        tot_mult += mult[j];
    }
    if (tot_mult != P - 1) return fail(QMSORT_EINVAL, "splitter multiplicities must sum to P-1");
    for (uint32_t r = 0; r < P; ++r) {
        recv_n[r] = lo_fill[r] = hi_fill[r] = 0;
        lo_val[r] = hi_val[r] = -1;
    }
    uint32_t p = 0;  // splitters below the current value
    for (uint32_t j = 0; j < m; ++j) {
        bin_rank[2 * j] = (int32_t)p;  // open bin: rank #{splitters < key}
        if (mult[j] == 1) {
            bin_rank[2 * j + 1] = (int32_t)p;  // keys equal to a single splitter: the lower rank
        } else {
            bin_rank[2 * j + 1] = -1;  // filled by ranks p .. p + c
            uint64_t e = 0;
            for (uint32_t s = 0; s < P; ++s) e += counts[(size_t)s * nb + 2 * j + 1];
            const uint64_t c = mult[j];
            for (uint64_t i = 0; i <= c; ++i) {
                const uint64_t share = e * (i + 1) / (c + 1) - e * i / (c + 1);
                const uint32_t r = p + (uint32_t)i;
                if (i == 0) {
                    hi_fill[r] = share;
                    hi_val[r] = (int32_t)j;
                } else {
                    lo_fill[r] = share;
                    lo_val[r] = (int32_t)j;
                }
            }
        }
        p += mult[j];
    }
    bin_rank[2 * m] = (int32_t)p;
    // receive offsets: senders in rank order, each sender's bins in order
    for (uint32_t s = 0; s < P; ++s)
        for (uint32_t b = 0; b < nb; ++b) {
            const int32_t r = bin_rank[b];
            bin_off[(size_t)s * nb + b] = r < 0 ? 0 : recv_n[r];
            if (r >= 0) recv_n[r] += counts[(size_t)s * nb + b];
        }
    return QMSORT_OK;
}

// Sub-buckets per rank of the folded exchange.  The exchange's bucket count
// P * K0 starts at 256 -- an exchange tile writes runs of ~TILE / (P K0)
// keys per bucket, and 512-way runs measured 1.5x slower than 256-way (C2 at
// P = 1: 1.50 ms against 0.99 ms) -- and doubles (up to 2^LOGKMAX) only while
// a sub-bucket of n_total / (P K0) keys would need more than one further
// partition level (C3 at P = 1: 2^30 uint64 keys in 256 sub-buckets need two
// local levels, 45.0 ms; in 512, one, 37.3 ms).
template <class K>
static uint32_t shard_subbuckets_t(uint32_t P, uint64_t n_total) {
    using TU = Tune<K>;
    constexpr uint64_t cap = class_cap<K>(kNumClasses - 1);
    const uint64_t one_level = (cap * 3 / 4) << TU::LOGKMAX;  // choose_logk's single-level bound
    const uint32_t kmax = 1u << TU::LOGKMAX;
    uint32_t k0 = 1;
    while (P * k0 * 2 <= std::min<uint32_t>(kmax, 256)) k0 *= 2;
    while (P * k0 * 2 <= kmax && n_total > one_level * P * k0) k0 *= 2;
    return k0;
}
static uint32_t shard_subbuckets(int dt, uint32_t P, uint64_t n_total) {
    switch (core_dtype(dt)) {
        case QMSORT_DT_U32: return shard_subbuckets_t<uint32_t>(P, n_total);
        case QMSORT_DT_U64: return shard_subbuckets_t<uint64_t>(P, n_total);
        case QMSORT_DT_REC32: return shard_subbuckets_t<Rec32>(P, n_total);
    }
    return 1;
}

// Host: the folded plan from the P x (2M+1) count matrix of the P*K0 - 1
// global splitters (M distinct values u_j, multiplicities c_j; p_j = number
// of splitters below u_j).  Rank r takes the splitter indices [r K0, (r+1) K0):
// the open bin O_j goes to rank floor(p_j / K0); the keys equal to u_j go to
// the ranks floor(p_j / K0) .. floor((p_j + c_j) / K0), in even shares, as
// fills (never sent).  Every rank's slice is then a three-way bin list of its
// own -- local distinct values loc_uniq (indices into u) with loc_m entries
// and 2 loc_m + 1 bin counts loc_cnt (open, equal, open, ... , open) -- the
// level-0 result of its local sort.  bin_off[s][b]: where sender s's open
// bin b starts in its rank's buffer (that bin's local offset plus the
// earlier senders' parts).  LM = K0 + 1 local values at most.
static int shard_plan_folded_host(uint32_t P, uint32_t K0, uint32_t M, const uint32_t* mult, const uint64_t* C,
                                  int32_t* bin_rank, uint64_t* bin_off, uint64_t* out_n, uint32_t* loc_m,
                                  int32_t* loc_uniq, uint64_t* loc_cnt) {
    if (P < 1 || P > (uint32_t)kMaxPeers || K0 < 1) return fail(QMSORT_EINVAL, "1 <= P <= 8 ranks, K0 >= 1");
    const uint32_t nb = 2 * M + 1, LM = K0 + 1, LB = 2 * LM + 1;
    if (nb > (uint32_t)kMaxPeerBins) return fail(QMSORT_EINVAL, "too many splitters");
    uint64_t S = 0;
    std::vector<uint64_t> pj(M + 1, 0);
    for (uint32_t j = 0; j < M; ++j) {
        if (mult[j] == 0) return fail(QMSORT_EINVAL, "splitter multiplicity 0");
        pj[j] = S;
        S += mult[j];
    }
    pj[M] = S;
    if (S != (uint64_t)P * K0 - 1) return fail(QMSORT_EINVAL, "splitter multiplicities must sum to P*K0-1");
    auto rank_of_open = [&](uint32_t j) { return (uint32_t)std::min<uint64_t>(P - 1, pj[j] / K0); };
    std::vector<uint64_t> tot(nb, 0);
    for (uint32_t s = 0; s < P; ++s)
        for (uint32_t b = 0; b < nb; ++b) tot[b] += C[(size_t)s * nb + b];
    std::vector<int32_t> open_local(M + 1, -1);  // local bin index of global open bin j (in its rank)
    for (uint32_t r = 0; r < P; ++r) {
        uint32_t k = 0;  // local distinct values so far; the current open bin is 2k
        uint64_t* cnt = loc_cnt + (size_t)r * LB;
        for (uint32_t i = 0; i < LB; ++i) cnt[i] = 0;
        for (uint32_t j = 0; j <= M; ++j) {
            if (rank_of_open(j) == r) {
                cnt[2 * k] += tot[2 * j];
                open_local[j] = (int32_t)(2 * k);
            }
            if (j == M) break;
            const uint32_t lo = rank_of_open(j), hi = rank_of_open(j + 1);
            if (lo <= r && r <= hi) {
                if (k >= LM) return fail(QMSORT_EINTERNAL, "folded plan: too many local values");
                const uint64_t e = tot[2 * j + 1], parts = hi - lo + 1, i = r - lo;
                loc_uniq[(size_t)r * LM + k] = (int32_t)j;
                cnt[2 * k + 1] = e * (i + 1) / parts - e * i / parts;
                ++k;
            }
        }
        loc_m[r] = k;
        uint64_t n = 0;
        for (uint32_t i = 0; i < 2 * k + 1; ++i) n += cnt[i];
        out_n[r] = n;
    }
    // sender offsets: open bin j at its local bin's start in rank r, senders in order
    for (uint32_t j = 0; j <= M; ++j) {
        const uint32_t r = rank_of_open(j);
        bin_rank[2 * j] = (int32_t)r;
        if (j < M) bin_rank[2 * j + 1] = -1;
        uint64_t start = 0;
        const uint64_t* cnt = loc_cnt + (size_t)r * LB;
        for (int32_t i = 0; i < open_local[j]; ++i) start += cnt[i];
        for (uint32_t s = 0; s < P; ++s) {
            bin_off[(size_t)s * nb + 2 * j] = start;
            start += C[(size_t)s * nb + 2 * j];
            if (j < M) bin_off[(size_t)s * nb + 2 * j + 1] = 0;
        }
    }
    return QMSORT_OK;
}

// Partition workspace of one rank's count + scatter (the plan stays in it).
static size_t shard_ws_bytes(int dt, size_t n) { return ws_bytes_for(dt, std::max<size_t>(n, 2)); }

// Where one sender's bins go (host side of PeerArgs): bin b of the 2 nuniq + 1
// three-way bins -> rank bin_rank[b] (-1: not sent) at offset bin_off[b] of
// that rank's buffer rank_dest[r], which holds recv_n[r] keys.
struct ShardRoute {
    const int32_t* bin_rank;
    const uint64_t* bin_off;
    void* const* rank_dest;
    const uint64_t* recv_n;
    uint32_t P;
    bool raw;  // ship the caller's keys (else core keys)
};

// PeerArgs from a route: the ranks' virtual bases and every bin's first
// virtual position for this sender, copied into the workspace's misc area.
// three_way = false: the classifier's bin j is the route's open bin 2j (the
// splitters are distinct, so the keys equal to one go with the open bin below
// it -- the same rank; nothing is filled).
static int make_peer_args(uint32_t nbins, bool three_way, const ShardRoute& rt, size_t n_sender,
                          uint32_t* d_bin_base, cudaStream_t st, PeerArgs* pa) {
    if (rt.P < 1 || rt.P > (uint32_t)kMaxPeers) return fail(QMSORT_EINVAL, "1 <= P <= 8 ranks");
    if (nbins > (uint32_t)kMaxPeerBins) return fail(QMSORT_EINVAL, "too many splitters");
    *pa = PeerArgs{};
    pa->nranks = rt.P;
    pa->raw = rt.raw ? 1u : 0u;
    uint64_t v = 0;
    for (uint32_t r = 0; r < rt.P; ++r) {
        pa->dest[r] = reinterpret_cast<unsigned long long>(rt.rank_dest[r]);
        pa->vbase[r] = (uint32_t)v;
        v += rt.recv_n[r];
    }
    for (uint32_t r = rt.P; r <= (uint32_t)kMaxPeers; ++r) pa->vbase[r] = (uint32_t)v;
    if (v + n_sender >= (1ull << 32)) return fail(QMSORT_EINVAL, "the exchange moves >= 2^32 keys");
    uint32_t base[kMaxPeerBins];
    for (uint32_t b = 0; b < (uint32_t)kMaxPeerBins; ++b) base[b] = (uint32_t)v;  // empty / not-sent bins
    for (uint32_t b = 0; b < nbins; ++b) {
        const int32_t r = rt.bin_rank[b];
        if (r >= (int32_t)rt.P) return fail(QMSORT_EINVAL, "bin routed to a rank >= P");
        if (r < 0) continue;
        if (!three_way && (b & 1)) continue;  // two-way: no equal bins (their counts are 0)
        if (rt.rank_dest[r] == nullptr) return fail(QMSORT_EINVAL, "null receive buffer");
        base[three_way ? b : b / 2] = pa->vbase[r] + (uint32_t)rt.bin_off[b];
    }
    QCK(cudaMemcpyAsync(d_bin_base, base, sizeof(base), cudaMemcpyHostToDevice, st));
    pa->bin_base = d_bin_base;
    return QMSORT_OK;
}

// Count (parts 1) or scatter to the route (parts 2) of one rank's n caller keys.
// three_way = false (distinct splitters): two-way bins, nuniq + 1 counts.
static int shard_partition(int dt, int cmp, const void* d_in, size_t n, const void* uniq, uint32_t nuniq,
                           uint64_t* counts, void* ws, size_t ws_bytes, cudaStream_t st, int parts,
                           const ShardRoute* route, Ledger& led, bool three_way = true) {
    QTRY(validate(dt, cmp, n, d_in));
    if (2 * nuniq + 1 > (uint32_t)kMaxPeerBins) return fail(QMSORT_EINVAL, "too many splitters");
    if (!ws) return fail(QMSORT_EINVAL, "the shard partition needs a caller workspace");
    const size_t nn = std::max<size_t>(n, 2);
    if (ws_bytes < shard_ws_bytes(dt, n)) return fail(QMSORT_ENOWS, "shard workspace too small");
    unsigned char* w = static_cast<unsigned char*>(ws);
    const Xf xf = make_xf(dt, cmp);
    PeerArgs pa{};
    const PeerArgs* peers = nullptr;
    if (route) {
        size_t misc = 0;
        switch (core_dtype(dt)) {
            case QMSORT_DT_U32: misc = make_layout<uint32_t>(nn).misc_off; break;
            case QMSORT_DT_U64: misc = make_layout<uint64_t>(nn).misc_off; break;
            case QMSORT_DT_REC32: misc = make_layout<Rec32>(nn).misc_off; break;
        }
        QTRY(make_peer_args(2 * nuniq + 1, three_way, *route, n, reinterpret_cast<uint32_t*>(w + misc), st, &pa));
        peers = &pa;
    }
    switch (core_dtype(dt)) {
        case QMSORT_DT_U32:
            return partition_given<uint32_t>((const uint32_t*)d_in, n, (const uint32_t*)uniq, nuniq, nullptr, counts,
                                             w, make_layout<uint32_t>(nn), st, led, parts, peers, three_way, xf);
        case QMSORT_DT_U64:
            return partition_given<uint64_t>((const uint64_t*)d_in, n, (const uint64_t*)uniq, nuniq, nullptr, counts,
                                             w, make_layout<uint64_t>(nn), st, led, parts, peers, three_way, xf);
        case QMSORT_DT_REC32:
            return partition_given<Rec32>((const Rec32*)d_in, n, (const Rec32*)uniq, nuniq, nullptr, counts, w,
                                          make_layout<Rec32>(nn), st, led, parts, peers, three_way, xf);
    }
    return fail(QMSORT_EINVAL, "unknown dtype");
}

// One rank's output: [lo fill | sorted received keys | hi fill], the received
// keys (caller dtype) sorted out of place with the fused transform.
static int shard_finish(int dt, int cmp, const void* recv, size_t n_recv, const void* uniq, int32_t lo_val,
                        uint64_t lo_fill, int32_t hi_val, uint64_t hi_fill, void* out,
                        const qmsort_gpu_config* cfg, void* ws, size_t ws_bytes, qmsort_gpu_metrics* m,
                        cudaStream_t st) {
    QTRY(validate(dt, cmp, n_recv + lo_fill + hi_fill, out));
    const size_t w = dtype_size(dt);
    unsigned char* o = static_cast<unsigned char*>(out);
    QTRY(sort_device(dt, cmp, o + lo_fill * w, n_recv, cfg, ws, ws_bytes, m, st, recv));
    const Xf xf = make_xf(dt, cmp);
    for (int side = 0; side < 2; ++side) {
        const uint64_t len = side ? hi_fill : lo_fill;
        const int32_t vi = side ? hi_val : lo_val;
        if (len == 0) continue;
        if (vi < 0 || !uniq) return fail(QMSORT_EINVAL, "fill without a splitter value");
        unsigned char* at = o + (side ? (lo_fill + n_recv) * w : 0);
        const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((len + 255) / 256, 148 * 8));
        switch (core_dtype(dt)) {
            case QMSORT_DT_U32:
                shard_fill_kernel<uint32_t><<<grid, 256, 0, st>>>((uint32_t*)at, len, (const uint32_t*)uniq, vi, xf);
                break;
            case QMSORT_DT_U64:
                shard_fill_kernel<uint64_t><<<grid, 256, 0, st>>>((uint64_t*)at, len, (const uint64_t*)uniq, vi, xf);
                break;
            case QMSORT_DT_REC32:
                shard_fill_kernel<Rec32><<<grid, 256, 0, st>>>((Rec32*)at, len, (const Rec32*)uniq, vi, xf);
                break;
        }
        QCK(cudaGetLastError());
        if (m) ++m->kernel_launches;
    }
    return QMSORT_OK;
}

// ---------------------------------------------------------------------------
// Single-process driver over P devices (the C-level sharded entry).  Device
// buffers of different ranks are addressed directly (peer access enabled
// between distinct devices); a device may appear more than once, which runs
// P ranks on one GPU with the same kernels and the same exchange.
// ---------------------------------------------------------------------------
struct DevGuard {
    int prev = 0;
    DevGuard() { cudaGetDevice(&prev); }
    ~DevGuard() { cudaSetDevice(prev); }
};

struct ShardRank {
    int dev = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t scattered = nullptr, ready = nullptr;
    void *smp = nullptr, *uniq = nullptr, *counts = nullptr, *pws = nullptr, *recv = nullptr, *fws = nullptr;
    size_t pws_bytes = 0, fws_bytes = 0;
};

static int sort_sharded_sp(int dt, int cmp, uint32_t P, const int* devices, const void* const* d_in,
                           const size_t* n_in, void* const* d_out, const size_t* out_cap, size_t* out_n,
                           const qmsort_gpu_config* cfgp, qmsort_gpu_metrics* metrics) {
    if (P < 1 || P > (uint32_t)kMaxPeers) return fail(QMSORT_EINVAL, "1 <= P <= 8 ranks");
    if (!devices || !d_in || !n_in || !d_out || !out_cap || !out_n) return fail(QMSORT_EINVAL, "null argument");
    if (dtype_size(dt) == 0) return fail(QMSORT_EINVAL, "unknown dtype");
    qmsort_gpu_config tmp;
    const qmsort_gpu_config& cfg = cfg_or_default(cfgp, tmp);
    const int core = core_dtype(dt);
    const size_t w = dtype_size(dt);
    uint64_t total = 0;
    for (uint32_t r = 0; r < P; ++r) {
        QTRY(validate(dt, cmp, n_in[r], d_in[r]));
        total += n_in[r];
    }
    if (total >= (1ull << 32) * P) return fail(QMSORT_EINVAL, "too many keys");
    const auto t0 = std::chrono::steady_clock::now();
    DevGuard guard;
    int ndev = 0;
    QCK(cudaGetDeviceCount(&ndev));
    for (uint32_t r = 0; r < P; ++r)
        if (devices[r] < 0 || devices[r] >= ndev) return fail(QMSORT_EINVAL, "bad device ordinal");
    // peer access between every pair of distinct devices (idempotent)
    for (uint32_t a = 0; a < P; ++a)
        for (uint32_t b = 0; b < P; ++b) {
            if (devices[a] == devices[b]) continue;
            int can = 0;
            QCK(cudaDeviceCanAccessPeer(&can, devices[a], devices[b]));
            if (!can) return fail(QMSORT_ECUDA, "no peer access between devices " + std::to_string(devices[a]) +
                                                    " and " + std::to_string(devices[b]));
            QCK(cudaSetDevice(devices[a]));
            const cudaError_t e = cudaDeviceEnablePeerAccess(devices[b], 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) QCK(e);
            cudaGetLastError();  // clear "already enabled"
        }
    const uint32_t K0 = shard_subbuckets(dt, P, total);  // folded exchange: K0 sub-buckets per rank
    const uint32_t LM = K0 + 1;                   // local distinct splitters per rank, at most
    const uint32_t s = std::max(64 * P, 32 * K0);  // samples per rank: >= 32 per global bucket
    std::vector<ShardRank> R(P);
    uint32_t launches = 0;
    uint64_t alg = 0;
    auto cleanup = [&]() {
        for (ShardRank& x : R) {
            cudaSetDevice(x.dev);
            if (x.st) cudaStreamSynchronize(x.st);
            for (void* p : {x.smp, x.uniq, x.counts, x.pws, x.recv, x.fws})
                if (p) cudaFree(p);
            if (x.scattered) cudaEventDestroy(x.scattered);
            if (x.ready) cudaEventDestroy(x.ready);
            if (x.st) cudaStreamDestroy(x.st);
        }
    };
    struct Cleanup {
        std::function<void()> f;
        ~Cleanup() { f(); }
    } cl{cleanup};
    // 1. samples (core keys) of every rank, gathered on rank 0's device
    for (uint32_t r = 0; r < P; ++r) {
        ShardRank& x = R[r];
        x.dev = devices[r];
        QCK(cudaSetDevice(x.dev));
        QCK(cudaStreamCreateWithFlags(&x.st, cudaStreamNonBlocking));
        QCK(cudaEventCreateWithFlags(&x.scattered, cudaEventDisableTiming));
        QCK(cudaEventCreateWithFlags(&x.ready, cudaEventDisableTiming));
        QCK(cudaMalloc(&x.smp, (size_t)s * P * w));
        QCK(cudaMalloc(&x.uniq, (size_t)(kMaxPeerBins / 2 + LM) * w));  // global | local distinct splitters
        QCK(cudaMalloc(&x.counts, kMaxPeerBins * sizeof(uint64_t)));
        x.pws_bytes = shard_ws_bytes(dt, n_in[r]);
        QCK(cudaMalloc(&x.pws, x.pws_bytes));
    }
    std::vector<unsigned char> smp_h((size_t)s * P * w);
    for (uint32_t r = 0; r < P; ++r) {
        ShardRank& x = R[r];
        QCK(cudaSetDevice(x.dev));
        unsigned char* mine = static_cast<unsigned char*>(R[0].smp) + (size_t)r * s * w;
        if (n_in[r] > 0) {
            // sample into this rank's buffer, then copy to rank 0's gather slot
            QTRY(dispatch_sample(dt, cmp, d_in[r], n_in[r], s, shard_seed(cfg.seed, r), x.smp, x.st));
            ++launches;
            QCK(cudaMemcpyPeerAsync(mine, R[0].dev, x.smp, x.dev, (size_t)s * w, x.st));
        } else {  // an empty shard contributes maximum keys (never chosen as splitters below)
            QCK(cudaSetDevice(R[0].dev));
            QCK(cudaMemsetAsync(mine, 0xFF, (size_t)s * w, R[0].st));
            QCK(cudaSetDevice(x.dev));
        }
        QCK(cudaEventRecord(x.ready, x.st));
    }
    QCK(cudaSetDevice(R[0].dev));
    for (uint32_t r = 1; r < P; ++r) QCK(cudaStreamWaitEvent(R[0].st, R[r].ready, 0));
    {
        qmsort_gpu_config scfg;
        qmsort_gpu_config_init(&scfg, 0);
        qmsort_gpu_metrics sm_;
        QTRY(sort_device(core, 0, R[0].smp, (size_t)s * P, &scfg, nullptr, 0, &sm_, R[0].st));
        launches += sm_.kernel_launches;
        QCK(cudaMemcpyAsync(smp_h.data(), R[0].smp, smp_h.size(), cudaMemcpyDeviceToHost, R[0].st));
        QCK(cudaStreamSynchronize(R[0].st));
    }
    // 2. the P*K0 - 1 global splitters (host), to every device
    std::vector<unsigned char> uniq_h((size_t)(kMaxPeerBins / 2) * w);
    std::vector<uint32_t> mult(kMaxPeerBins / 2, 0);
    uint32_t nuniq = 0;
    QTRY(shard_splitters_host(core, smp_h.data(), (size_t)s * P, P * K0, uniq_h.data(), mult.data(), &nuniq));
    const uint32_t nb = 2 * nuniq + 1;
    // 3. counts of every rank: three-way when a splitter value repeats (its
    // equal keys are spread as fills), else two-way (cheaper; no equal bins)
    bool three_way = false;
    for (uint32_t j = 0; j < nuniq; ++j) three_way |= mult[j] > 1;
    const uint32_t ncnt = three_way ? nb : nuniq + 1;
    std::vector<uint64_t> C((size_t)P * nb, 0), C2((size_t)P * ncnt, 0);
    for (uint32_t r = 0; r < P; ++r) {
        ShardRank& x = R[r];
        QCK(cudaSetDevice(x.dev));
        if (nuniq) QCK(cudaMemcpyAsync(x.uniq, uniq_h.data(), nuniq * w, cudaMemcpyHostToDevice, x.st));
        Ledger led;
        QTRY(shard_partition(dt, cmp, d_in[r], n_in[r], x.uniq, nuniq, (uint64_t*)x.counts, x.pws, x.pws_bytes,
                             x.st, 1, nullptr, led, three_way));
        launches += led.launches;
        alg += led.alg_bytes;
        QCK(cudaMemcpyAsync(&C2[(size_t)r * ncnt], x.counts, ncnt * sizeof(uint64_t), cudaMemcpyDeviceToHost, x.st));
    }
    for (uint32_t r = 0; r < P; ++r) {
        QCK(cudaSetDevice(R[r].dev));
        QCK(cudaStreamSynchronize(R[r].st));
    }
    for (uint32_t r = 0; r < P; ++r)  // as three-way bins (two-way: bin j = open bin 2j)
        for (uint32_t b = 0; b < ncnt; ++b) C[(size_t)r * nb + (three_way ? b : 2 * b)] = C2[(size_t)r * ncnt + b];
    // 4. the folded plan (host, identical for every rank)
    std::vector<int32_t> bin_rank(nb);
    std::vector<uint64_t> bin_off((size_t)P * nb), recv_n(P), loc_cnt((size_t)P * (2 * LM + 1));
    std::vector<uint32_t> loc_m(P);
    std::vector<int32_t> loc_uniq((size_t)P * LM);
    QTRY(shard_plan_folded_host(P, K0, nuniq, mult.data(), C.data(), bin_rank.data(), bin_off.data(), recv_n.data(),
                                loc_m.data(), loc_uniq.data(), loc_cnt.data()));
    bool fits = true;
    for (uint32_t r = 0; r < P; ++r) {
        out_n[r] = recv_n[r];
        if (out_n[r] > out_cap[r]) fits = false;
        if (out_n[r] > 0 && d_out[r] == nullptr) return fail(QMSORT_EINVAL, "null output buffer");
    }
    if (!fits) return fail(QMSORT_ENOWS, "an output buffer is smaller than its slice (see out_n)");
    // every rank's local-sort workspace is its receive buffer (its B half),
    // and its local distinct splitters go next to the global ones
    std::vector<void*> dest(P, nullptr);
    for (uint32_t r = 0; r < P; ++r) {
        ShardRank& x = R[r];
        QCK(cudaSetDevice(x.dev));
        x.fws_bytes = ws_bytes_for(dt, std::max<uint64_t>(2, recv_n[r]));
        QCK(cudaMalloc(&x.fws, x.fws_bytes));
        dest[r] = x.fws;
        std::vector<unsigned char> lu((size_t)LM * w);
        for (uint32_t k = 0; k < loc_m[r]; ++k)
            std::memcpy(&lu[(size_t)k * w], &uniq_h[(size_t)loc_uniq[(size_t)r * LM + k] * w], w);
        if (loc_m[r])
            QCK(cudaMemcpy(static_cast<unsigned char*>(x.uniq) + (size_t)(kMaxPeerBins / 2) * w, lu.data(),
                           (size_t)loc_m[r] * w, cudaMemcpyHostToDevice));
    }
    // 5. every rank's scatter stores its open bins into the peers' buffers:
    // level 0 of their local sorts (core keys)
    for (uint32_t r = 0; r < P; ++r) {
        ShardRank& x = R[r];
        QCK(cudaSetDevice(x.dev));
        const ShardRoute rt{bin_rank.data(), &bin_off[(size_t)r * nb], dest.data(), recv_n.data(), P, false};
        Ledger led;
        QTRY(shard_partition(dt, cmp, d_in[r], n_in[r], x.uniq, nuniq, nullptr, x.pws, x.pws_bytes, x.st, 2, &rt,
                             led, three_way));
        launches += led.launches;
        alg += led.alg_bytes;
        QCK(cudaEventRecord(x.scattered, x.st));
    }
    // 6. local sorts once every sender's stores have landed (events, no host
    // wait): one host thread per rank, each sort has its own control read
    std::vector<int> rcs(P, QMSORT_OK);
    std::vector<std::string> errs(P);
    std::vector<qmsort_gpu_metrics> ms(P);
    auto finish_rank = [&](uint32_t r) {
        ShardRank& x = R[r];
        const int rc = [&]() -> int {
            QCK(cudaSetDevice(x.dev));
            for (uint32_t q = 0; q < P; ++q)
                if (q != r) QCK(cudaStreamWaitEvent(x.st, R[q].scattered, 0));
            std::memset(&ms[r], 0, sizeof(ms[r]));
            const int rc2 = sort_presplit_device(dt, cmp, d_out[r], recv_n[r],
                                                 static_cast<unsigned char*>(x.uniq) + (size_t)(kMaxPeerBins / 2) * w,
                                                 loc_m[r], &loc_cnt[(size_t)r * (2 * LM + 1)], &cfg, x.fws,
                                                 x.fws_bytes, &ms[r], x.st);
            if (rc2 != QMSORT_OK) return rc2;
            QCK(cudaStreamSynchronize(x.st));
            return QMSORT_OK;
        }();
        rcs[r] = rc;
        if (rc != QMSORT_OK) errs[r] = g_err;
    };
    {
        std::vector<std::thread> th;
        for (uint32_t r = 1; r < P; ++r) th.emplace_back(finish_rank, r);
        finish_rank(0);
        for (std::thread& t : th) t.join();
    }
    for (uint32_t r = 0; r < P; ++r) {
        if (rcs[r] != QMSORT_OK) return fail(rcs[r], "rank " + std::to_string(r) + ": " + errs[r]);
        launches += ms[r].kernel_launches;
        alg += ms[r].alg_bytes;
    }
    if (metrics) {
        std::memset(metrics, 0, sizeof(*metrics));
        metrics->elapsed_ns = (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                                  std::chrono::steady_clock::now() - t0).count();
        metrics->kernel_launches = launches;
        metrics->alg_bytes = alg;
        metrics->host_syncs = 3;
    }
    g_err.clear();
    return QMSORT_OK;
}

// ---------------------------------------------------------------------------
// PartitionResult (partition_result.hpp:12-17): a three-way partition of the
// caller's range around one pivot value -- [0, lt_end) < pivot, [lt_end,
// gt_begin) == pivot, [gt_begin, n) > pivot under cmp -- the one-splitter case
// of the given-splitter partition (three-way bins), like three_way_partition
// (partition.hpp:196-230) with the pivot passed by value.
// ---------------------------------------------------------------------------
static void xf_fwd_host(int dt, int cmp, const void* in, void* out) {
    const Xf f = make_xf(dt, cmp);
    const size_t w = dtype_size(dt);
    if (w == 4) {
        uint32_t x;
        std::memcpy(&x, in, 4);
        x ^= (uint32_t)f.b;
        std::memcpy(out, &x, 4);
    } else {
        for (size_t i = 0; i < w / 8; ++i) {
            uint64_t x;
            std::memcpy(&x, static_cast<const char*>(in) + 8 * i, 8);
            x = x ^ f.b ^ ((uint64_t)((int64_t)x >> 63) & f.a);
            std::memcpy(static_cast<char*>(out) + 8 * i, &x, 8);
        }
    }
}

static int partition3_device(int dt, int cmp, void* d, size_t n, const void* h_pivot, uint64_t* h_counts3,
                             const qmsort_gpu_config* cfgp, void* wsp, size_t ws_bytes, qmsort_gpu_metrics* m,
                             cudaStream_t st) {
    QTRY(validate(dt, cmp, n, d));
    if (!h_pivot || !h_counts3) return fail(QMSORT_EINVAL, "null pivot or counts");
    qmsort_gpu_config tmp;
    const qmsort_gpu_config& cfg = cfg_or_default(cfgp, tmp);
    const size_t w = dtype_size(dt);
    const size_t nn = std::max<size_t>(n, 2);
    const size_t need = ws_bytes_for(dt, nn) + 256;
    CallFrame f(st);
    QTRY(f.begin(cfg, wsp, ws_bytes, need));
    unsigned char* ws = static_cast<unsigned char*>(f.ws);
    unsigned char* extra = ws + ws_bytes_for(dt, nn);  // pivot (core key) | 3 counts
    unsigned char pv[32];
    xf_fwd_host(dt, cmp, h_pivot, pv);
    uint64_t* dcnt = reinterpret_cast<uint64_t*>(extra + 64);
    int rc = QMSORT_OK;
    auto run = [&]() -> int {
        QCK(cudaMemcpyAsync(extra, pv, w, cudaMemcpyHostToDevice, st));
        if (n == 0) {
            QCK(cudaMemsetAsync(dcnt, 0, 3 * sizeof(uint64_t), st));
            return QMSORT_OK;
        }
        const Xf xf = make_xf(dt, cmp);
        switch (core_dtype(dt)) {
#define QPART3(K)                                                                                             \
    {                                                                                                         \
        const WsLayout L = make_layout<K>(nn);                                                                \
        K* B = reinterpret_cast<K*>(ws + L.b_off);                                                            \
        QTRY(partition_given<K>(static_cast<const K*>(d), n, reinterpret_cast<const K*>(extra), 1, B, dcnt,   \
                                ws, L, st, f.led, 3, nullptr, true, xf));                                     \
        QCK(cudaMemcpyAsync(d, B, n * sizeof(K), cudaMemcpyDeviceToDevice, st));                              \
        if (xf.a | xf.b) QTRY(xf_range<K>(static_cast<K*>(d), n, xf, true, st, f.led));                       \
        break;                                                                                                \
    }
            case QMSORT_DT_U32: QPART3(uint32_t)
            case QMSORT_DT_U64: QPART3(uint64_t)
            case QMSORT_DT_REC32: QPART3(Rec32)
#undef QPART3
        }
        return QMSORT_OK;
    };
    rc = run();
    if (rc == QMSORT_OK) {
        uint64_t h[3] = {0, 0, 0};
        const cudaError_t e = cudaMemcpyAsync(h, dcnt, sizeof(h), cudaMemcpyDeviceToHost, st);
        rc = f.end(e == cudaSuccess ? QMSORT_OK : fail(QMSORT_ECUDA, cudaGetErrorString(e)), m);
        if (rc == QMSORT_OK) std::memcpy(h_counts3, h, sizeof(h));
        return rc;
    }
    return f.end(rc, m);
}
