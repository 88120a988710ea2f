// C-ABI and per-rank engine of libgnnstep.so (include/gnnstep.h).
//
// One step = the trainer-process work of PAPER.md §3 lines 237-242 (sampling → data
// fetching → forward/backward → local gradient) + the synchronous-SGD exchange of §2.2
// lines 173-175.  All buffers are sized once to worst-case bounds (DESIGN.md "Dynamic
// shapes"); every kernel reads its extent from a device StepState, so the training body is
// captured once as a CUDA graph and replayed per mini-batch.
//
// Overlap (the B200 analog of the paper's process-level overlap, §4.1): the
// batch-side buffers are double-buffered (two BatchSets).  While batch s trains on the
// model's stream from set A, batch s+1 is sampled into set B on the library's sampling stream;
// events order "sampled(B) -> train(B)" and "trained(A) -> sample into A".
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <climits>
#include <cstddef>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <cub/device/device_radix_sort.cuh>
#include <string>
#include <vector>

#include "../../include/gnnstep.h"
#include "kernels.h"

using namespace gs;

namespace {
thread_local std::string g_err;

gnn_status fail(gnn_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess)                                                                  \
            return fail(e_ == cudaErrorMemoryAllocation ? GNN_ERR_OOM : GNN_ERR_CUDA,           \
                        std::string(#x) + ": " + cudaGetErrorString(e_));                       \
    } while (0)
#define CKN(x)                                                                                  \
    do {                                                                                        \
        ncclResult_t r_ = (x);                                                                  \
        if (r_ != ncclSuccess) return fail(GNN_ERR_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
    } while (0)
#define TRY(x)                        \
    do {                              \
        gnn_status s_ = (x);          \
        if (s_ != GNN_OK) return s_;  \
    } while (0)

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// NVTX range around an ABI call (host side; Nsight tools attribute the enqueued kernels to it).
struct Range {
    explicit Range(const char* name) { nvtxRangePushA(name); }
    ~Range() { nvtxRangePop(); }
};

template <class T>
gnn_status dalloc(T** p, int64_t count, std::vector<void*>& owned) {
    *p = nullptr;
    if (count <= 0) count = 1;
    cudaError_t e = cudaMalloc((void**)p, sizeof(T) * (size_t)count);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(GNN_ERR_OOM, "cudaMalloc of " + std::to_string(sizeof(T) * count) + " bytes: " +
                                     cudaGetErrorString(e));
    }
    owned.push_back(*p);
    return GNN_OK;
}
}  // namespace

struct gnn_graph {
    int dev = 0;
    int64_t N = 0, nnz = 0;
    int F = 0, stride = 0, C = 0;
    int64_t* row_ptr = nullptr;
    int32_t* col = nullptr;
    float* X = nullptr;        // full table, or this process's shard (rows [row_begin, row_end))
    int32_t* y = nullptr;
    int64_t row_begin = 0, row_end = 0;
    bool symmetric = false;    // every entry has its reverse (checked at creation)
    // row-sharded features (config 4): peer shard pointers (device array) after gnn_shard_import
    int nshards = 0;
    int64_t rps = 0;
    const float** shard_ptrs = nullptr;
    std::vector<void*> ipc_opened;
    std::vector<void*> owned;
    // NEXT-2 feature cache of remote rows (sharded tables): device descriptor + its buffers
    // (allocated with a sharded graph, so every captured step reads the current descriptor)
    FeatCache* cache_desc = nullptr;
    int32_t* cmap = nullptr;
    float* cache_rows = nullptr;
    int64_t cache_n = 0;
    unsigned long long* cache_stats = nullptr;   // {local, peer, cache} row reads (gnn_cache_stats)
    bool stats_on = false;
    FeatRows rows() const {
        return FeatRows{X, nshards ? shard_ptrs : nullptr, rps, nshards ? cache_desc : nullptr,
                        rps ? (int)(row_begin / rps) : 0, nshards ? 0 : N};
    }
};

namespace {
// Capacities and sampling-kernel scratch of one block (hop h or the ShaDow induced block).
struct HopBufs {
    int64_t cap_dst = 0, cap_edges = 0, cap_src = 0;
    bool need_t = false;
    bool count_only = false;   // only the out-degrees (transposed row pointer): GCN's layer-1 block
    int32_t *tcount = nullptr, *tcursor = nullptr, *tdst = nullptr;   // shared by both batch sets
    int32_t* erow = nullptr;             // destination row of every edge (transposed fill)
};

// What one batch is made of, double-buffered: sizes, node list, per-block CSR + transposed CSR.
struct BatchSet {
    StepState* st = nullptr;
    int32_t* nodes = nullptr;
    int32_t* seeds_in = nullptr;     // device copy of host seeds (e2e)
    int32_t* seeds_stage = nullptr;  // pinned host staging of those seeds
    int32_t *rowptr[kMaxHops + 1] = {}, *nbr[kMaxHops + 1] = {}, *col[kMaxHops + 1] = {};
    int32_t *trowptr[kMaxHops + 1] = {}, *tdst_s[kMaxHops + 1] = {};
    SampleParams sp{};
    cudaEvent_t sampled = nullptr, trained = nullptr;
    cudaEvent_t l1done = nullptr;    // recorded after this set's layer-1 aggregation (GS_SAMPLE_AFTER_L1)
    bool trained_once = false;
    // the batch this set holds (valid until trained or overwritten)
    bool valid = false;
    bool host_seeds = false;         // seeds came from a host array (e2e) rather than the epoch permutation
    int64_t epoch = -1, g = -1;
    int32_t n = -1, b_total = -1;
    cudaGraphExec_t gexec = nullptr, prof_gexec = nullptr;
    std::vector<struct ProfPair> prof_pairs;
};

struct Layer {
    int in = 0, out = 0, in_pad = 0, k_pad = 0, n_pad = 0, rows = 0;  // rows of W (2in or in)
    int64_t poff = 0, pcnt = 0;
    int blk = 0;           // block (hop or ShaDow slot) this layer aggregates over
    int64_t m_cap = 0;     // max rows of this layer's output
    int splits = 1;
    int64_t rows_alloc = 0;  // operand-plane rows (m_cap rounded to the 128-row GEMM tile)
    Split A{}, dPre{}, Wkn{};   // bf16 split planes (GEMM operands); W as [K_pad x N_pad]
    float *H = nullptr, *dA = nullptr, *wpart = nullptr;
    uint32_t* hmask = nullptr;   // ReLU decisions of H (bit per element; layers with ReLU)
    int mask_ld = 0;             // words per hmask row
    TcGemmMaps map_fwd{}, map_dgrad{}, map_wgrad{};
    // layer 1 with its gather on the sampling stream (gnn_model::l1_on_sampler): batch set 1's
    // copy of the operand planes and of the maps that read them (set 0 uses A / map_fwd / map_wgrad)
    Split A1{};
    TcGemmMaps map_fwd1{}, map_wgrad1{};
};

struct ProfPair { int kid; cudaEvent_t a, b; };
}  // namespace

struct gnn_model {
    gnn_graph* g = nullptr;
    gnn_model_config cfg{};
    int L = 0, hops = 0, slot = -1;
    bool sage = true, shadow = false;
    std::vector<int> dims;
    cudaStream_t stream = nullptr;       // training (the caller's, or own_stream)
    cudaStream_t own_stream = nullptr;
    cudaStream_t sstream = nullptr;      // sampling (library-owned)
    cudaStream_t wstream = nullptr;      // weight-gradient branch of the training step
    cudaEvent_t ev_dpre[kMaxHops] = {}, ev_join = nullptr;
    std::vector<void*> owned;
    std::vector<void*> owned_host;

    BatchSet bs[2];
    int last = -1;                       // set trained last
    int fetch_set = 0;                   // set gnn_sample filled
    int32_t *map = nullptr, *icount = nullptr, *hubs = nullptr;
    // ShaDow: balanced-aggregation partials/counters and the last layer's receptive-field mask
    float* bal_part = nullptr;
    int32_t* bal_cnt = nullptr;
    uint32_t* rf_mask = nullptr;
    // receptive-field compaction of layer L-1 (R19): its rows, their positions, the
    // traversal row pointers (block; transposed block when not symmetric), scratch
    bool rf_compact = false;
    int32_t *rf_list = nullptr, *rf_pos = nullptr, *rf_sub = nullptr, *rf_sub_t = nullptr;
    void* rf_scratch = nullptr;
    uint32_t seq = 0;                    // sampling-launch sequence number (scan-word tags)
    bool full_train = true;              // training needs the last hop's relabel (GCN, ShaDow)
    bool last_full = true;               // mode of the last sampling launch (phase readout)
    unsigned long long* status = nullptr;
    GridBarrier* bar = nullptr;
    uint32_t* bits = nullptr;
    int64_t nwords = 0, nodes_cap = 0;
    HopBufs hb[kMaxHops + 1];
    std::vector<Layer> layers;
    float *params = nullptr, *grads = nullptr;
    int64_t pcount = 0;
    OptState opt{};                      // Adam moments + step count (m == nullptr: SGD)
    bool overlap = true;                 // prefetch the next batch during training

    std::vector<int64_t> schedule;       // NEXT-3: step s, rank r trains batch schedule[s*world + r] (empty: g = s*world + r)
    int32_t *perm = nullptr, *train_sorted = nullptr;
    uint64_t *keys = nullptr, *keys_alt = nullptr;
    void* cub_tmp = nullptr;
    size_t cub_bytes = 0;
    int64_t n_train = 0, train_cap = 0, perm_epoch = -1;

    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
    int exchange = GNN_EXCH_AUTO;        // gradient exchange (gnn_set_exchange)
    // GNN_EXCH_PEER: this rank's region {inbox [2][world][pcount] fp32, flags [world] u64}, the
    // peers' regions (CUDA IPC), device arrays of their addresses, sequence number and counters
    void* xregion = nullptr;
    std::vector<void*> xopened;
    PeerX px{};
    bool peer_ready = false;

    bool bf16x3 = true;                  // fp32 parity mode: 3-term bf16 split GEMMs
    int64_t launches_per_step = 0;

    int64_t reuse_hits = 0, reuse_misses = 0;   // steps that found / did not find their batch prefetched
    // step timeline (GS_TIMELINE=1, diagnostics): events around every sampling launch (sampling
    // stream) and every training launch (training stream), read back by gnn_debug_get
    bool timeline = false;
    // A batch's sampling waits until the training step in flight has finished its layer-1
    // aggregation: the bulk-copy gather (3 x 58 KB of shared memory per SM) then runs alone at full
    // bandwidth, and the sampling kernel overlaps the rest of the step (timeline, DESIGN.md §6.1:
    // products 3780 -> 4290 mini-batches/s, epoch 51.8 -> 43.9 ms; with sampling co-running the
    // gather the training span grew from ~186 to ~267 µs)
    bool sample_after_l1 = false;
    // layer 1's gather + mean (S4+S5) runs on the sampling stream right after the batch's sampling
    // kernel, into the batch set's own operand planes: the training graph starts at the first GEMM,
    // and the gather of step s+1 overlaps the tail of step s (GS_L1_ON_SAMPLER)
    bool l1_on_sampler = false;
    bool last_fused = false;             // GS_LAST_FUSED=1 at model creation: k_last_layer (§6.9)
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tl_sample, tl_train;
    bool profiling = false;
    std::vector<ProfPair> pending;
    std::vector<cudaEvent_t> free_events;
    double prof_ms[GNN_K_COUNT] = {};
    int64_t prof_n[GNN_K_COUNT] = {};
};

namespace {
// ---------------------------------------------------------------- profiling wrapper
cudaEvent_t take_event(gnn_model* m) {
    if (!m->free_events.empty()) {
        cudaEvent_t e = m->free_events.back();
        m->free_events.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

template <class Fn>
void K(gnn_model* m, cudaStream_t s, int kid, Fn&& fn) {
    if (m->profiling) {
        ProfPair p{kid, take_event(m), take_event(m)};
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(s, &cs);
        // inside a capture, only an "external" record node really records at replay time
        const unsigned fl = cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
        cudaEventRecordWithFlags(p.a, s, fl);
        fn();
        cudaEventRecordWithFlags(p.b, s, fl);
        m->pending.push_back(p);
    } else {
        fn();
    }
}

void drain_profile(gnn_model* m) {
    for (auto& p : m->pending) {
        float ms = 0.f;
        cudaEventSynchronize(p.b);
        cudaEventElapsedTime(&ms, p.a, p.b);
        m->prof_ms[p.kid] += ms;
        m->prof_n[p.kid] += 1;
        m->free_events.push_back(p.a);
        m->free_events.push_back(p.b);
    }
    m->pending.clear();
}

PackAll pack_desc(gnn_model* m) {
    PackAll p{};
    p.n = m->L;
    p.sage = m->sage;
    for (int li = 0; li < m->L; ++li) {
        const Layer& ly = m->layers[li];
        p.l[li] = PackLayer{ly.poff, ly.rows, ly.out, ly.in, ly.in_pad, ly.k_pad, ly.n_pad, ly.Wkn, ly.wpart,
                            ly.splits, (int64_t)ly.k_pad * ly.n_pad};
    }
    return p;
}

const int32_t* rows_ptr(gnn_model* m, int set, int li) {   // output rows of layer li (0-based)
    StepState* st = m->bs[set].st;
    if (m->shadow && li == m->L - 1) return &st->batch_n;
    if (m->rf_compact && li == m->L - 2) return &st->n_rf;
    return &st->n_dst[m->layers[li].blk];
}

// layer 1's operand planes and GEMM maps of batch set `set` (per set when layer 1's gather runs
// on the sampling stream: the gather of the next batch writes the other set's planes)
const TcGemmMaps& fwd_map(const gnn_model* m, const Layer& ly, int li, int set) {
    return (li == 0 && m->l1_on_sampler && set == 1) ? ly.map_fwd1 : ly.map_fwd;
}
const TcGemmMaps& wgrad_map(const gnn_model* m, const Layer& ly, int li, int set) {
    return (li == 0 && m->l1_on_sampler && set == 1) ? ly.map_wgrad1 : ly.map_wgrad;
}

// The gradient exchange of a step (§2.2): NCCL all-reduce between the
// reduce and the update (any world with GNN_EXCH_NCCL, world > 1 by default), else one rank's
// reduce fused into the update.
bool uses_nccl(const gnn_model* m) {
    return m->exchange == GNN_EXCH_NCCL || (m->exchange == GNN_EXCH_AUTO && m->world > 1);
}
// GNN_EXCH_HOST: the step stops at the reduced gradient; the caller all-reduces it (with host
// ranks, §3) and calls gnn_apply_update
bool uses_host(const gnn_model* m) { return m->exchange == GNN_EXCH_HOST; }
// GS_LAST_FUSED=1 (A/B): the last layer on the CUDA cores (k_last_layer, with the layer's
// aggregation for SAGE) when its classes fit a warp pair and W fits shared memory.  Measured: 30 µs
// per step against 33 µs for the aggregation + tensor-core GEMM/CE + dgrad GEMM it replaces, and
// the step no faster (products 4060-4110 vs 4235-4245 mini-batches/s): off by default
bool fused_last(const gnn_model* m) {
    const Layer& ly = m->layers[m->L - 1];
    return m->last_fused && last_layer_fits(ly.k_pad, ly.out);
}

// ---------------------------------------------------------------- step bodies
void enqueue_training(gnn_model* m, int set) {
    gnn_graph* g = m->g;
    BatchSet& B = m->bs[set];
    cudaStream_t s = m->stream;
    const int L = m->L;
    // ShaDow: rows the last layer reads (layer L-1 computes only these, R19)
    if (m->shadow && L >= 2)
        K(m, s, GNN_K_AGG, [&] {
            launch_rf_mark(&B.st->batch_n, B.rowptr[m->slot], B.col[m->slot], &B.st->seq, m->rf_mask, s);
            if (m->rf_compact)
                launch_rf_compact(m->rf_mask, &B.st->seq, (int)m->nodes_cap, B.rowptr[m->slot],
                                  B.trowptr[m->slot] ? B.trowptr[m->slot] : B.rowptr[m->slot], m->rf_scratch,
                                  m->rf_list, m->rf_pos, m->rf_sub, m->rf_sub_t, &B.st->n_rf, s);
        });
    auto bal = [&](bool bwd, int li, const int32_t* rows) {
        const Layer& ly = m->layers[li];
        const int blk = ly.blk;
        BalLaunch b{};
        b.bwd = bwd;
        b.gcn = !m->sage;
        b.ndst_ptr = &B.st->n_dst[blk];
        const bool cmp = m->rf_compact;
        b.rmask = !cmp && li == L - 2 ? m->rf_mask : nullptr;
        b.tag_ptr = &B.st->seq;
        b.in_pad = ly.in_pad;
        b.part = m->bal_part;
        b.cnt = m->bal_cnt;
        const int32_t* trow = B.trowptr[blk] ? B.trowptr[blk] : B.rowptr[blk];   // symmetric block: its own transpose
        if (!bwd) {
            b.n_ptr = rows;
            b.rowptr = B.rowptr[blk]; b.col = B.col[blk];
            b.orow = trow;
            b.H = li == 0 ? g->rows() : FeatRows{m->layers[li - 1].H, nullptr, 0};
            b.gmap = li == 0 ? B.nodes : nullptr;
            if (cmp && li == L - 2) {   // only the receptive field's rows, written compactly
                b.rlist = m->rf_list; b.rowptr = m->rf_sub; b.brow = B.rowptr[blk];
            }
            if (cmp && li == L - 1) b.gmap = m->rf_pos;   // H of layer L-1 is compact
            b.out = ly.A;
            b.out_w = m->sage ? 2 * ly.in_pad : ly.k_pad;
        } else {
            b.n_ptr = &B.st->n_src[blk];
            b.dlim_ptr = rows;
            b.rowptr = trow;
            b.col = B.tdst_s[blk] ? B.tdst_s[blk] : B.col[blk];
            b.orow = B.rowptr[blk];
            b.dA = ly.dA;
            if (cmp && li == L - 1) {   // gradient reaches only the receptive field: compact dPre of layer L-1
                b.n_ptr = &B.st->n_rf;
                b.rlist = m->rf_list; b.rowptr = m->rf_sub_t; b.brow = trow;
            }
            if (cmp && li == L - 2) b.dmap = m->rf_pos;   // dA of layer L-1 is compact
            b.hmask = m->layers[li - 1].hmask;
            b.mask_ld = m->layers[li - 1].mask_ld;
            b.out = m->layers[li - 1].dPre;
            b.out_w = ly.in_pad;
        }
        launch_agg_bal(b, s);
    };
    // ---- forward
    for (int li = 0; li < L; ++li) {
        Layer& ly = m->layers[li];
        const int blk = ly.blk;
        const int32_t* rows = rows_ptr(m, set, li);
        // layer 1 reads the feature table (local or row-sharded over peers); later layers H_{l-1}
        const FeatRows Hrows = li == 0 ? g->rows()
                                       : FeatRows{m->layers[li - 1].H, nullptr, 0, nullptr, 0, m->layers[li - 1].m_cap};
        const int kid = li == 0 ? GNN_K_AGG_L1 : GNN_K_AGG;
        const int32_t* self_ids = li == 0 ? B.nodes : nullptr;
        // the last layer of SAGE + neighbour gathers its A inside k_last_layer (no aggregation launch)
        const bool agg_in_last = li == L - 1 && li > 0 && fused_last(m) && m->sage && !m->shadow;
        if (li == 0 && m->l1_on_sampler) {
            // gathered by the sampling stream (issue_sample) before B.sampled was recorded
        } else if (agg_in_last) {
        } else if (m->shadow) {
            K(m, s, kid, [&] { bal(false, li, rows); });
        } else if (m->sage) {
            // layer 1 of the neighbour sampler reads X rows directly by global neighbour id
            const bool direct = li == 0 && !m->shadow;
            // the training-only sampling run writes the last hop fixed-stride (no count scan)
            const int fixed_k = direct && !m->full_train ? m->bs[set].sp.hop[blk].k : 0;
            K(m, s, kid, [&] {
                launch_agg_sage(rows, Hrows, ly.in_pad, direct ? nullptr : self_ids, self_ids, B.rowptr[blk],
                                direct ? B.nbr[blk] : B.col[blk], ly.A, fixed_k, m->bs[set].sp.hop[blk].k, s);
            });
        } else {
            K(m, s, kid, [&] {
                launch_agg_gcn(rows, &B.st->n_dst[blk], Hrows, ly.in_pad, ly.k_pad, self_ids, self_ids,
                               B.rowptr[blk], B.col[blk], B.trowptr[blk], ly.A, s);
            });
        }
        if (li == 0 && m->sample_after_l1) {   // the next batch's sampling may start now (see issue_sample)
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            cudaStreamIsCapturing(s, &cs);
            cudaEventRecordWithFlags(B.l1done, s, cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal
                                                                                    : cudaEventRecordDefault);
        }
        if (li == L - 1 && fused_last(m)) {
            // logits, cross-entropy and dA = dZ W^T in one CUDA-core pass (dense.cu k_last_layer)
            K(m, s, GNN_K_CE, [&] {
                launch_last_layer(rows, (int)ly.m_cap, ly.A, ly.k_pad, ly.in, ly.in_pad, m->sage, m->params + ly.poff,
                                  g->C, ly.n_pad, ly.H, ly.dPre, ly.dA, B.st, g->y, B.nodes,
                                  agg_in_last ? m->layers[li - 1].H : nullptr, B.rowptr[blk], B.col[blk], s);
            });
            break;
        }
        if (li == L - 1 && ly.n_pad <= 64) {
            // logits = A W with the softmax cross-entropy in the GEMM epilogue
            K(m, s, GNN_K_GEMM_FWD, [&] {
                launch_gemm_tc_ce(m->bf16x3, fwd_map(m, ly, li, set), rows, (int)ly.m_cap, ly.n_pad, ly.k_pad, ly.H, B.st, g->C,
                                  g->y, B.nodes, ly.dPre, s);
            });
            break;
        }
        // Pre = A W (+ReLU) -> H (fp32)
        K(m, s, GNN_K_GEMM_FWD, [&] {
            launch_gemm_tc(2, m->bf16x3, fwd_map(m, ly, li, set), rows, 0, (int)ly.m_cap, ly.n_pad, ly.k_pad, ly.H, ly.n_pad,
                           ly.n_pad, li < L - 1, 1, 0, s, ly.hmask, ly.mask_ld);
        });
        if (li == L - 1) {   // ---- loss (wide logits rows: separate kernel)
            K(m, s, GNN_K_CE, [&] { launch_ce(B.st, ly.H, ly.n_pad, g->C, g->y, B.nodes, ly.dPre, s); });
        }
    }
    // ---- backward.  The weight gradients are off the critical path (nothing in the step reads
    // them before the update): they run on a forked stream as soon as their dPre is ready,
    // concurrently with the dgrad -> backward-aggregation chain, and join before the update.
    cudaStream_t ws = m->wstream;
    const bool nccl = uses_nccl(m), peer = m->exchange == GNN_EXCH_PEER, host = uses_host(m);
    for (int li = L - 1; li >= 0; --li) {
        Layer& ly = m->layers[li];
        const int32_t* rows = rows_ptr(m, set, li);
        const int64_t stride = (int64_t)ly.k_pad * ly.n_pad;
        cudaEventRecord(m->ev_dpre[li], s);
        cudaStreamWaitEvent(ws, m->ev_dpre[li], 0);
        // dW = A^T dPre (deterministic split over rows)
        K(m, ws, GNN_K_GEMM_WGRAD, [&] {
            launch_gemm_tc(1, m->bf16x3, wgrad_map(m, ly, li, set), rows, ly.k_pad, ly.k_pad, ly.n_pad, 0, ly.wpart, ly.n_pad,
                           ly.n_pad, false, ly.splits, stride, ws);
        });
        // the exchange of layer li's gradient starts now, while the backward of the layers below
        // runs on the training stream (per-layer buckets, §4.1: overlap)
        if (nccl) {
            K(m, ws, GNN_K_ALLREDUCE, [&] {
                launch_wgrad_reduce(pack_desc(m), li, li + 1, m->grads, PeerX{}, ws);
                ncclAllReduce(m->grads + ly.poff, m->grads + ly.poff, (size_t)ly.pcnt, ncclFloat, ncclSum, m->comm, ws);
            });
        } else if (host) {   // this layer's reduced gradient, for the caller's all-reduce
            K(m, ws, GNN_K_ALLREDUCE, [&] { launch_wgrad_reduce(pack_desc(m), li, li + 1, m->grads, PeerX{}, ws); });
        } else if (peer) {
            PeerX x = m->px;
            x.signal = li == 0;   // the last bucket publishes the step
            K(m, ws, GNN_K_ALLREDUCE, [&] { launch_wgrad_reduce(pack_desc(m), li, li + 1, nullptr, x, ws); });
        }
        if (li == 0) break;
        // dA = dPre W^T (fp32); the fused last layer computed it already
        if (!(li == L - 1 && fused_last(m))) K(m, s, GNN_K_GEMM_DGRAD, [&] {
            launch_gemm_tc(0, m->bf16x3, ly.map_dgrad, rows, 0, (int)ly.m_cap, ly.k_pad, ly.n_pad, ly.dA, ly.k_pad,
                           ly.k_pad, false, 1, 0, s);
        });
        Layer& prev = m->layers[li - 1];
        const int blk = ly.blk;
        if (m->shadow) K(m, s, GNN_K_SPMM_BWD, [&] { bal(true, li, rows); });
        else K(m, s, GNN_K_SPMM_BWD, [&] {
            launch_spmm_bwd(!m->sage, blk, B.st, rows, ly.dA, ly.in_pad, B.rowptr[blk], B.trowptr[blk], B.tdst_s[blk],
                            prev.hmask, prev.mask_ld, prev.dPre, s);
        });
    }
    cudaEventRecord(m->ev_join, ws);
    cudaStreamWaitEvent(s, m->ev_join, 0);
    if (host) {
        // ---- no update here: gnn_apply_update after the caller's all-reduce
    } else if (nccl) {
        // ---- every layer's bucket is all-reduced: update
        K(m, s, GNN_K_SGD, [&] { launch_sgd_pack(pack_desc(m), m->params, m->grads, m->cfg.lr, false, m->opt, s); });
    } else if (peer) {
        // ---- wait for every rank's gradient, sum the inbox in rank order, update
        K(m, s, GNN_K_SGD, [&] {
            launch_sgd_pack(pack_desc(m), m->params, m->grads, m->cfg.lr, false, m->opt, s, m->px);
        });
    } else {
        // ---- one rank: the reduce of the partials is fused into the update
        K(m, s, GNN_K_SGD, [&] { launch_sgd_pack(pack_desc(m), m->params, m->grads, m->cfg.lr, true, m->opt, s); });
    }
}

// Capture the training body of batch set `set` once.  With profiling on, the capture also
// records an event pair around every kernel-class launch (event-record nodes).
gnn_status build_graph(gnn_model* m, int set, bool prof) {
    BatchSet& B = m->bs[set];
    cudaGraphExec_t* target = prof ? &B.prof_gexec : &B.gexec;
    if (*target) return GNN_OK;
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(m->stream, cudaStreamCaptureModeThreadLocal));
    const size_t before = m->pending.size();
    enqueue_training(m, set);
    if (prof) {
        B.prof_pairs.assign(m->pending.begin() + before, m->pending.end());
        m->pending.resize(before);
    }
    cudaError_t e = cudaStreamEndCapture(m->stream, &graph);
    if (e != cudaSuccess) return fail(GNN_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    size_t n = 0;
    CK(cudaGraphGetNodes(graph, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    CK(cudaGraphGetNodes(graph, nodes.data(), &n));
    int64_t kernels = 0;
    for (auto nd : nodes) {
        cudaGraphNodeType t;
        cudaGraphNodeGetType(nd, &t);
        if (t == cudaGraphNodeTypeKernel) ++kernels;
    }
    if (!prof) m->launches_per_step = kernels + 1;   // + k_sample_step (sampling stream)
    CK(cudaGraphInstantiate(target, graph, 0));
    CK(cudaGraphDestroy(graph));
    return GNN_OK;
}

void drop_graphs(gnn_model* m) {
    for (auto& B : m->bs) {
        if (B.gexec) { cudaGraphExecDestroy(B.gexec); B.gexec = nullptr; }
        if (B.prof_gexec) { cudaGraphExecDestroy(B.prof_gexec); B.prof_gexec = nullptr; }
    }
}

// Checked before a batch is sampled into a set (a started batch must be trainable).
gnn_status check_ready(gnn_model* m) {
    if (m->g->nshards && !m->g->shard_ptrs)
        return fail(GNN_ERR_STATE, "row-sharded features: call gnn_shard_import before training");
    if (uses_nccl(m) && !m->comm) {
        if (m->world > 1) return fail(GNN_ERR_STATE, "world > 1 without a communicator (gnn_comm_init)");
        ncclUniqueId id;   // GNN_EXCH_NCCL on one rank: a communicator of one
        CKN(ncclGetUniqueId(&id));
        CKN(ncclCommInitRank(&m->comm, 1, id, 0));
        (void)cudaGetLastError();   // NCCL's probing may leave a stale runtime error
    }
    return GNN_OK;
}

gnn_status ensure_perm(gnn_model* m, int64_t epoch) {   // on the sampling stream
    if (m->perm_epoch == epoch) return GNN_OK;
    if (m->n_train > 0) {
        launch_perm_keys(m->train_sorted, m->n_train, m->cfg.seed, epoch, m->keys, m->sstream);
        size_t bytes = m->cub_bytes;
        CK(cub::DeviceRadixSort::SortPairs(m->cub_tmp, bytes, m->keys, m->keys_alt, m->train_sorted, m->perm,
                                           (int)m->n_train, 0, 64, m->sstream));
    }
    m->perm_epoch = epoch;
    return GNN_OK;
}

int64_t num_batches(const gnn_model* m) {
    return (m->n_train + m->cfg.batch_size - 1) / m->cfg.batch_size;
}

int64_t steps_per_epoch(const gnn_model* m) {
    return (num_batches(m) + m->world - 1) / m->world;
}

gnn_status set_device(int dev) {
    CK(cudaSetDevice(dev));
    // every API call starts here: drop a stale error another library left in the runtime's
    // per-thread "last error" (NCCL's device probing leaves cudaErrorInvalidDevice behind), so
    // the launch checks below see only this call's launches
    (void)cudaGetLastError();
    return GNN_OK;
}

// Batch -> rank rule of synchronous SGD (R8/R9; §2.2).
void plan_step(int64_t n_train, int64_t B, int64_t world, int64_t rank, int64_t step, int64_t* g, int32_t* n,
               int64_t* offset, int32_t* b_total) {
    const int64_t nb = (n_train + B - 1) / B;
    *g = step * world + rank;
    *n = *g < nb ? (int32_t)std::min<int64_t>(B, n_train - *g * B) : 0;
    *offset = *g * B;
    const int64_t done = step * world * B;
    *b_total = (int32_t)std::max<int64_t>(0, std::min<int64_t>(n_train - done, world * B));
}

// Sample a batch into set `set` on the sampling stream (after the set's previous training).
// seeds_dev: device seed list (the epoch permutation slice) or nullptr with seeds_host.
gnn_status issue_sample(gnn_model* m, int set, const int32_t* seeds_dev, const int32_t* seeds_host, int32_t n,
                        int32_t b_total, int64_t epoch, int64_t g, bool full) {
    BatchSet& B = m->bs[set];
    if (B.trained_once) CK(cudaStreamWaitEvent(m->sstream, B.trained, 0));
    // A/B diagnostic GS_SERIAL=1: sampling never runs concurrently with training (it also waits for
    // the step trained last, whichever set it used)
    static const bool serial = [] { const char* e = std::getenv("GS_SERIAL"); return e && e[0] == '1'; }();
    if (serial && m->last >= 0 && m->bs[m->last].trained_once) CK(cudaStreamWaitEvent(m->sstream, m->bs[m->last].trained, 0));
    if (m->sample_after_l1 && m->last >= 0 && m->last != set && m->bs[m->last].trained_once)
        CK(cudaStreamWaitEvent(m->sstream, m->bs[m->last].l1done, 0));
    const int32_t* src = seeds_dev;
    if (!src) {
        if (n) {
            CK(cudaEventSynchronize(B.sampled));   // the staging slot's previous copy is done
            std::memcpy(B.seeds_stage, seeds_host, sizeof(int32_t) * n);
            CK(cudaMemcpyAsync(B.seeds_in, B.seeds_stage, sizeof(int32_t) * n, cudaMemcpyHostToDevice, m->sstream));
        }
        src = B.seeds_in;
    }
    SampleParams sp = B.sp;
    sp.seed_src = src;
    sp.n_seeds = n;
    sp.b_total = b_total;
    sp.epoch = (uint32_t)epoch;
    sp.g = (uint32_t)g;
    if (++m->seq == 0) m->seq = 1;   // 32-bit scan-word tag, never 0
    sp.tag = m->seq;
    sp.full = full ? 1 : 0;
    m->last_full = full;
    cudaEvent_t ta = nullptr, tb = nullptr;
    if (m->timeline) { ta = take_event(m); tb = take_event(m); CK(cudaEventRecord(ta, m->sstream)); }
    K(m, m->sstream, GNN_K_SAMPLE, [&] { launch_sample_step(sp, m->sstream); });
    if (m->l1_on_sampler && !full) {
        // layer 1's fused gather + mean of this batch (its fixed-stride last hop, X by global id)
        const Layer& ly = m->layers[0];
        const int blk = ly.blk;
        K(m, m->sstream, GNN_K_AGG_L1, [&] {
            launch_agg_sage(rows_ptr(m, set, 0), m->g->rows(), ly.in_pad, nullptr, B.nodes, B.rowptr[blk], B.nbr[blk],
                            set == 1 ? ly.A1 : ly.A, B.sp.hop[blk].k, B.sp.hop[blk].k, m->sstream);
        });
    }
    if (m->timeline) { CK(cudaEventRecord(tb, m->sstream)); m->tl_sample.emplace_back(ta, tb); }
    CK(cudaGetLastError());
    CK(cudaEventRecord(B.sampled, m->sstream));
    B.valid = true;
    B.host_seeds = seeds_dev == nullptr;
    B.epoch = epoch;
    B.g = g;
    B.n = n;
    B.b_total = b_total;
    return GNN_OK;
}

// The batch this rank trains at `step`: the engine's rule (plan_step), or the workload-balanced
// schedule set with gnn_set_schedule (reading R8 with the batch order of NEXT-3).
gnn_status plan_model_step(const gnn_model* m, int64_t step, int64_t* g, int32_t* n, int64_t* offset, int32_t* b_total) {
    if (m->schedule.empty()) {
        plan_step(m->n_train, m->cfg.batch_size, m->world, m->rank, step, g, n, offset, b_total);
        return GNN_OK;
    }
    const int64_t B = m->cfg.batch_size, nb = (int64_t)m->schedule.size();
    if (nb != num_batches(m)) return fail(GNN_ERR_STATE, "schedule does not cover the current batches (set it again)");
    auto seeds = [&](int64_t gg) { return (int32_t)std::min<int64_t>(B, m->n_train - gg * B); };
    const int64_t i = step * m->world + m->rank;
    *g = i < nb ? m->schedule[i] : nb + i;   // past the end: inactive (joins the exchange with zeros)
    *n = i < nb ? seeds(*g) : 0;
    *offset = i < nb ? *g * B : 0;
    int64_t bt = 0;
    for (int64_t r = 0; r < m->world; ++r)
        if (step * m->world + r < nb) bt += seeds(m->schedule[step * m->world + r]);
    *b_total = (int32_t)bt;
    return GNN_OK;
}

gnn_status issue_sample_step(gnn_model* m, int set, int64_t epoch, int64_t step) {
    TRY(ensure_perm(m, epoch));
    int64_t g, offset;
    int32_t n, b_total;
    TRY(plan_model_step(m, step, &g, &n, &offset, &b_total));
    return issue_sample(m, set, n > 0 ? m->perm + offset : m->perm, nullptr, n, b_total, epoch, g, m->full_train);
}

// The set holding this batch, if one was prefetched.  A set sampled from host seeds serves only a
// host-seeded call with the same seeds (compared with the pinned staging copy), and a set sampled
// from the epoch permutation only a permutation-driven step.
int find_set(gnn_model* m, int64_t epoch, int64_t g, int32_t n, int32_t b_total, const int32_t* seeds_host = nullptr) {
    for (int k = 0; k < 2; ++k) {
        const BatchSet& B = m->bs[k];
        if (!B.valid || B.epoch != epoch || B.g != g || B.n != n || B.b_total != b_total) continue;
        if (B.host_seeds != (seeds_host != nullptr)) continue;
        if (seeds_host && n && std::memcmp(B.seeds_stage, seeds_host, sizeof(int32_t) * n) != 0) continue;
        return k;
    }
    return -1;
}

// Host seeds must be node ids in [0, N) without repeats: the sampling kernel indexes the CSR and
// the node map with them (an out-of-range id would write outside device memory).
gnn_status check_seeds(const gnn_model* m, const int32_t* seeds, int32_t n) {
    thread_local std::vector<int32_t> tmp;
    tmp.assign(seeds, seeds + n);
    std::sort(tmp.begin(), tmp.end());
    for (int32_t i = 0; i < n; ++i) {
        if (tmp[i] < 0 || tmp[i] >= m->g->N) return fail(GNN_ERR_RANGE, "seed id " + std::to_string(tmp[i]) + " out of [0, N)");
        if (i && tmp[i] == tmp[i - 1]) return fail(GNN_ERR_PARAM, "duplicate seed id " + std::to_string(tmp[i]));
    }
    return GNN_OK;
}

int other_set(gnn_model* m) { return m->last < 0 ? 0 : 1 - m->last; }

// Train the batch held by `set` on the model's stream.
// loss_dst (nullable, host or device): the batch's loss is copied there on the training stream
// before the set is released for resampling (its StepState is reset by the next sampling).
gnn_status train_set(gnn_model* m, int set, float* loss_dst = nullptr) {
    BatchSet& B = m->bs[set];
    CK(cudaStreamWaitEvent(m->stream, B.sampled, 0));
    cudaEvent_t ta = nullptr, tb = nullptr;
    if (m->timeline) { ta = take_event(m); tb = take_event(m); CK(cudaEventRecord(ta, m->stream)); }
    if (m->cfg.use_graph && !m->profiling) {
        TRY(build_graph(m, set, false));
        CK(cudaGraphLaunch(B.gexec, m->stream));
    } else if (m->cfg.use_graph) {
        // instrumented replay: the same graph body with event-record nodes; read them back now
        TRY(build_graph(m, set, true));
        CK(cudaGraphLaunch(B.prof_gexec, m->stream));
        CK(cudaStreamSynchronize(m->stream));
        drain_profile(m);                       // the sampling kernel's pair (eager)
        for (auto& p : B.prof_pairs) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, p.a, p.b));
            m->prof_ms[p.kid] += ms;
            m->prof_n[p.kid] += 1;
        }
    } else {
        enqueue_training(m, set);
        CK(cudaGetLastError());
    }
    if (m->timeline) { CK(cudaEventRecord(tb, m->stream)); m->tl_train.emplace_back(ta, tb); }
    if (loss_dst) CK(cudaMemcpyAsync(loss_dst, &B.st->loss, sizeof(float), cudaMemcpyDefault, m->stream));
    CK(cudaEventRecord(B.trained, m->stream));
    B.trained_once = true;
    B.valid = false;
    m->last = set;
    return GNN_OK;
}

// One step of the epoch loop: use the prefetched sample if it is this step's batch, prefetch
// the next step's batch into the other set, train.
gnn_status step_from_perm(gnn_model* m, int64_t epoch, int64_t step, float* loss_dst = nullptr) {
    int64_t g, offset;
    int32_t n, b_total;
    TRY(plan_model_step(m, step, &g, &n, &offset, &b_total));
    int cur = find_set(m, epoch, g, n, b_total);
    ++(cur < 0 ? m->reuse_misses : m->reuse_hits);
    if (cur < 0) {
        cur = other_set(m);
        TRY(issue_sample_step(m, cur, epoch, step));
    }
    // training is enqueued first, the next step's sampling after it: the GPU then never waits
    // for the host between steps (the sampling runs while the host comes back for the next call)
    TRY(train_set(m, cur, loss_dst));
    if (m->overlap && !m->profiling && step + 1 < steps_per_epoch(m)) TRY(issue_sample_step(m, 1 - cur, epoch, step + 1));
    return GNN_OK;
}

gnn_status sync_all(gnn_model* m) {
    CK(cudaStreamSynchronize(m->sstream));
    CK(cudaStreamSynchronize(m->stream));
    return GNN_OK;
}

gnn_status copy_state(gnn_model* m, int set, StepState* out) {
    TRY(sync_all(m));
    CK(cudaMemcpy(out, m->bs[set].st, sizeof(StepState), cudaMemcpyDeviceToHost));
    return GNN_OK;
}

int shown_set(gnn_model* m) { return m->last < 0 ? 0 : m->last; }
}  // namespace

// ====================================================================== C ABI
extern "C" {

const char* gnn_last_error(void) { return g_err.c_str(); }
int32_t gnn_abi_version(void) { return GNN_ABI_VERSION; }

static gnn_status graph_create(int64_t num_nodes, const int64_t* row_ptr_host, const int32_t* col_idx_host,
                               int32_t feat_dim, int32_t feat_stride, const float* features_host,
                               const int32_t* labels_host, int32_t num_classes, int32_t device, int32_t nshards,
                               int32_t shard, gnn_graph** out);

gnn_status gnn_graph_create(int64_t num_nodes, const int64_t* row_ptr_host, const int32_t* col_idx_host,
                            int32_t feat_dim, int32_t feat_stride, const float* features_host,
                            const int32_t* labels_host, int32_t num_classes, int32_t device, gnn_graph** out) {
    Range nvtx_("gnn_graph_create");
    return graph_create(num_nodes, row_ptr_host, col_idx_host, feat_dim, feat_stride, features_host, labels_host,
                        num_classes, device, 1, 0, out);
}

gnn_status gnn_graph_create_sharded(int64_t num_nodes, const int64_t* row_ptr_host, const int32_t* col_idx_host,
                                    int32_t feat_dim, int32_t feat_stride, int32_t nshards, int32_t shard,
                                    const float* shard_features_host, const int32_t* labels_host,
                                    int32_t num_classes, int32_t device, gnn_graph** out) {
    if (nshards < 1 || shard < 0 || shard >= nshards) return fail(GNN_ERR_PARAM, "bad shard index");
    return graph_create(num_nodes, row_ptr_host, col_idx_host, feat_dim, feat_stride, shard_features_host,
                        labels_host, num_classes, device, nshards, shard, out);
}

gnn_status gnn_shard_export(gnn_graph* g, uint8_t handle_out_host[64]) {
    if (!g || !handle_out_host) return fail(GNN_ERR_PARAM, "NULL argument");
    TRY(set_device(g->dev));
    cudaIpcMemHandle_t h;
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    CK(cudaIpcGetMemHandle(&h, g->X));
    std::memcpy(handle_out_host, &h, 64);
    return GNN_OK;
}

gnn_status gnn_cache_rows(gnn_graph* g, const int32_t* ids_host, int64_t n) {
    if (!g || (n > 0 && !ids_host) || n < 0) return fail(GNN_ERR_PARAM, "bad arguments");
    if (g->nshards < 1) return fail(GNN_ERR_STATE, "graph is not sharded");
    if (!g->shard_ptrs) return fail(GNN_ERR_STATE, "gnn_cache_rows needs gnn_shard_import first");
    TRY(set_device(g->dev));
    std::vector<char> seen(n ? g->N : 0, 0);
    for (int64_t i = 0; i < n; ++i) {
        const int32_t v = ids_host[i];
        if (v < 0 || v >= g->N) return fail(GNN_ERR_RANGE, "cache row id out of range");
        if (v >= g->row_begin && v < g->row_end) return fail(GNN_ERR_PARAM, "cache row " + std::to_string(v) + " is local");
        if (seen[v]) return fail(GNN_ERR_PARAM, "duplicate cache row id");
        seen[v] = 1;
    }
    CK(cudaDeviceSynchronize());   // no kernel may be reading the previous cache
    unsigned long long* stats = g->stats_on ? g->cache_stats : nullptr;
    FeatCache off{nullptr, nullptr, stats};
    CK(cudaMemcpy(g->cache_desc, &off, sizeof(FeatCache), cudaMemcpyHostToDevice));
    if (g->cache_rows) { cudaFree(g->cache_rows); g->cache_rows = nullptr; }
    g->cache_n = 0;
    if (n == 0) return GNN_OK;
    if (!g->cmap) {
        CK(cudaMalloc(&g->cmap, sizeof(int32_t) * g->N));
    }
    CK(cudaMemset(g->cmap, 0xff, sizeof(int32_t) * g->N));
    int32_t* ids_dev = nullptr;
    CK(cudaMalloc(&ids_dev, sizeof(int32_t) * n));
    CK(cudaMalloc(&g->cache_rows, sizeof(float) * n * g->stride));
    CK(cudaMemcpy(ids_dev, ids_host, sizeof(int32_t) * n, cudaMemcpyHostToDevice));
    launch_cache_fill(g->rows(), ids_dev, n, g->stride, g->cache_rows, nullptr);
    std::vector<int32_t> slots(g->N, -1);
    for (int64_t i = 0; i < n; ++i) slots[ids_host[i]] = (int32_t)i;
    CK(cudaMemcpy(g->cmap, slots.data(), sizeof(int32_t) * g->N, cudaMemcpyHostToDevice));
    CK(cudaDeviceSynchronize());
    cudaFree(ids_dev);
    FeatCache on{g->cmap, g->cache_rows, stats};
    CK(cudaMemcpy(g->cache_desc, &on, sizeof(FeatCache), cudaMemcpyHostToDevice));
    g->cache_n = n;
    return GNN_OK;
}

gnn_status gnn_cache_stats(gnn_graph* g, int32_t enable, int64_t* counts_out_host) {
    if (!g) return fail(GNN_ERR_PARAM, "NULL graph");
    if (g->nshards < 1) return fail(GNN_ERR_STATE, "graph is not sharded");
    TRY(set_device(g->dev));
    CK(cudaDeviceSynchronize());   // the counts of every step enqueued so far
    unsigned long long h[3] = {0, 0, 0};
    CK(cudaMemcpy(h, g->cache_stats, sizeof(h), cudaMemcpyDeviceToHost));
    if (counts_out_host)
        for (int i = 0; i < 3; ++i) counts_out_host[i] = (int64_t)h[i];
    if (enable >= 0) {
        CK(cudaMemset(g->cache_stats, 0, 3 * sizeof(unsigned long long)));
        g->stats_on = enable != 0;
        // the descriptor lives at a fixed address: captured steps see the switch
        unsigned long long* stats = g->stats_on ? g->cache_stats : nullptr;
        CK(cudaMemcpy(reinterpret_cast<char*>(g->cache_desc) + offsetof(FeatCache, stats), &stats, sizeof(stats),
                      cudaMemcpyHostToDevice));
    }
    return GNN_OK;
}

gnn_status gnn_cache_plan_by_degree(const int64_t* row_ptr_host, int64_t num_nodes, int32_t nshards, int32_t shard,
                                    int64_t capacity, int32_t* ids_out_host, int64_t* n_out_host) {
    if (!row_ptr_host || !ids_out_host || !n_out_host || num_nodes < 0 || nshards < 1 || shard < 0 ||
        shard >= nshards || capacity < 0)
        return fail(GNN_ERR_PARAM, "bad arguments");
    const int64_t rps = (num_nodes + nshards - 1) / nshards;
    const int64_t b = std::min<int64_t>(num_nodes, (int64_t)shard * rps), e = std::min<int64_t>(num_nodes, b + rps);
    std::vector<int32_t> cand;
    cand.reserve(num_nodes - (e - b));
    for (int64_t v = 0; v < num_nodes; ++v)
        if (v < b || v >= e) cand.push_back((int32_t)v);
    auto deg = [&](int32_t v) { return row_ptr_host[v + 1] - row_ptr_host[v]; };
    const int64_t k = std::min<int64_t>(capacity, (int64_t)cand.size());
    // hottest rows: highest degree first (a node is sampled about in proportion to its degree), ties by id
    std::partial_sort(cand.begin(), cand.begin() + k, cand.end(), [&](int32_t a, int32_t c) {
        return deg(a) != deg(c) ? deg(a) > deg(c) : a < c;
    });
    std::sort(cand.begin(), cand.begin() + k);
    std::copy(cand.begin(), cand.begin() + k, ids_out_host);
    *n_out_host = k;
    return GNN_OK;
}

gnn_status gnn_shard_import(gnn_graph* g, const uint8_t* handles_host) {
    if (!g || !handles_host) return fail(GNN_ERR_PARAM, "NULL argument");
    if (g->nshards < 1) return fail(GNN_ERR_STATE, "graph is not sharded");
    TRY(set_device(g->dev));
    std::vector<const float*> ptrs(g->nshards, nullptr);
    const int mine = (int)(g->row_begin / g->rps);
    for (int s = 0; s < g->nshards; ++s) {
        if (s == mine) { ptrs[s] = g->X; continue; }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handles_host + 64 * s, 64);
        void* p = nullptr;
        CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        g->ipc_opened.push_back(p);
        ptrs[s] = static_cast<const float*>(p);
    }
    if (!g->shard_ptrs) {
        gnn_status st = dalloc(&g->shard_ptrs, g->nshards, g->owned);
        if (st != GNN_OK) return st;
    }
    CK(cudaMemcpy(g->shard_ptrs, ptrs.data(), sizeof(float*) * g->nshards, cudaMemcpyHostToDevice));
    return GNN_OK;
}

static gnn_status graph_create(int64_t num_nodes, const int64_t* row_ptr_host, const int32_t* col_idx_host,
                               int32_t feat_dim, int32_t feat_stride, const float* features_host,
                               const int32_t* labels_host, int32_t num_classes, int32_t device, int32_t nshards,
                               int32_t shard, gnn_graph** out) {
    if (!out) return fail(GNN_ERR_PARAM, "out is NULL");
    *out = nullptr;
    if (num_nodes <= 0 || num_nodes >= INT32_MAX) return fail(GNN_ERR_PARAM, "num_nodes out of (0, 2^31-1)");
    if (!row_ptr_host || !features_host || !labels_host) return fail(GNN_ERR_PARAM, "NULL input array");
    if (feat_dim <= 0 || feat_stride < feat_dim || feat_stride % 4) return fail(GNN_ERR_PARAM, "feat_stride must be >= feat_dim and a multiple of 4");
    if (num_classes <= 0) return fail(GNN_ERR_PARAM, "num_classes must be > 0");
    if (row_ptr_host[0] != 0) return fail(GNN_ERR_SHAPE, "row_ptr[0] != 0");
    for (int64_t v = 0; v < num_nodes; ++v)
        if (row_ptr_host[v + 1] < row_ptr_host[v]) return fail(GNN_ERR_SHAPE, "row_ptr not non-decreasing at " + std::to_string(v));
    const int64_t nnz = row_ptr_host[num_nodes];
    if (nnz > 0 && !col_idx_host) return fail(GNN_ERR_PARAM, "col_idx is NULL");
    for (int64_t v = 0; v < num_nodes; ++v)
        for (int64_t p = row_ptr_host[v]; p < row_ptr_host[v + 1]; ++p) {
            const int32_t c = col_idx_host[p];
            if (c < 0 || c >= num_nodes) return fail(GNN_ERR_RANGE, "col_idx out of range at " + std::to_string(p));
            if (p > row_ptr_host[v] && c <= col_idx_host[p - 1]) return fail(GNN_ERR_SHAPE, "row " + std::to_string(v) + " not ascending/duplicate-free");
        }
    for (int64_t v = 0; v < num_nodes; ++v)
        if (labels_host[v] < 0 || labels_host[v] >= num_classes) return fail(GNN_ERR_RANGE, "label out of range at " + std::to_string(v));
    TRY(set_device(device));
    auto* g = new gnn_graph();
    g->dev = device; g->N = num_nodes; g->nnz = nnz; g->F = feat_dim; g->stride = feat_stride; g->C = num_classes;
    g->rps = (num_nodes + nshards - 1) / nshards;      // uniform row blocks (config 4 sharding)
    g->row_begin = std::min<int64_t>(num_nodes, (int64_t)shard * g->rps);
    g->row_end = std::min<int64_t>(num_nodes, g->row_begin + g->rps);
    g->nshards = nshards > 1 ? nshards : 0;
    const int64_t local_rows = g->row_end - g->row_begin;
    auto cleanup = [&](gnn_status s) { for (void* p : g->owned) cudaFree(p); delete g; return s; };
    gnn_status s;
    if ((s = dalloc(&g->row_ptr, num_nodes + 1, g->owned)) != GNN_OK) return cleanup(s);
    if ((s = dalloc(&g->col, nnz, g->owned)) != GNN_OK) return cleanup(s);
    if ((s = dalloc(&g->X, std::max<int64_t>(local_rows, 1) * feat_stride, g->owned)) != GNN_OK) return cleanup(s);
    if ((s = dalloc(&g->y, num_nodes, g->owned)) != GNN_OK) return cleanup(s);
    cudaError_t e = cudaMemcpy(g->row_ptr, row_ptr_host, sizeof(int64_t) * (num_nodes + 1), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && nnz) e = cudaMemcpy(g->col, col_idx_host, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && local_rows)
        e = cudaMemcpy(g->X, features_host, sizeof(float) * local_rows * feat_stride, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(g->y, labels_host, sizeof(int32_t) * num_nodes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && feat_stride > feat_dim && local_rows)   // padding columns are zero (DESIGN.md layout)
        e = cudaMemset2D(g->X + feat_dim, sizeof(float) * feat_stride, 0, sizeof(float) * (feat_stride - feat_dim),
                         local_rows);
    if (e != cudaSuccess) return cleanup(fail(GNN_ERR_CUDA, std::string("graph upload: ") + cudaGetErrorString(e)));
    if (g->nshards) {   // the NEXT-2 cache descriptor (empty) and its counters, at fixed addresses
        if ((s = dalloc(&g->cache_desc, 1, g->owned)) != GNN_OK) return cleanup(s);
        if ((s = dalloc(&g->cache_stats, 3, g->owned)) != GNN_OK) return cleanup(s);
        e = cudaMemset(g->cache_desc, 0, sizeof(FeatCache));
        if (e == cudaSuccess) e = cudaMemset(g->cache_stats, 0, 3 * sizeof(unsigned long long));
        if (e != cudaSuccess) return cleanup(fail(GNN_ERR_CUDA, std::string("cache descriptor: ") + cudaGetErrorString(e)));
    }
    if (!check_symmetric(g->row_ptr, g->col, num_nodes, &g->symmetric))
        return cleanup(fail(GNN_ERR_CUDA, "symmetry check failed"));
    *out = g;
    return GNN_OK;
}

// Start address of the allocation holding p (driver entry point; the library links only cudart).
static bool alloc_base(const void* p, const void** base) {
    typedef int (*Fn)(unsigned long long*, size_t*, unsigned long long);
    static Fn fn = [] {
        void* q = nullptr;
        cudaDriverEntryPointQueryResult r;
        cudaGetDriverEntryPoint("cuMemGetAddressRange", &q, cudaEnableDefault, &r);
        return r == cudaDriverEntryPointSuccess ? (Fn)q : (Fn) nullptr;
    }();
    unsigned long long b = 0;
    size_t sz = 0;
    if (!fn || fn(&b, &sz, (unsigned long long)(uintptr_t)p) != 0) return false;
    *base = (const void*)(uintptr_t)b;
    return true;
}

gnn_status gnn_graph_create_device(int64_t num_nodes, const int64_t* row_ptr_dev, const int32_t* col_idx_dev,
                                   int32_t feat_dim, int32_t feat_stride, int32_t nshards, int32_t shard,
                                   const float* features_dev, const int32_t* labels_dev, int32_t num_classes,
                                   int32_t device, gnn_graph** out) {
    Range nvtx_("gnn_graph_create_device");
    if (!out) return fail(GNN_ERR_PARAM, "out is NULL");
    *out = nullptr;
    if (num_nodes <= 0 || num_nodes >= INT32_MAX) return fail(GNN_ERR_PARAM, "num_nodes out of (0, 2^31-1)");
    if (!row_ptr_dev || !col_idx_dev || !features_dev || !labels_dev) return fail(GNN_ERR_PARAM, "NULL input array");
    if (feat_dim <= 0 || feat_stride < feat_dim || feat_stride % 4) return fail(GNN_ERR_PARAM, "feat_stride must be >= feat_dim and a multiple of 4");
    if (num_classes <= 0) return fail(GNN_ERR_PARAM, "num_classes must be > 0");
    if (nshards < 1 || shard < 0 || shard >= nshards) return fail(GNN_ERR_PARAM, "bad shard index");
    TRY(set_device(device));
    for (const void* p : {(const void*)row_ptr_dev, (const void*)col_idx_dev, (const void*)features_dev, (const void*)labels_dev}) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, p) != cudaSuccess || a.type != cudaMemoryTypeDevice || a.device != device) {
            cudaGetLastError();
            return fail(GNN_ERR_PARAM, "input arrays must be device memory of the graph's device");
        }
    }
    if (nshards > 1) {   // the shard is exported by CUDA IPC, which maps whole allocations
        const void* b = nullptr;
        if (!alloc_base(features_dev, &b) || b != (const void*)features_dev)
            return fail(GNN_ERR_PARAM, "a sharded features_dev must be the start of its cudaMalloc allocation");
    }
    const int bad = validate_graph(row_ptr_dev, col_idx_dev, num_nodes, labels_dev, num_classes);
    if (bad < 0) return fail(GNN_ERR_CUDA, "graph validation kernel failed");
    if (bad & 1) return fail(GNN_ERR_SHAPE, "row_ptr[0] != 0 or row_ptr not non-decreasing");
    if (bad & 2) return fail(GNN_ERR_RANGE, "col_idx out of range");
    if (bad & 4) return fail(GNN_ERR_SHAPE, "a row is not ascending/duplicate-free");
    if (bad & 8) return fail(GNN_ERR_RANGE, "label out of range");
    int64_t nnz = 0;
    CK(cudaMemcpy(&nnz, row_ptr_dev + num_nodes, sizeof(int64_t), cudaMemcpyDeviceToHost));
    auto* g = new gnn_graph();
    g->dev = device; g->N = num_nodes; g->nnz = nnz; g->F = feat_dim; g->stride = feat_stride; g->C = num_classes;
    g->rps = (num_nodes + nshards - 1) / nshards;
    g->row_begin = std::min<int64_t>(num_nodes, (int64_t)shard * g->rps);
    g->row_end = std::min<int64_t>(num_nodes, g->row_begin + g->rps);
    g->nshards = nshards > 1 ? nshards : 0;
    // borrowed: referenced, never freed by the library
    g->row_ptr = const_cast<int64_t*>(row_ptr_dev);
    g->col = const_cast<int32_t*>(col_idx_dev);
    g->X = const_cast<float*>(features_dev);
    g->y = const_cast<int32_t*>(labels_dev);
    auto cleanup = [&](gnn_status st) { for (void* p : g->owned) cudaFree(p); delete g; return st; };
    if (g->nshards) {
        gnn_status st;
        if ((st = dalloc(&g->cache_desc, 1, g->owned)) != GNN_OK) return cleanup(st);
        if ((st = dalloc(&g->cache_stats, 3, g->owned)) != GNN_OK) return cleanup(st);
        cudaError_t e = cudaMemset(g->cache_desc, 0, sizeof(FeatCache));
        if (e == cudaSuccess) e = cudaMemset(g->cache_stats, 0, 3 * sizeof(unsigned long long));
        if (e != cudaSuccess) return cleanup(fail(GNN_ERR_CUDA, std::string("cache descriptor: ") + cudaGetErrorString(e)));
    }
    if (!check_symmetric(g->row_ptr, g->col, num_nodes, &g->symmetric))
        return cleanup(fail(GNN_ERR_CUDA, "symmetry check failed"));
    *out = g;
    return GNN_OK;
}

gnn_status gnn_graph_destroy(gnn_graph* g) {
    if (!g) return GNN_OK;
    cudaSetDevice(g->dev);
    for (void* p : g->ipc_opened) cudaIpcCloseMemHandle(p);
    for (void* p : g->owned) cudaFree(p);
    if (g->cmap) cudaFree(g->cmap);
    if (g->cache_rows) cudaFree(g->cache_rows);
    delete g;
    return GNN_OK;
}

gnn_status gnn_model_create(gnn_graph* g, const gnn_model_config* cfg, gnn_model** out) {
    Range nvtx_("gnn_model_create");
    if (!g || !cfg || !out) return fail(GNN_ERR_PARAM, "NULL argument");
    *out = nullptr;
    const gnn_model_config& c = *cfg;
    if (c.model != GNN_SAGE_MEAN && c.model != GNN_GCN) return fail(GNN_ERR_CONFIG, "unknown model");
    if (c.sampler != GNN_NEIGHBOR && c.sampler != GNN_SHADOW) return fail(GNN_ERR_CONFIG, "unknown sampler");
    if (c.num_layers < 1 || c.num_layers > kMaxHops) return fail(GNN_ERR_CONFIG, "num_layers must be 1..8");
    if (c.num_fanouts < 1 || c.num_fanouts > kMaxHops) return fail(GNN_ERR_CONFIG, "num_fanouts must be 1..8");
    if (c.sampler == GNN_NEIGHBOR && c.num_fanouts != c.num_layers) return fail(GNN_ERR_CONFIG, "neighbour sampler needs num_fanouts == num_layers");
    for (int i = 0; i < c.num_fanouts; ++i)
        if (c.fanouts[i] < 1 || c.fanouts[i] > 32) return fail(GNN_ERR_CONFIG, "fanouts must be 1..32");
    if (c.batch_size < 1 || c.batch_size > 1024) return fail(GNN_ERR_CONFIG, "batch_size must be 1..1024");
    if (c.num_layers > 1 && (c.hidden < 16 || c.hidden % 16)) return fail(GNN_ERR_CONFIG, "hidden must be a positive multiple of 16");
    if (c.precision != GNN_FP32 && c.precision != GNN_BF16_GEMM) return fail(GNN_ERR_CONFIG, "unknown precision");
    if (c.optimizer != GNN_SGD && c.optimizer != GNN_ADAM) return fail(GNN_ERR_CONFIG, "unknown optimizer");
    if (c.optimizer == GNN_ADAM && !(c.beta1 >= 0.f && c.beta1 < 1.f && c.beta2 >= 0.f && c.beta2 < 1.f && c.eps > 0.f))
        return fail(GNN_ERR_CONFIG, "Adam needs 0 <= beta1, beta2 < 1 and eps > 0");
    if (!(c.lr >= 0.f)) return fail(GNN_ERR_PARAM, "lr must be >= 0");
    TRY(set_device(g->dev));

    auto* m = new gnn_model();
    m->g = g; m->cfg = c;
    m->L = c.num_layers; m->hops = c.num_fanouts;
    m->sage = c.model == GNN_SAGE_MEAN; m->shadow = c.sampler == GNN_SHADOW;
    m->slot = m->shadow ? m->hops : -1;
    m->bf16x3 = c.precision == GNN_FP32;
    m->full_train = !(m->sage && !m->shadow);
    { const char* e = std::getenv("GS_L1_ON_SAMPLER"); m->l1_on_sampler = !m->full_train && e && e[0] == '1'; }
    { const char* e = std::getenv("GS_LAST_FUSED"); m->last_fused = e && e[0] == '1'; }
    auto cleanup = [&](gnn_status s) {
        for (void* p : m->owned) cudaFree(p);
        for (void* p : m->owned_host) cudaFreeHost(p);
        delete m;
        return s;
    };
    gnn_status s;
#define AL(p, n) do { if ((s = dalloc(&(p), (n), m->owned)) != GNN_OK) return cleanup(s); } while (0)

    // ---- capacities
    int64_t cap_dst = c.batch_size;
    for (int h = 0; h < m->hops; ++h) {
        HopBufs& b = m->hb[h];
        const int k = c.fanouts[m->hops - 1 - h];
        b.cap_dst = cap_dst;
        b.cap_edges = cap_dst * k;
        b.cap_src = std::min<int64_t>(g->N, cap_dst + b.cap_edges);
        b.cap_src = std::max(b.cap_src, cap_dst);
        b.need_t = !m->shadow && (!m->sage || h <= m->L - 2);
        // GCN's layer-1 block (the last hop) needs only d_out for its normalisation: no backward
        // aggregation runs over it, so its transposed block is not filled or sorted
        b.count_only = !m->shadow && !m->sage && h == m->hops - 1;
        cap_dst = b.cap_src;
    }
    m->nodes_cap = m->hb[m->hops - 1].cap_src;
    if (m->shadow) {
        HopBufs& b = m->hb[m->slot];
        b.cap_dst = b.cap_src = m->nodes_cap;
        b.cap_edges = std::max<int64_t>(1, g->nnz);
        // a symmetric graph induces a symmetric block: it is its own transpose (the backward
        // sums row u in the block's CSR order, a fixed order), so no transposed build/sort.
        // GS_SHADOW_TRANSPOSE=1 forces the transposed build (tests of that path).
        const char* ft = std::getenv("GS_SHADOW_TRANSPOSE");
        b.need_t = !g->symmetric || (ft && ft[0] == '1');
    }
    m->nwords = (g->N + 31) / 32;
    // shared sampling scratch (sampling runs are serialised on the sampling stream)
    AL(m->map, g->N);
    AL(m->bits, m->nwords);
    AL(m->icount, m->nodes_cap);
    {   // hub-row list of the transposed sort: rows longer than 256 entries, over all blocks
        int64_t cap = 3;
        for (int h = 0; h <= m->hops; ++h)
            if (m->hb[h].need_t && (h < m->hops || m->shadow)) cap += m->hb[h].cap_edges / 257 + 1;
        AL(m->hubs, cap);
    }
    const int sgrid = sample_step_grid();
    AL(m->status, (int64_t)sample_step_sites(m->hops) * sgrid);
    AL(m->bar, 1);
    CK(cudaMemset(m->status, 0, sizeof(unsigned long long) * sample_step_sites(m->hops) * sgrid));
    CK(cudaMemset(m->bar, 0, sizeof(GridBarrier)));
    CK(cudaMemset(m->map, 0xff, sizeof(int32_t) * g->N));
    CK(cudaMemset(m->bits, 0, sizeof(uint32_t) * m->nwords));
    for (int h = 0; h <= m->hops; ++h) {
        if (h == m->hops && !m->shadow) break;
        HopBufs& b = m->hb[h];
        if (b.need_t) {
            AL(b.tcount, b.cap_src + 1);
            AL(b.tcursor, b.cap_src + 1);
            if (!b.count_only) {
                AL(b.erow, b.cap_edges);
                AL(b.tdst, b.cap_edges);
            }
            CK(cudaMemset(b.tcount, 0, sizeof(int32_t) * (b.cap_src + 1)));
        }
    }
    // ---- the two batch sets
    for (int k = 0; k < 2; ++k) {
        BatchSet& B = m->bs[k];
        AL(B.st, 1);
        CK(cudaMemset(B.st, 0, sizeof(StepState)));
        AL(B.nodes, m->nodes_cap);
        AL(B.seeds_in, c.batch_size);
        CK(cudaMallocHost(&B.seeds_stage, sizeof(int32_t) * c.batch_size));
        m->owned_host.push_back(B.seeds_stage);
        CK(cudaEventCreateWithFlags(&B.sampled, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&B.trained, cudaEventDisableTiming));
        SampleParams& sp = B.sp;
        sp.st = B.st;
        sp.row_ptr = g->row_ptr;
        sp.col = g->col;
        sp.nodes = B.nodes;
        sp.map = m->map;
        sp.bits = m->bits;
        sp.nwords = (int)m->nwords;
        sp.seed = c.seed;
        sp.hops = m->hops;
        sp.shadow = m->shadow ? 1 : 0;
        sp.slot = m->shadow ? m->slot : -1;
        sp.icount = m->icount;
        sp.hubs = m->hubs;
        sp.status = m->status;
        sp.bar = m->bar;
        for (int h = 0; h <= m->hops; ++h) {
            if (h == m->hops && !m->shadow) break;
            HopBufs& b = m->hb[h];
            AL(B.rowptr[h], b.cap_dst + 1);
            AL(B.col[h], b.cap_edges);
            if (h < m->hops) AL(B.nbr[h], b.cap_edges);
            if (b.need_t) {
                AL(B.trowptr[h], b.cap_src + 1);
                if (!b.count_only) AL(B.tdst_s[h], b.cap_edges);
            }
            HopIO& io = sp.hop[h];
            io.k = h < m->hops ? c.fanouts[m->hops - 1 - h] : 0;
            io.rowptr = B.rowptr[h]; io.nbr = B.nbr[h]; io.col = B.col[h];
            io.tcount = b.need_t ? b.tcount : nullptr;
            io.trowptr = B.trowptr[h]; io.tcursor = b.tcursor; io.tdst = b.tdst; io.tdst_s = B.tdst_s[h];
            io.erow = b.need_t ? b.erow : nullptr;
            io.count_only = b.count_only ? 1 : 0;
        }
    }

    // ---- layers
    m->dims.push_back(g->F);
    for (int l = 1; l < m->L; ++l) m->dims.push_back(c.hidden);
    m->dims.push_back(g->C);
    int64_t poff = 0;
    for (int li = 0; li < m->L; ++li) {
        Layer ly;
        ly.in = m->dims[li];
        ly.out = m->dims[li + 1];
        // layer 1 reads the feature table in place: its padded width is the table's row stride
        ly.in_pad = li == 0 ? g->stride : (int)round_up(ly.in, 4);
        ly.rows = (m->sage ? 2 : 1) * ly.in;
        // GEMM reduction width; a multiple of 8 so bf16 rows are 16-byte strided (TMA)
        ly.k_pad = m->sage ? 2 * ly.in_pad : (int)round_up(ly.in_pad, 8);
        ly.n_pad = (int)round_up(ly.out, 16);
        ly.poff = poff;
        ly.pcnt = (int64_t)ly.rows * ly.out;
        poff += ly.pcnt;
        ly.blk = m->shadow ? m->slot : (m->hops - 1 - li);
        ly.m_cap = m->shadow ? (li == m->L - 1 ? c.batch_size : m->nodes_cap) : m->hb[ly.blk].cap_dst;
        {   // wgrad split over the reduction so that tiles x splits fills the 148 SMs once
            const int bn = tc_tile_n(ly.n_pad);
            const int64_t tiles = ((ly.k_pad + 127) / 128) * ((ly.n_pad + bn - 1) / bn);
            ly.splits = (int)std::max<int64_t>(1, std::min<int64_t>(148 / tiles, ly.m_cap / 128));
        }
        m->layers.push_back(ly);
    }
    m->pcount = poff;
    if (m->shadow) {
        int maxw = 4;
        for (const Layer& ly : m->layers) maxw = std::max(maxw, ly.in_pad);
        AL(m->bal_part, 2 * (int64_t)bal_units_cap() * maxw);
        AL(m->bal_cnt, m->nodes_cap + 1);
        AL(m->rf_mask, m->nodes_cap + 1);
        // GS_RF_COMPACT=0: the uncompacted receptive-field path (rows outside it skipped in place)
        const char* rc = std::getenv("GS_RF_COMPACT");
        m->rf_compact = m->L >= 2 && !(rc && rc[0] == '0');
        if (m->rf_compact) {
            AL(m->rf_list, m->nodes_cap + 1);
            AL(m->rf_pos, m->nodes_cap + 1);
            AL(m->rf_sub, m->nodes_cap + 1);
            if (m->hb[m->slot].need_t) {
                AL(m->rf_sub_t, m->nodes_cap + 1);
            } else {
                m->rf_sub_t = m->rf_sub;
            }
            if ((s = dalloc((char**)&m->rf_scratch, (int64_t)rf_compact_scratch_bytes((int)m->nodes_cap), m->owned)) != GNN_OK)
                return cleanup(s);
        }
        CK(cudaMemset(m->bal_cnt, 0, sizeof(int32_t) * (m->nodes_cap + 1)));
        CK(cudaMemset(m->rf_mask, 0, sizeof(uint32_t) * (m->nodes_cap + 1)));
    }
    for (int li = 0; li < m->L; ++li) {
        Layer& ly = m->layers[li];
        ly.rows_alloc = round_up(ly.m_cap, 128);
        const bool x3 = m->bf16x3;
        auto split = [&](Split& sp, int64_t count) -> gnn_status {
            gnn_status r = dalloc(&sp.hi, count, m->owned);
            if (r == GNN_OK && x3) r = dalloc(&sp.lo, count, m->owned);
            if (r == GNN_OK) { cudaMemset(sp.hi, 0, 2 * count); if (sp.lo) cudaMemset(sp.lo, 0, 2 * count); }
            return r;
        };
        // activation / gradient operand planes are k-block-tiled (Split::rows, kernels.h)
        if ((s = split(ly.A, ly.rows_alloc * round_up(ly.k_pad, 64))) != GNN_OK) return cleanup(s);
        if ((s = split(ly.dPre, ly.rows_alloc * round_up(ly.n_pad, 64))) != GNN_OK) return cleanup(s);
        ly.A.rows = ly.rows_alloc;
        ly.dPre.rows = ly.rows_alloc;
        if ((s = split(ly.Wkn, (int64_t)ly.k_pad * ly.n_pad)) != GNN_OK) return cleanup(s);
        AL(ly.H, ly.m_cap * ly.n_pad);
        if (li < m->L - 1) {   // the ReLU layers' sign masks (read by the backward aggregation)
            ly.mask_ld = (ly.n_pad + 31) / 32;
            AL(ly.hmask, ly.m_cap * ly.mask_ld);
            CK(cudaMemset(ly.hmask, 0, sizeof(uint32_t) * ly.m_cap * ly.mask_ld));
        }
        if (li > 0) AL(ly.dA, ly.m_cap * ly.k_pad);
        AL(ly.wpart, (int64_t)ly.splits * ly.k_pad * ly.n_pad);
        // TMA descriptors (128B swizzle) of this layer's three GEMMs
        auto lo_or_hi = [](const Split& sp) { return sp.lo ? (const void*)sp.lo : (const void*)sp.hi; };
        bool ok = true;
        const int bn_d = tc_tile_n(ly.k_pad);
        ok &= make_tmap_bf16_tiled(&ly.map_fwd.a_hi, ly.A.hi, ly.rows_alloc, ly.k_pad, 128);
        ok &= make_tmap_bf16_tiled(&ly.map_fwd.a_lo, lo_or_hi(ly.A), ly.rows_alloc, ly.k_pad, 128);
        ok &= make_tmap_bf16(&ly.map_fwd.b_hi, ly.Wkn.hi, ly.k_pad, ly.n_pad, 64);     // MN-major B
        ok &= make_tmap_bf16(&ly.map_fwd.b_lo, lo_or_hi(ly.Wkn), ly.k_pad, ly.n_pad, 64);
        ok &= make_tmap_bf16_tiled(&ly.map_dgrad.a_hi, ly.dPre.hi, ly.rows_alloc, ly.n_pad, 128);
        ok &= make_tmap_bf16_tiled(&ly.map_dgrad.a_lo, lo_or_hi(ly.dPre), ly.rows_alloc, ly.n_pad, 128);
        ok &= make_tmap_bf16(&ly.map_dgrad.b_hi, ly.Wkn.hi, ly.k_pad, ly.n_pad, bn_d);
        ok &= make_tmap_bf16(&ly.map_dgrad.b_lo, lo_or_hi(ly.Wkn), ly.k_pad, ly.n_pad, bn_d);
        ok &= make_tmap_bf16_tiled(&ly.map_wgrad.a_hi, ly.A.hi, ly.rows_alloc, ly.k_pad, 64);
        ok &= make_tmap_bf16_tiled(&ly.map_wgrad.a_lo, lo_or_hi(ly.A), ly.rows_alloc, ly.k_pad, 64);
        ok &= make_tmap_bf16_tiled(&ly.map_wgrad.b_hi, ly.dPre.hi, ly.rows_alloc, ly.n_pad, 64);
        ok &= make_tmap_bf16_tiled(&ly.map_wgrad.b_lo, lo_or_hi(ly.dPre), ly.rows_alloc, ly.n_pad, 64);
        ok &= make_tmap_f32(&ly.map_fwd.c, ly.H, ly.m_cap, ly.n_pad, ly.n_pad, 1, 0);
        ok &= make_tmap_f32(&ly.map_wgrad.c, ly.wpart, ly.k_pad, ly.n_pad, ly.n_pad, ly.splits,
                            (int64_t)ly.k_pad * ly.n_pad);
        if (li > 0) ok &= make_tmap_f32(&ly.map_dgrad.c, ly.dA, ly.m_cap, ly.k_pad, ly.k_pad, 1, 0);
        if (li == 0 && m->l1_on_sampler) {   // set 1's planes and the maps that read them
            if ((s = split(ly.A1, ly.rows_alloc * round_up(ly.k_pad, 64))) != GNN_OK) return cleanup(s);
            ly.A1.rows = ly.rows_alloc;
            ly.map_fwd1 = ly.map_fwd;
            ly.map_wgrad1 = ly.map_wgrad;
            ok &= make_tmap_bf16_tiled(&ly.map_fwd1.a_hi, ly.A1.hi, ly.rows_alloc, ly.k_pad, 128);
            ok &= make_tmap_bf16_tiled(&ly.map_fwd1.a_lo, lo_or_hi(ly.A1), ly.rows_alloc, ly.k_pad, 128);
            ok &= make_tmap_bf16_tiled(&ly.map_wgrad1.a_hi, ly.A1.hi, ly.rows_alloc, ly.k_pad, 64);
            ok &= make_tmap_bf16_tiled(&ly.map_wgrad1.a_lo, lo_or_hi(ly.A1), ly.rows_alloc, ly.k_pad, 64);
        }
        if (!ok) return cleanup(fail(GNN_ERR_CUDA, "cuTensorMapEncodeTiled failed for layer " + std::to_string(li)));
        // one dynamic-scheduler counter pair per GEMM launch site (the set-1 copies of layer 1's
        // maps share set 0's: the two sets' steps never run concurrently)
        for (TcGemmMaps* mp : {&ly.map_fwd, &ly.map_dgrad, &ly.map_wgrad}) {
            AL(mp->sched, 2);
            CK(cudaMemset(mp->sched, 0, 2 * sizeof(int)));
        }
        ly.map_fwd1.sched = ly.map_fwd.sched;
        ly.map_wgrad1.sched = ly.map_wgrad.sched;
    }
    AL(m->params, m->pcount);
    AL(m->grads, m->pcount);
    if (c.optimizer == GNN_ADAM) {
        AL(m->opt.m, m->pcount);
        AL(m->opt.v, m->pcount);
        AL(m->opt.t, 1);
        AL(m->opt.done, 1);
        CK(cudaMemset(m->opt.m, 0, sizeof(float) * m->pcount));
        CK(cudaMemset(m->opt.v, 0, sizeof(float) * m->pcount));
        CK(cudaMemset(m->opt.t, 0, sizeof(int32_t)));
        CK(cudaMemset(m->opt.done, 0, sizeof(unsigned)));
        m->opt.beta1 = c.beta1; m->opt.beta2 = c.beta2; m->opt.eps = c.eps;
    }
#undef AL
    { const char* e = std::getenv("GS_TIMELINE"); m->timeline = e && e[0] == '1'; }
    {   // default: on when layer 1 is a bulk-copy gather (SAGE + neighbour sampler, local table,
        // k_agg_l1_bulk / k_agg_l1_stream; dense.cu launch_agg_sage); GS_SAMPLE_AFTER_L1=0/1 overrides
        const char* e = std::getenv("GS_SAMPLE_AFTER_L1");
        const char* b = std::getenv("GS_L1_BULK");
        const bool bulk = m->sage && !m->shadow && !g->nshards && g->stride <= 1024 && c.fanouts[0] <= 31 &&
                          !(b && b[0] == '0');
        m->sample_after_l1 = m->l1_on_sampler ? false : e ? e[0] == '1' : bulk;
    }
    for (auto& B : m->bs) CK(cudaEventCreateWithFlags(&B.l1done, cudaEventDisableTiming));
    CK(cudaStreamCreateWithFlags(&m->own_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&m->sstream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&m->wstream, cudaStreamNonBlocking));
    for (int li = 0; li < m->L; ++li) CK(cudaEventCreateWithFlags(&m->ev_dpre[li], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&m->ev_join, cudaEventDisableTiming));
    m->stream = m->own_stream;
    // ---- Glorot-uniform init (per layer block)
    for (int li = 0; li < m->L; ++li) {
        Layer& ly = m->layers[li];
        const float bound = std::sqrt(6.0f / (float)(ly.in + ly.out));
        launch_init_params(m->params + ly.poff, ly.pcnt, bound, c.init_seed, (uint32_t)li, m->stream);
    }
    launch_sgd_pack(pack_desc(m), m->params, nullptr, 0.f, false, OptState{}, m->stream);
    CK(cudaMemsetAsync(m->grads, 0, sizeof(float) * m->pcount, m->stream));
    CK(cudaStreamSynchronize(m->stream));
    CK(cudaDeviceSynchronize());
    CK(cudaGetLastError());
    *out = m;
    return GNN_OK;
}

gnn_status gnn_model_destroy(gnn_model* m) {
    if (!m) return GNN_OK;
    cudaSetDevice(m->g->dev);
    if (m->stream) cudaStreamSynchronize(m->stream);
    if (m->sstream) cudaStreamSynchronize(m->sstream);
    drain_profile(m);
    for (auto e : m->free_events) cudaEventDestroy(e);
    drop_graphs(m);
    for (auto& B : m->bs) {
        for (auto& p : B.prof_pairs) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
        if (B.sampled) cudaEventDestroy(B.sampled);
        if (B.trained) cudaEventDestroy(B.trained);
        if (B.l1done) cudaEventDestroy(B.l1done);
    }
    if (m->comm) ncclCommDestroy(m->comm);
    for (void* p : m->xopened) cudaIpcCloseMemHandle(p);
    if (m->xregion) cudaFree(m->xregion);
    for (void* p : m->owned) cudaFree(p);
    for (void* p : m->owned_host) cudaFreeHost(p);
    for (void* p : {(void*)m->train_sorted, (void*)m->perm, (void*)m->keys, (void*)m->keys_alt, m->cub_tmp})
        if (p) cudaFree(p);
    if (m->own_stream) cudaStreamDestroy(m->own_stream);
    if (m->sstream) cudaStreamDestroy(m->sstream);
    if (m->wstream) cudaStreamDestroy(m->wstream);
    for (auto e : m->ev_dpre) if (e) cudaEventDestroy(e);
    if (m->ev_join) cudaEventDestroy(m->ev_join);
    delete m;
    return GNN_OK;
}

gnn_status gnn_set_stream(gnn_model* m, void* stream) {
    if (!m) return fail(GNN_ERR_PARAM, "NULL model");
    TRY(set_device(m->g->dev));
    TRY(sync_all(m));
    m->stream = stream ? (cudaStream_t)stream : m->own_stream;
    return GNN_OK;
}

gnn_status gnn_set_overlap(gnn_model* m, int32_t enable) {
    if (!m) return fail(GNN_ERR_PARAM, "NULL model");
    m->overlap = enable != 0;
    return GNN_OK;
}

gnn_status gnn_set_train_nodes(gnn_model* m, const int32_t* ids_host, int64_t n) {
    if (!m || n < 0 || (n > 0 && !ids_host)) return fail(GNN_ERR_PARAM, "bad arguments");
    if (n >= INT32_MAX) return fail(GNN_ERR_PARAM, "too many train nodes");
    std::vector<int32_t> ids(ids_host, ids_host + n);
    std::sort(ids.begin(), ids.end());
    for (int64_t i = 0; i < n; ++i) {
        if (ids[i] < 0 || ids[i] >= m->g->N) return fail(GNN_ERR_RANGE, "train id out of range");
        if (i && ids[i] == ids[i - 1]) return fail(GNN_ERR_PARAM, "duplicate train id");
    }
    TRY(set_device(m->g->dev));
    TRY(sync_all(m));
    if (n > m->train_cap) {
        for (void* p : {(void*)m->train_sorted, (void*)m->perm, (void*)m->keys, (void*)m->keys_alt, m->cub_tmp})
            if (p) cudaFree(p);
        CK(cudaMalloc(&m->train_sorted, sizeof(int32_t) * n));
        CK(cudaMalloc(&m->perm, sizeof(int32_t) * n));
        CK(cudaMalloc(&m->keys, sizeof(uint64_t) * n));
        CK(cudaMalloc(&m->keys_alt, sizeof(uint64_t) * n));
        m->cub_bytes = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, m->cub_bytes, m->keys, m->keys_alt, m->train_sorted, m->perm,
                                           (int)n, 0, 64, m->sstream));
        CK(cudaMalloc(&m->cub_tmp, m->cub_bytes));
        m->train_cap = n;
    }
    if (n) CK(cudaMemcpy(m->train_sorted, ids.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
    m->n_train = n;
    m->perm_epoch = -1;
    m->schedule.clear();   // a schedule lists the previous split's batches
    for (auto& B : m->bs) B.valid = false;
    return GNN_OK;
}

int64_t gnn_param_count(const gnn_model* m) { return m ? m->pcount : -1; }
int64_t gnn_num_batches(const gnn_model* m) { return m ? num_batches(m) : -1; }

gnn_status gnn_get_params(gnn_model* m, float* out_host, int64_t n) {
    if (!m || !out_host) return fail(GNN_ERR_PARAM, "NULL argument");
    if (n != m->pcount) return fail(GNN_ERR_SHAPE, "n != param_count");
    TRY(set_device(m->g->dev));
    CK(cudaMemcpyAsync(out_host, m->params, sizeof(float) * n, cudaMemcpyDeviceToHost, m->stream));
    CK(cudaStreamSynchronize(m->stream));
    return GNN_OK;
}

gnn_status gnn_set_params(gnn_model* m, const float* in_host, int64_t n) {
    if (!m || !in_host) return fail(GNN_ERR_PARAM, "NULL argument");
    if (n != m->pcount) return fail(GNN_ERR_SHAPE, "n != param_count");
    TRY(set_device(m->g->dev));
    CK(cudaMemcpyAsync(m->params, in_host, sizeof(float) * n, cudaMemcpyHostToDevice, m->stream));
    launch_sgd_pack(pack_desc(m), m->params, nullptr, 0.f, false, OptState{}, m->stream);
    CK(cudaStreamSynchronize(m->stream));
    return GNN_OK;
}

gnn_status gnn_comm_get_unique_id(uint8_t out_host[128]) {
    if (!out_host) return fail(GNN_ERR_PARAM, "NULL argument");
    ncclUniqueId id;
    CKN(ncclGetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(out_host, &id, 128);
    return GNN_OK;
}

gnn_status gnn_plan_step(int64_t n_train, int32_t batch_size, int32_t world, int32_t rank, int64_t step,
                         int64_t* g_out, int32_t* n_out, int64_t* offset_out, int32_t* b_total_out) {
    if (n_train < 0 || batch_size < 1 || world < 1 || rank < 0 || rank >= world || step < 0)
        return fail(GNN_ERR_PARAM, "bad arguments");
    if (!g_out || !n_out || !offset_out || !b_total_out) return fail(GNN_ERR_PARAM, "NULL output");
    plan_step(n_train, batch_size, world, rank, step, g_out, n_out, offset_out, b_total_out);
    return GNN_OK;
}

int64_t gnn_steps_per_epoch(int64_t n_train, int32_t batch_size, int32_t world) {
    if (n_train < 0 || batch_size < 1 || world < 1) return -1;
    const int64_t nb = (n_train + batch_size - 1) / batch_size;
    return (nb + world - 1) / world;
}

gnn_status gnn_comm_init(gnn_model* m, int32_t rank, int32_t world, const uint8_t id_host[128]) {
    if (!m || !id_host || world < 1 || rank < 0 || rank >= world) return fail(GNN_ERR_PARAM, "bad arguments");
    TRY(set_device(m->g->dev));
    TRY(sync_all(m));
    if (m->comm) { ncclCommDestroy(m->comm); m->comm = nullptr; }
    if (world > 1) {
        ncclUniqueId id;
        std::memcpy(&id, id_host, 128);
        CKN(ncclCommInitRank(&m->comm, world, id, rank));
        (void)cudaGetLastError();   // NCCL's probing may leave a stale runtime error
    }
    m->rank = rank;
    m->world = world;
    drop_graphs(m);
    for (auto& B : m->bs) B.valid = false;
    return GNN_OK;
}

gnn_status gnn_set_exchange(gnn_model* m, int32_t mode) {
    if (!m) return fail(GNN_ERR_PARAM, "NULL model");
    if (mode != GNN_EXCH_AUTO && mode != GNN_EXCH_NCCL && mode != GNN_EXCH_PEER && mode != GNN_EXCH_HOST)
        return fail(GNN_ERR_PARAM, "unknown exchange mode");
    if (mode == GNN_EXCH_PEER && !m->peer_ready)
        return fail(GNN_ERR_STATE, "GNN_EXCH_PEER needs gnn_exchange_export + gnn_exchange_import first");
    TRY(set_device(m->g->dev));
    TRY(sync_all(m));
    if (mode != m->exchange) {
        m->exchange = mode;
        drop_graphs(m);   // the captured step holds the previous exchange
    }
    return GNN_OK;
}

gnn_status gnn_set_rank(gnn_model* m, int32_t rank, int32_t world) {
    if (!m || world < 1 || rank < 0 || rank >= world) return fail(GNN_ERR_PARAM, "bad arguments");
    if (m->comm && m->world != world) return fail(GNN_ERR_PARAM, "world differs from the NCCL communicator's");
    TRY(set_device(m->g->dev));
    TRY(sync_all(m));
    m->rank = rank;
    m->world = world;
    for (auto& B : m->bs) B.valid = false;   // prefetched batches followed the previous rule
    return GNN_OK;
}

gnn_status gnn_apply_update(gnn_model* m, const float* grads_host, int64_t n) {
    Range nvtx_("gnn_apply_update");
    if (!m) return fail(GNN_ERR_PARAM, "NULL model");
    if (!uses_host(m)) return fail(GNN_ERR_STATE, "gnn_apply_update needs GNN_EXCH_HOST");
    if (grads_host && n != m->pcount) return fail(GNN_ERR_SHAPE, "n != param_count");
    TRY(set_device(m->g->dev));
    if (grads_host)
        CK(cudaMemcpyAsync(m->grads, grads_host, sizeof(float) * m->pcount, cudaMemcpyHostToDevice, m->stream));
    launch_sgd_pack(pack_desc(m), m->params, m->grads, m->cfg.lr, false, m->opt, m->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(m->stream));
    return GNN_OK;
}

gnn_status gnn_exchange_export(gnn_model* m, int32_t rank, int32_t world, uint8_t handle_out_host[64]) {
    if (!m || !handle_out_host || world < 1 || rank < 0 || rank >= world) return fail(GNN_ERR_PARAM, "bad arguments");
    if (m->comm && m->world != world) return fail(GNN_ERR_PARAM, "world differs from the NCCL communicator's");
    TRY(set_device(m->g->dev));
    TRY(sync_all(m));
    if (m->xregion) return fail(GNN_ERR_STATE, "exchange region already exported");
    const size_t inbox = sizeof(float) * 2 * (size_t)world * m->pcount;
    const size_t bytes = inbox + sizeof(unsigned long long) * world;
    CK(cudaMalloc(&m->xregion, bytes));   // its own allocation: exported whole by CUDA IPC
    CK(cudaMemset(m->xregion, 0, bytes));
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, m->xregion));
    std::memcpy(handle_out_host, &h, 64);
    m->rank = rank;
    m->world = world;
    drop_graphs(m);
    for (auto& B : m->bs) B.valid = false;
    return GNN_OK;
}

gnn_status gnn_exchange_import(gnn_model* m, const uint8_t* handles_host) {
    if (!m || !handles_host) return fail(GNN_ERR_PARAM, "NULL argument");
    if (!m->xregion) return fail(GNN_ERR_STATE, "gnn_exchange_export first");
    if (m->peer_ready) return fail(GNN_ERR_STATE, "exchange already imported");
    TRY(set_device(m->g->dev));
    const int W = m->world;
    const size_t inbox = sizeof(float) * 2 * (size_t)W * m->pcount;
    std::vector<float*> ib(W);
    std::vector<unsigned long long*> fl(W);
    for (int q = 0; q < W; ++q) {
        void* p = m->xregion;
        if (q != m->rank) {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, handles_host + 64 * q, 64);
            CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
            m->xopened.push_back(p);
        }
        ib[q] = static_cast<float*>(p);
        fl[q] = reinterpret_cast<unsigned long long*>(static_cast<char*>(p) + inbox);
    }
    float** d_ib = nullptr;
    unsigned long long** d_fl = nullptr;
    unsigned long long* seq = nullptr;
    unsigned* done = nullptr;
    TRY(dalloc(&d_ib, W, m->owned));
    TRY(dalloc(&d_fl, W, m->owned));
    TRY(dalloc(&seq, 1, m->owned));
    TRY(dalloc(&done, 2, m->owned));
    CK(cudaMemcpy(d_ib, ib.data(), sizeof(float*) * W, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_fl, fl.data(), sizeof(void*) * W, cudaMemcpyHostToDevice));
    const unsigned long long one = 1;
    CK(cudaMemcpy(seq, &one, sizeof(one), cudaMemcpyHostToDevice));
    CK(cudaMemset(done, 0, 2 * sizeof(unsigned)));
    PeerX& x = m->px;
    x.inbox = d_ib;
    x.flags = d_fl;
    x.my_inbox = ib[m->rank];
    x.my_flags = fl[m->rank];
    x.seq = seq;
    x.world = W;
    x.rank = m->rank;
    x.pcount = m->pcount;
    x.done = done;
    x.done2 = done + 1;
    m->peer_ready = true;
    return GNN_OK;
}

gnn_status gnn_epoch_permutation(gnn_model* m, int64_t epoch, int32_t* out_host, int64_t n) {
    if (!m || (!out_host && m->n_train)) return fail(GNN_ERR_PARAM, "NULL argument");
    if (n < m->n_train) return fail(GNN_ERR_BUFFER, "need n_train = " + std::to_string(m->n_train));
    TRY(set_device(m->g->dev));
    TRY(ensure_perm(m, epoch));
    if (m->n_train)
        CK(cudaMemcpyAsync(out_host, m->perm, sizeof(int32_t) * m->n_train, cudaMemcpyDeviceToHost, m->sstream));
    CK(cudaStreamSynchronize(m->sstream));
    return GNN_OK;
}

gnn_status gnn_sample(gnn_model* m, int64_t epoch, int64_t g, gnn_batch_sizes* sizes_host) {
    Range nvtx_("gnn_sample");
    if (!m || !sizes_host) return fail(GNN_ERR_PARAM, "NULL argument");
    const int64_t nb = num_batches(m);
    if (g < 0 || g >= nb) return fail(GNN_ERR_RANGE, "batch index out of range");
    TRY(set_device(m->g->dev));
    TRY(ensure_perm(m, epoch));
    const int64_t B = m->cfg.batch_size;
    const int32_t n = (int32_t)std::min<int64_t>(B, m->n_train - g * B);
    const int set = other_set(m);
    const bool prof = m->profiling;
    m->profiling = false;
    gnn_status st_ = issue_sample(m, set, m->perm + g * B, nullptr, n, n, epoch, g, true);
    m->profiling = prof;
    TRY(st_);
    m->bs[set].valid = false;   // a parity sample is not a training batch
    m->fetch_set = set;
    StepState st;
    TRY(copy_state(m, set, &st));
    sizes_host->num_hops = m->hops;
    for (int h = 0; h <= kMaxHops; ++h) {
        sizes_host->n_dst[h] = st.n_dst[h];
        sizes_host->n_src[h] = st.n_src[h];
        sizes_host->n_edges[h] = st.n_edges[h];
    }
    return GNN_OK;
}

gnn_status gnn_sample_fetch(gnn_model* m, int32_t hop, int32_t what, int32_t* out_host, int64_t n) {
    if (!m || !out_host) return fail(GNN_ERR_PARAM, "NULL argument");
    const int maxhop = m->shadow ? m->hops : m->hops - 1;
    if (hop < 0 || hop > maxhop) return fail(GNN_ERR_RANGE, "hop out of range");
    TRY(set_device(m->g->dev));
    const BatchSet& B = m->bs[m->fetch_set];
    StepState st;
    TRY(copy_state(m, m->fetch_set, &st));
    int64_t len = 0;
    const int32_t* src = nullptr;
    switch (what) {
        case GNN_SRC_IDS: len = st.n_src[hop]; src = B.nodes; break;
        case GNN_BLK_ROWPTR: len = st.n_dst[hop] + 1; src = B.rowptr[hop]; break;
        case GNN_BLK_COL: len = st.n_edges[hop]; src = B.col[hop]; break;
        case GNN_BLK_NBR: len = st.n_edges[hop]; src = hop < m->hops ? B.nbr[hop] : B.col[hop]; break;
        default: return fail(GNN_ERR_PARAM, "unknown array");
    }
    if (n < len) return fail(GNN_ERR_BUFFER, "buffer too small: need " + std::to_string(len));
    if (len) CK(cudaMemcpy(out_host, src, sizeof(int32_t) * len, cudaMemcpyDeviceToHost));
    if (what == GNN_BLK_NBR && hop == m->hops && len) {   // induced block: global id of each source
        std::vector<int32_t> ids(st.n_src[hop]);
        if (!ids.empty()) CK(cudaMemcpy(ids.data(), B.nodes, sizeof(int32_t) * ids.size(), cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < len; ++i) out_host[i] = ids[out_host[i]];
    }
    return GNN_OK;
}

gnn_status gnn_train_minibatch(gnn_model* m, int64_t epoch, int64_t step, float* loss_out_host) {
    Range nvtx_("gnn_train_minibatch");
    if (!m) return fail(GNN_ERR_PARAM, "NULL model");
    if (step < 0 || epoch < 0) return fail(GNN_ERR_PARAM, "negative epoch/step");
    TRY(set_device(m->g->dev));
    TRY(check_ready(m));
    TRY(step_from_perm(m, epoch, step));
    if (loss_out_host) {
        CK(cudaMemcpyAsync(loss_out_host, &m->bs[m->last].st->loss, sizeof(float), cudaMemcpyDeviceToHost, m->stream));
        CK(cudaStreamSynchronize(m->stream));
    }
    return GNN_OK;
}

gnn_status gnn_train_batch_host(gnn_model* m, const int32_t* seeds_host, int32_t n_seeds, int32_t b_total,
                                int64_t epoch, int64_t g, const int32_t* next_seeds_host, int32_t next_n,
                                int32_t next_b_total, int64_t next_g, float* loss_out_host) {
    Range nvtx_("gnn_train_batch_host");
    if (!m || (n_seeds > 0 && !seeds_host) || !loss_out_host) return fail(GNN_ERR_PARAM, "NULL argument");
    if (n_seeds < 0 || n_seeds > m->cfg.batch_size) return fail(GNN_ERR_SHAPE, "n_seeds must be 0..batch_size");
    if (b_total < n_seeds) return fail(GNN_ERR_PARAM, "b_total < n_seeds");
    const bool prefetch = next_g >= 0;
    if (prefetch && (next_n < 0 || next_n > m->cfg.batch_size || next_b_total < next_n || (next_n > 0 && !next_seeds_host)))
        return fail(GNN_ERR_PARAM, "bad next batch");
    TRY(set_device(m->g->dev));
    TRY(check_ready(m));
    int cur = find_set(m, epoch, g, n_seeds, b_total, seeds_host ? seeds_host : m->bs[0].seeds_stage);
    ++(cur < 0 ? m->reuse_misses : m->reuse_hits);
    if (cur < 0) {
        TRY(check_seeds(m, seeds_host, n_seeds));
        cur = other_set(m);
        TRY(issue_sample(m, cur, nullptr, seeds_host, n_seeds, b_total, epoch, g, m->full_train));
    }
    TRY(train_set(m, cur));
    CK(cudaMemcpyAsync(loss_out_host, &m->bs[cur].st->loss, sizeof(float), cudaMemcpyDeviceToHost, m->stream));
    if (prefetch && m->overlap && !m->profiling) {   // after the training launch (see step_from_perm)
        TRY(check_seeds(m, next_seeds_host, next_n));   // host work that overlaps the step on the device
        TRY(issue_sample(m, 1 - cur, nullptr, next_seeds_host, next_n, next_b_total, epoch, next_g, m->full_train));
    }
    CK(cudaStreamSynchronize(m->stream));
    return GNN_OK;
}

gnn_status gnn_train_epoch(gnn_model* m, int64_t epoch, gnn_epoch_stats* out_host) {
    Range nvtx_("gnn_train_epoch");
    if (!m) return fail(GNN_ERR_PARAM, "NULL model");
    TRY(set_device(m->g->dev));
    const int64_t nb = num_batches(m);
    const int64_t steps = steps_per_epoch(m);
    TRY(check_ready(m));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    // per-step losses land in a device array (copied back once, after the timed epoch)
    float* dloss = nullptr;
    CK(cudaMalloc(&dloss, sizeof(float) * std::max<int64_t>(steps, 1)));
    std::vector<float> losses(std::max<int64_t>(steps, 1));
    TRY(sync_all(m));
    CK(cudaEventRecord(e0, m->stream));
    for (int64_t s = 0; s < steps; ++s) TRY(step_from_perm(m, epoch, s, dloss + s));
    CK(cudaEventRecord(e1, m->stream));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double tot = 0;
    CK(cudaMemcpy(losses.data(), dloss, sizeof(float) * steps, cudaMemcpyDeviceToHost));
    cudaFree(dloss);
    for (int64_t s = 0; s < steps; ++s) tot += losses[s];
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (out_host) {
        out_host->seconds = ms * 1e-3;
        out_host->steps = steps;
        int64_t mine = 0;
        for (int64_t s = 0; s < steps; ++s) mine += (s * m->world + m->rank) < nb;   // same count under a schedule
        out_host->minibatches = mine;
        out_host->mean_loss = steps ? tot / (double)steps : 0.0;
    }
    return GNN_OK;
}

gnn_status gnn_synchronize(gnn_model* m) {
    if (!m) return fail(GNN_ERR_PARAM, "NULL model");
    TRY(set_device(m->g->dev));
    TRY(sync_all(m));
    return GNN_OK;
}

gnn_status gnn_debug_get(gnn_model* m, int32_t what, float* out_host, int64_t n) {
    if (!m || !out_host) return fail(GNN_ERR_PARAM, "NULL argument");
    TRY(set_device(m->g->dev));
    StepState st;
    TRY(copy_state(m, shown_set(m), &st));
    if (what == GNN_DBG_LOSS) {
        if (n < 1) return fail(GNN_ERR_BUFFER, "need 1");
        out_host[0] = st.loss;
        return GNN_OK;
    }
    if (what == GNN_DBG_GRADS) {
        if (n < m->pcount) return fail(GNN_ERR_BUFFER, "need param_count");
        CK(cudaMemcpy(out_host, m->grads, sizeof(float) * m->pcount, cudaMemcpyDeviceToHost));
        return GNN_OK;
    }
    if (what == GNN_DBG_LOGITS) {
        const Layer& ly = m->layers[m->L - 1];
        const int64_t need = (int64_t)st.batch_n * ly.out;
        if (n < need) return fail(GNN_ERR_BUFFER, "need batch_n*C = " + std::to_string(need));
        if (need)
            CK(cudaMemcpy2D(out_host, sizeof(float) * ly.out, ly.H, sizeof(float) * ly.n_pad, sizeof(float) * ly.out,
                            st.batch_n, cudaMemcpyDeviceToHost));
        return GNN_OK;
    }
    if (what == GNN_DBG_TIMELINE) {
        // 4 values per step (µs from the first recorded training start): sampling start, sampling
        // end, training start, training end (step k = k-th sampling and k-th training launch
        // recorded; with overlap the k-th sampling belongs to training k+1); resets the record
        const size_t k = std::min(m->tl_sample.size(), m->tl_train.size());
        if (n < (int64_t)(4 * k + 1)) return fail(GNN_ERR_BUFFER, "need 4*steps+1 = " + std::to_string(4 * k + 1));
        out_host[0] = (float)k;
        if (k) {
            cudaEvent_t t0 = m->tl_train[0].first;
            auto rel = [&](cudaEvent_t e) { float ms = 0.f; cudaEventElapsedTime(&ms, t0, e); return ms * 1e3f; };
            for (size_t i = 0; i < k; ++i) {
                out_host[1 + 4 * i] = rel(m->tl_sample[i].first);
                out_host[2 + 4 * i] = rel(m->tl_sample[i].second);
                out_host[3 + 4 * i] = rel(m->tl_train[i].first);
                out_host[4 + 4 * i] = rel(m->tl_train[i].second);
            }
        }
        for (auto& v : {&m->tl_sample, &m->tl_train})
            for (auto& pr : *v) { m->free_events.push_back(pr.first); m->free_events.push_back(pr.second); }
        m->tl_sample.clear();
        m->tl_train.clear();
        return GNN_OK;
    }
    if (what == GNN_DBG_REUSE) {   // steps whose batch was / was not found prefetched (since creation)
        if (n < 2) return fail(GNN_ERR_BUFFER, "need 2");
        out_host[0] = (float)m->reuse_hits;
        out_host[1] = (float)m->reuse_misses;
        return GNN_OK;
    }
    if (what == GNN_DBG_PHASES) {   // sampling-kernel phase durations of the last sampling run (us)
        GridBarrier hb{};
        CK(cudaMemcpy(&hb, m->bar, sizeof(GridBarrier), cudaMemcpyDeviceToHost));
        const int nb = std::min(32, std::max(0, (int)(hb.nts - hb.pad)));   // barriers of the last launch
        if (n < nb + 1) return fail(GNN_ERR_BUFFER, "need " + std::to_string(nb + 1));
        unsigned long long prev = hb.t0;
        for (int i = 0; i < nb; ++i) {
            const unsigned long long t = hb.ts[(hb.nts - nb + i) & 31u];
            out_host[i] = (float)((double)(t - prev) * 1e-3);
            prev = t;
        }
        out_host[nb] = hb.t_end > prev ? (float)((double)(hb.t_end - prev) * 1e-3) : 0.f;   // last phase
        return GNN_OK;
    }
    if (what >= GNN_DBG_ACT && what < GNN_DBG_ACT + m->L) {
        const int li = what - GNN_DBG_ACT;
        const Layer& ly = m->layers[li];
        const int rows = (m->shadow && li == m->L - 1) ? st.batch_n : st.n_dst[ly.blk];
        const int64_t need = (int64_t)rows * ly.out;
        if (n < need) return fail(GNN_ERR_BUFFER, "need rows*out = " + std::to_string(need));
        if (m->rf_compact && li == m->L - 2) {   // compact receptive-field rows -> block rows (others 0)
            std::memset(out_host, 0, sizeof(float) * need);
            std::vector<int32_t> list(std::max(st.n_rf, 1));
            std::vector<float> h((size_t)std::max(st.n_rf, 1) * ly.out);
            if (st.n_rf) {
                CK(cudaMemcpy(list.data(), m->rf_list, sizeof(int32_t) * st.n_rf, cudaMemcpyDeviceToHost));
                CK(cudaMemcpy2D(h.data(), sizeof(float) * ly.out, ly.H, sizeof(float) * ly.n_pad, sizeof(float) * ly.out,
                                st.n_rf, cudaMemcpyDeviceToHost));
            }
            for (int p = 0; p < st.n_rf; ++p)
                std::memcpy(out_host + (int64_t)list[p] * ly.out, h.data() + (size_t)p * ly.out, sizeof(float) * ly.out);
            return GNN_OK;
        }
        if (need)
            CK(cudaMemcpy2D(out_host, sizeof(float) * ly.out, ly.H, sizeof(float) * ly.n_pad, sizeof(float) * ly.out,
                            rows, cudaMemcpyDeviceToHost));
        return GNN_OK;
    }
    return fail(GNN_ERR_PARAM, "unknown debug array");
}

gnn_status gnn_last_sizes(gnn_model* m, gnn_batch_sizes* sizes_host) {
    if (!m || !sizes_host) return fail(GNN_ERR_PARAM, "NULL argument");
    TRY(set_device(m->g->dev));
    StepState st;
    TRY(copy_state(m, shown_set(m), &st));
    sizes_host->num_hops = m->hops;
    for (int h = 0; h <= kMaxHops; ++h) {
        sizes_host->n_dst[h] = st.n_dst[h];
        sizes_host->n_src[h] = st.n_src[h];
        sizes_host->n_edges[h] = st.n_edges[h];
    }
    return GNN_OK;
}

gnn_status gnn_profile_enable(gnn_model* m, int32_t enable) {
    if (!m) return fail(GNN_ERR_PARAM, "NULL model");
    TRY(set_device(m->g->dev));
    TRY(sync_all(m));
    for (auto& B : m->bs) B.valid = false;   // instrumented steps sample and train serially
    m->profiling = enable != 0;
    return GNN_OK;
}

gnn_status gnn_profile_read(gnn_model* m, int32_t kid, double* ms_out_host, int64_t* launches_out_host) {
    if (!m || kid < 0 || kid >= GNN_K_COUNT) return fail(GNN_ERR_PARAM, "bad arguments");
    TRY(set_device(m->g->dev));
    TRY(sync_all(m));
    drain_profile(m);
    if (ms_out_host) *ms_out_host = m->prof_ms[kid];
    if (launches_out_host) *launches_out_host = m->prof_n[kid];
    return GNN_OK;
}

gnn_status gnn_profile_reset(gnn_model* m) {
    if (!m) return fail(GNN_ERR_PARAM, "NULL model");
    TRY(sync_all(m));
    drain_profile(m);
    for (int i = 0; i < GNN_K_COUNT; ++i) { m->prof_ms[i] = 0; m->prof_n[i] = 0; }
    return GNN_OK;
}

int64_t gnn_launches_per_step(const gnn_model* m) { return m ? m->launches_per_step : -1; }
// ---------------------------------------------------------------- NEXT-3: workload-aware batch assignment
gnn_status gnn_estimate_workload(gnn_model* m, int64_t epoch, int64_t* work_out_host, int64_t n) {
    Range nvtx_("gnn_estimate_workload");
    if (!m || !work_out_host) return fail(GNN_ERR_PARAM, "NULL argument");
    const int64_t nb = num_batches(m);
    if (n != nb) return fail(GNN_ERR_SHAPE, "n must equal the number of batches " + std::to_string(nb));
    TRY(set_device(m->g->dev));
    TRY(sync_all(m));
    TRY(ensure_perm(m, epoch));
    const int64_t B = m->cfg.batch_size;
    const bool prof = m->profiling;
    m->profiling = false;
    gnn_status st_ = GNN_OK;
    for (int64_t g = 0; g < nb && st_ == GNN_OK; ++g) {
        const int set = other_set(m);
        const int32_t cnt = (int32_t)std::min<int64_t>(B, m->n_train - g * B);
        st_ = issue_sample(m, set, m->perm + g * B, nullptr, cnt, cnt, epoch, g, true);
        if (st_ != GNN_OK) break;
        m->bs[set].valid = false;
        StepState ss;
        st_ = copy_state(m, set, &ss);
        // aggregations of the computational graph: the edges every layer aggregates over
        int64_t w = 0;
        for (int li = 0; li < m->L; ++li) w += ss.n_edges[m->layers[li].blk];
        work_out_host[g] = w;
    }
    m->profiling = prof;
    return st_;
}

gnn_status gnn_plan_balanced(const int64_t* work_host, int64_t n, int32_t world, int64_t* order_out_host) {
    if (n < 0 || world < 1 || (n > 0 && (!work_host || !order_out_host))) return fail(GNN_ERR_PARAM, "bad arguments");
    std::vector<int64_t> idx(n);
    for (int64_t i = 0; i < n; ++i) idx[i] = i;
    // heaviest first (ties: lower batch index first); consecutive groups of `world` are the steps,
    // so every step's batches have similar work and the lightest batches share the ragged last step
    std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return work_host[a] > work_host[b]; });
    const int64_t steps = (n + world - 1) / world;
    std::vector<int64_t> first(steps);
    for (int64_t s = 0; s < steps; ++s) {
        int64_t mn = INT64_MAX;
        for (int64_t i = s * world; i < std::min<int64_t>(n, (s + 1) * world); ++i) mn = std::min(mn, idx[i]);
        first[s] = mn;
    }
    // steps in the order of their smallest batch index (the epoch permutation's order)
    std::vector<int64_t> sorder(steps);
    for (int64_t s = 0; s < steps; ++s) sorder[s] = s;
    std::sort(sorder.begin(), sorder.end(), [&](int64_t a, int64_t b) { return first[a] < first[b]; });
    int64_t o = 0;
    for (int64_t s : sorder) {
        if (s == steps - 1 && n % world) continue;   // the ragged group stays last
        for (int64_t i = s * world; i < (s + 1) * world; ++i) order_out_host[o++] = idx[i];
    }
    if (n % world)
        for (int64_t i = (steps - 1) * world; i < n; ++i) order_out_host[o++] = idx[i];
    return GNN_OK;
}

gnn_status gnn_set_schedule(gnn_model* m, const int64_t* order_host, int64_t n) {
    if (!m) return fail(GNN_ERR_PARAM, "NULL model");
    if (n == 0) { m->schedule.clear(); return GNN_OK; }
    const int64_t nb = num_batches(m);
    if (!order_host || n != nb) return fail(GNN_ERR_SHAPE, "schedule must list every batch once");
    std::vector<char> seen(nb, 0);
    for (int64_t i = 0; i < n; ++i) {
        if (order_host[i] < 0 || order_host[i] >= nb || seen[order_host[i]]) return fail(GNN_ERR_PARAM, "schedule is not a permutation of the batches");
        seen[order_host[i]] = 1;
    }
    TRY(sync_all(m));
    m->schedule.assign(order_host, order_host + n);
    for (auto& B : m->bs) B.valid = false;   // prefetched batches followed the previous rule
    return GNN_OK;
}

int32_t gnn_graph_symmetric(const gnn_graph* g) { return g ? (g->symmetric ? 1 : 0) : -1; }

}  // extern "C"
