/*
 * gnnstep.h — C ABI of the B200-native per-mini-batch GNN training step of
 * "A Unified CPU-GPU Protocol for GNN Training" (arXiv 2403.17092).
 *
 * The library (paper_2403_17092_b200/libgnnstep.so) runs, per mini-batch and per
 * trainer (one process per GPU), the step the paper's trainer processes run
 * (§3: "sampling → data fetching → forward/backward →
 * local gradient", then the synchronous-SGD exchange of §2.2):
 *
 *   neighbour / ShaDow sampling (§2.2)  → dedup + relabel
 *   → input-feature gather (§2.2, "data fetching")
 *   → Â·H aggregation + dense update, GCN Eq. (1) / GraphSAGE Eq. (2) (lines 131-142)
 *   → softmax cross-entropy and the Eq. (3) mini-batch gradient (lines 161-165)
 *   → gradient all-reduce across trainers (NCCL) → SGD update.
 *
 * Conventions (all entry points):
 *   - Every call returns gnn_status; no C++ exception crosses the ABI.  On a non-OK
 *     return gnn_last_error() holds a thread-local message.
 *   - Pointers named *_host are HOST memory; the library copies what it needs
 *     (inputs) or copies into them (outputs).  The caller keeps ownership.
 *   - Handles (gnn_graph*, gnn_model*) are created and destroyed by the caller.
 *   - Work is enqueued on the model's CUDA stream (gnn_set_stream, default: a
 *     stream the library owns).  Calls that return host data synchronize that
 *     stream before returning; the others return after enqueueing.
 *   - A call with world > 1 (after gnn_comm_init) is collective: every rank must
 *     make the same sequence of such calls.
 *   - Device index: the graph's device; the library makes it current on each call.
 */
#ifndef GNNSTEP_H
#define GNNSTEP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GNN_ABI_VERSION 2

typedef enum {
    GNN_OK = 0,
    GNN_ERR_RANGE = -1,   /* an id or label out of range          */
    GNN_ERR_PARAM = -2,   /* an invalid scalar argument                  */
    GNN_ERR_SHAPE = -3,   /* a size/shape contract violation      */
    GNN_ERR_CONFIG = -4,  /* an unsupported model/sampler configuration */
    GNN_ERR_STATE = -5,   /* call out of order (e.g. training before set_train_nodes)     */
    GNN_ERR_BUFFER = -6,  /* caller buffer too small                                        */
    GNN_ERR_OOM = -7,     /* device allocation failed                                       */
    GNN_ERR_CUDA = -8,    /* a CUDA runtime error (message in gnn_last_error)              */
    GNN_ERR_NCCL = -9     /* an NCCL error                                                   */
} gnn_status;

enum { GNN_SAGE_MEAN = 0, GNN_GCN = 1 };          /* Eq. (2) / Eq. (1)                  */
enum { GNN_NEIGHBOR = 0, GNN_SHADOW = 1 };        /* §2.2 Neighbor / ShaDow K-hop       */
enum { GNN_FP32 = 0, GNN_BF16_GEMM = 1 };         /* dense-update GEMM arithmetic        */

typedef struct gnn_graph gnn_graph;
typedef struct gnn_model gnn_model;

/* Thread-local message for the last non-OK status of this thread. */
const char* gnn_last_error(void);
int32_t gnn_abi_version(void);

/* ---------------------------------------------------------------- graph
 * G = (V, E), N = |V|, adjacency as CSR, H^0 = features, y = labels (§2.1
 * lines 119-124; SPEC.md Graph lines 22-28).
 *   row_ptr_host  int64[num_nodes+1], non-decreasing, row_ptr[0] = 0.
 *   col_idx_host  int32[row_ptr[N]]; row v lists the message sources of v (in-
 *                 neighbours), ascending and duplicate-free; every id in [0, N).
 *   features_host fp32[num_nodes * feat_stride], row-major; feat_stride >= feat_dim,
 *                 a multiple of 4; columns >= feat_dim are ignored (treated as 0).
 *   labels_host   int32[num_nodes] in [0, num_classes).
 * Everything is copied to HBM of `device`.  Errors: RANGE for an id/label out of
 * range, SHAPE for a malformed CSR, PARAM for bad sizes, OOM. */
gnn_status gnn_graph_create(int64_t num_nodes, const int64_t* row_ptr_host,
                            const int32_t* col_idx_host, int32_t feat_dim, int32_t feat_stride,
                            const float* features_host, const int32_t* labels_host,
                            int32_t num_classes, int32_t device, gnn_graph** out);
gnn_status gnn_graph_destroy(gnn_graph* g);

/* Row-sharded feature table (BASELINE.json configs[4]: papers100M-scale features split across
 * the GPUs of a box).  Rows are split into nshards uniform blocks of rps = ceil(N/nshards);
 * this process holds block `shard`, i.e. rows [shard*rps, min(N, (shard+1)*rps)), given in
 * shard_features_host (row-major, feat_stride).  CSR and labels are full (replicated).
 * gnn_shard_export writes the CUDA IPC handle (64 bytes) of the local block; after all
 * processes exchanged handles (the caller's collective), gnn_shard_import(handles = nshards
 * x 64 bytes, in shard order) maps every peer block; the layer-1 gather then reads row r
 * from block r / rps with direct peer loads (NVLink on a multi-GPU box).  Training a
 * sharded graph before the import returns STATE. */
gnn_status gnn_graph_create_sharded(int64_t num_nodes, const int64_t* row_ptr_host,
                                    const int32_t* col_idx_host, int32_t feat_dim, int32_t feat_stride,
                                    int32_t nshards, int32_t shard, const float* shard_features_host,
                                    const int32_t* labels_host, int32_t num_classes, int32_t device,
                                    gnn_graph** out);
/* The same graph from DEVICE memory of `device`, borrowed (not copied): for tables too large to
 * stage through host memory (configs[4]: 111M x 128 fp32 features = 57 GB, 1.6B CSR entries).
 * The library references row_ptr_dev, col_idx_dev, features_dev (this process's feature block:
 * all N rows if nshards == 1, else block `shard` as in gnn_graph_create_sharded) and labels_dev;
 * they must stay valid and unchanged until gnn_graph_destroy, which does not free them.
 * Columns >= feat_dim of the feature rows must be 0.  The CSR and labels are validated on the
 * device (SHAPE / RANGE as gnn_graph_create).  With nshards > 1, features_dev must be the start
 * of its own cudaMalloc allocation (it is exported by CUDA IPC): else PARAM.  PARAM if a pointer
 * is not device memory of `device`. */
gnn_status gnn_graph_create_device(int64_t num_nodes, const int64_t* row_ptr_dev, const int32_t* col_idx_dev,
                                   int32_t feat_dim, int32_t feat_stride, int32_t nshards, int32_t shard,
                                   const float* features_dev, const int32_t* labels_dev, int32_t num_classes,
                                   int32_t device, gnn_graph** out);
gnn_status gnn_shard_export(gnn_graph* g, uint8_t handle_out_host[64]);
gnn_status gnn_shard_import(gnn_graph* g, const uint8_t* handles_host);
/* NEXT-2: GPU feature cache (§3.3), re-aimed at the
 * NVLink-sharded table: a local replica of hot REMOTE rows, so their layer-1 gathers read local
 * HBM instead of a peer.  gnn_cache_rows (after gnn_shard_import): replicate rows ids[0:n) (host
 * array, distinct, none owned by this process: PARAM; out of range: RANGE) read from their
 * owners; n = 0 drops the cache.  Results are unchanged (a replica is an exact copy); models and
 * captured CUDA graphs pick the cache up at their next step.  Synchronous; call it while no
 * step of a model on this graph is in flight.  STATE if the graph is not sharded or not imported.
 * gnn_cache_plan_by_degree (host only): the `capacity` remote rows of shard `shard` (of
 * nshards, uniform blocks of ceil(N/nshards) rows) with the highest CSR degree (ties: lower
 * id), ascending in ids_out_host; *n_out_host = their count (a static hot set: a node is
 * sampled about in proportion to its degree). */
gnn_status gnn_cache_rows(gnn_graph* g, const int32_t* ids_host, int64_t n);
/* Row-read counters of a sharded graph's layer-1 gathers (evidence that the cache is read, and
 * the share of remote gathers it removes): counts_out_host[0..2] = row reads served by
 * {this process's shard, a peer's shard (NVLink), the cache replica} since the last reset, one
 * count per warp-level row read (an edge's neighbour row or a destination's self row).
 * Synchronizes the device, then: enable = 1 resets the counters and turns counting on (one
 * atomic per row read), 0 resets and turns it off, -1 only reads.  counts_out_host may be NULL.
 * Captured steps see the switch (the descriptor lives at a fixed address).  STATE if the graph
 * is not sharded. */
gnn_status gnn_cache_stats(gnn_graph* g, int32_t enable, int64_t* counts_out_host);
gnn_status gnn_cache_plan_by_degree(const int64_t* row_ptr_host, int64_t num_nodes, int32_t nshards, int32_t shard,
                                    int64_t capacity, int32_t* ids_out_host, int64_t* n_out_host);

/* ---------------------------------------------------------------- model
 * Layers l = 1..L are numbered input-first; dims = [F, hidden, ..., hidden, C].
 * fanouts are listed input-layer-first (R1): hop h (seeds = hop 0)
 * samples fanouts[L-1-h] neighbours per node.  NEIGHBOR needs num_fanouts ==
 * num_layers; SHADOW samples L' = num_fanouts hops and runs num_layers layers on the
 * induced subgraph (§2.2).  batch_size is per rank.
 * Parameters (flat fp32, layer order): SAGE layer l is the (2*in) x out row-major
 * matrix [W_1; W_2] (self; neighbour) of Eq. (2); GCN layer l is W^(l), in x out.
 * Initialised Glorot-uniform from init_seed. */
typedef struct {
    int32_t model;          /* GNN_SAGE_MEAN | GNN_GCN                        */
    int32_t sampler;        /* GNN_NEIGHBOR | GNN_SHADOW                      */
    int32_t num_layers;     /* L, 1..8                                        */
    int32_t hidden;         /* d                                              */
    int32_t batch_size;     /* b per rank, >= 1                               */
    int32_t num_fanouts;    /* 1..8                                           */
    int32_t fanouts[8];     /* input-layer-first, each 1..32                  */
    int32_t precision;      /* GNN_FP32 | GNN_BF16_GEMM                       */
    int32_t use_graph;      /* 1: replay the step as one CUDA graph           */
    float lr;               /* learning rate                                  */
    uint64_t seed;          /* sampler seed (permutation + sampling draws)    */
    uint64_t init_seed;     /* weight init                                    */
    int32_t optimizer;      /* GNN_SGD (0) | GNN_ADAM (the
                               listings' torch.optim.Adam, lines 398, 444)     */
    float beta1, beta2, eps;/* Adam (torch defaults 0.9, 0.999, 1e-8)         */
} gnn_model_config;
enum { GNN_SGD = 0, GNN_ADAM = 1 };

gnn_status gnn_model_create(gnn_graph* g, const gnn_model_config* cfg, gnn_model** out);
gnn_status gnn_model_destroy(gnn_model* m);
/* stream: a cudaStream_t (as void*) on the graph's device, or NULL for the library's own. */
gnn_status gnn_set_stream(gnn_model* m, void* stream);
/* Overlap (default on): gnn_train_minibatch / gnn_train_epoch sample step s+1 of the
 * epoch on the library's sampling stream while step s trains (two batch buffer sets,
 * ordered by events; §4.1 lines 256-263 overlap sampling with training).  Off:
 * every step samples then trains.  Results are identical either way. */
gnn_status gnn_set_overlap(gnn_model* m, int32_t enable);
/* The train split (copied).  ids in [0, N), duplicate-free (RANGE / PARAM).  n may be 0.
 * Drops any schedule set with gnn_set_schedule (it listed the previous split's batches). */
gnn_status gnn_set_train_nodes(gnn_model* m, const int32_t* ids_host, int64_t n);
int64_t gnn_param_count(const gnn_model* m);
int64_t gnn_num_batches(const gnn_model* m);   /* ceil(n_train / batch_size) */
gnn_status gnn_get_params(gnn_model* m, float* out_host, int64_t n);   /* n == param_count */
gnn_status gnn_set_params(gnn_model* m, const float* in_host, int64_t n);

/* ---------------------------------------------------------------- data parallel
 * Synchronous SGD across `world` trainers (§2.2): global batch
 * g of an epoch goes to rank g mod world at step floor(g / world); the gradient of a
 * step is Σ over ranks of (per-sample gradient sum) / b_total, b_total = seeds in the
 * step over all ranks (R8/R9), all-reduced with NCCL.
 * Rank 0 calls gnn_comm_get_unique_id; the caller broadcasts the 128 bytes (e.g.
 * torch.distributed); every rank then calls gnn_comm_init (collective). */
gnn_status gnn_comm_get_unique_id(uint8_t out_host[128]);
/* Host-only plan of one synchronous-SGD step (the engine's own batch -> rank rule):
 * g = step*world + rank; n = seeds of global batch g (0 if g >= ceil(n_train/B));
 * offset = g*B into the epoch permutation; b_total = seeds of the step over all ranks.
 * steps_per_epoch = ceil(ceil(n_train/B) / world).  PARAM on invalid sizes. */
gnn_status gnn_plan_step(int64_t n_train, int32_t batch_size, int32_t world, int32_t rank, int64_t step,
                         int64_t* g_out, int32_t* n_out, int64_t* offset_out, int32_t* b_total_out);
int64_t gnn_steps_per_epoch(int64_t n_train, int32_t batch_size, int32_t world);

/* ---- NEXT-3: the paper's Dynamic Load Balancer (§4)
 * applied to homogeneous trainers.  Workload of a mini-batch = "the total number of
 * aggregations ... using the computational graph of the mini-batches" (line 285): the edges of
 * every layer's block, Σ_l E(block_l), estimated in advance by running the sampler (line 284).
 * gnn_estimate_workload: work_out_host[g] for every global batch g of `epoch`
 * (n == ceil(n_train/B), else SHAPE); samples every batch (synchronous, a one-time cost).
 * gnn_plan_balanced (host only): sorts the batches by workload (heaviest first, ties by index,
 * line 287), groups consecutive `world` batches into one synchronous step (so the ranks of a
 * step have similar work and sync-SGD stragglers shrink), steps ordered by their smallest batch
 * index, the ragged group last; order_out_host[s*world + r] = batch of rank r at step s.
 * gnn_set_schedule: step s, rank r trains batch order[s*world + r] (a permutation of the
 * epoch's batches, else PARAM/SHAPE); b_total = seeds of that step's batches; n = 0 restores
 * the default rule g = s*world + r.  Every rank must set the same schedule. */
gnn_status gnn_estimate_workload(gnn_model* m, int64_t epoch, int64_t* work_out_host, int64_t n);
gnn_status gnn_plan_balanced(const int64_t* work_host, int64_t n, int32_t world, int64_t* order_out_host);
gnn_status gnn_set_schedule(gnn_model* m, const int64_t* order_host, int64_t n);
gnn_status gnn_comm_init(gnn_model* m, int32_t rank, int32_t world, const uint8_t id_host[128]);
/* How a step exchanges its gradient (§2.2, synchronous SGD):
 *   GNN_EXCH_AUTO (default): world 1 -> the fixed-order reduce of the weight-gradient partials
 *     fused into the update kernel; world > 1 -> as GNN_EXCH_NCCL.
 *   GNN_EXCH_NCCL: per layer, as soon as its weight gradient is ready: reduce kernel ->
 *     ncclAllReduce(sum, fp32) of that layer's bucket, on a side stream overlapping the backward of
 *     the layers below; then the update kernel; all captured in the step's CUDA graph; on world 1
 *     the library builds a one-rank
 *     communicator (the multi-rank branch, verifiable on one GPU: results are bit-identical to
 *     AUTO, since a one-rank all-reduce is a copy and both reduce in the same fixed order).
 * Synchronizes; the next step recaptures.  PARAM for an unknown mode. */
enum { GNN_EXCH_AUTO = 0, GNN_EXCH_NCCL = 1, GNN_EXCH_PEER = 2, GNN_EXCH_HOST = 3 };
gnn_status gnn_set_exchange(gnn_model* m, int32_t mode);
/* GNN_EXCH_HOST (the Unified CPU-GPU protocol, §3: GPU and host-core
 * trainer ranks "generate a local gradient; the local gradients are then gathered" for sync SGD):
 * a step ends with this rank's reduced gradient (read it with gnn_debug_get(GNN_DBG_GRADS)) and
 * does not update; the caller all-reduces it with the other ranks (e.g. torch.distributed gloo,
 * the host ranks of include/gnnhost.h) and calls gnn_apply_update(summed gradient, host, n =
 * param_count; NULL: the device gradient as it stands), which runs the update kernel
 * (SGD/Adam) and synchronizes.  STATE outside GNN_EXCH_HOST, SHAPE for a wrong n.
 * gnn_set_rank: this model's rank/world for the batch -> rank rule without an NCCL
 * communicator (PARAM for bad values or a world differing from an existing communicator's). */
gnn_status gnn_apply_update(gnn_model* m, const float* grads_host, int64_t n);
gnn_status gnn_set_rank(gnn_model* m, int32_t rank, int32_t world);
/* GNN_EXCH_PEER: a deterministic one-shot all-reduce over peer memory, fused with the update and
 * independent of NCCL.  Each rank owns an inbox [2 (step parity)][world][param_count] fp32 and a
 * flag array [world] u64 in one device allocation; gnn_exchange_export(rank, world) allocates it,
 * sets this model's rank/world (the batch -> rank rule of gnn_plan_step) and writes its CUDA IPC
 * handle (64 bytes); after the caller exchanged the handles (e.g. torch.distributed
 * all_gather), gnn_exchange_import(handles = world x 64 bytes, in rank order) maps every peer's
 * region.  Then gnn_set_exchange(GNN_EXCH_PEER): in every step, as soon as layer l's weight
 * gradient is reduced, rank r stores it into slot r of every rank's inbox (NVLink stores), while
 * the backward of the layers below runs; the last bucket publishes the step's sequence number in
 * every rank's flag array; the update kernel waits for all flags, sums the slots in rank order
 * (identical bits on every rank, summation order independent of arrival) and applies SGD/Adam.
 * Every rank must run the same sequence of steps (an absent rank stalls the others).  PARAM for
 * bad arguments or a world different from an NCCL communicator's; STATE out of order. */
gnn_status gnn_exchange_export(gnn_model* m, int32_t rank, int32_t world, uint8_t handle_out_host[64]);
gnn_status gnn_exchange_import(gnn_model* m, const uint8_t* handles_host);

/* The epoch's seed order (§2.2; SPEC.md partition_seeds lines 107-115):
 * train ids sorted by (Philox key64(id, epoch), id) (R7); batch g is
 * perm[g*B, min((g+1)*B, n_train)).  Computed on the device; copied into out_host
 * (int32[n_train]); BUFFER if n < n_train. */
gnn_status gnn_epoch_permutation(gnn_model* m, int64_t epoch, int32_t* out_host, int64_t n);

/* ---------------------------------------------------------------- sampling (parity hook)
 * Sample global batch g of `epoch` (any rank may sample any g), synchronously.
 * sizes: hop h = 0..num_hops-1 (seeds outward): n_dst, n_src, n_edges.  For SHADOW,
 * hop index num_hops holds the induced block (n_dst = n_src = |S|). */
typedef struct {
    int32_t num_hops;
    int64_t n_dst[9], n_src[9], n_edges[9];
} gnn_batch_sizes;
gnn_status gnn_sample(gnn_model* m, int64_t epoch, int64_t g, gnn_batch_sizes* sizes_host);

enum { GNN_SRC_IDS = 0, GNN_BLK_ROWPTR = 1, GNN_BLK_COL = 2, GNN_BLK_NBR = 3 };
/* Copy one array of hop `hop` of the last gnn_sample into out_host (int32).
 * Lengths: SRC_IDS n_src, BLK_ROWPTR n_dst+1, BLK_COL / BLK_NBR n_edges.
 * BUFFER if n is smaller; n larger is fine.  For SHADOW, hop = num_hops is the induced
 * block (BLK_NBR = global id of each source). */
gnn_status gnn_sample_fetch(gnn_model* m, int32_t hop, int32_t what, int32_t* out_host, int64_t n);

/* ---------------------------------------------------------------- training
 * One synchronous-SGD step: this rank trains global batch g = step*world + rank of
 * `epoch` (nothing if g >= num_batches, but it still joins the all-reduce), then the
 * all-reduce and the SGD update.  Device-resident inputs (the epoch permutation is
 * computed on the device when `epoch` changes).  loss_out_host: if non-NULL the call
 * synchronizes and writes this rank's loss Σ_{i in this rank's batch} ℓ_i / b_total
 * (the step's global loss is the sum over ranks); if NULL it returns after
 * enqueueing. */
gnn_status gnn_train_minibatch(gnn_model* m, int64_t epoch, int64_t step, float* loss_out_host);

/* End-to-end call: the seeds of this rank's batch come from HOST memory (copied into the
 * library's pinned staging, then to the device), the step runs (sampling keyed by
 * (epoch, g)), and this rank's loss is copied back; synchronous.  b_total = seeds in the
 * step over all ranks.  Seeds must be node ids in [0, N) (RANGE) without repeats (PARAM);
 * they are checked on the host before they reach the device.  Optional prefetch: with
 * next_g >= 0 the NEXT call's batch (next_seeds_host[0:next_n), next_b_total, global index
 * next_g, same epoch) is checked and sampled on the library's sampling stream while this batch
 * trains; the next call reuses it only if its (epoch, g, n_seeds, b_total) AND its seeds equal
 * the prefetched ones (else it samples its own seeds).  A batch prefetched by
 * gnn_train_minibatch (from the epoch permutation) is never reused here, nor the reverse.
 * next_g < 0: no prefetch (next_* ignored).  The seed arrays are not retained after the call. */
gnn_status gnn_train_batch_host(gnn_model* m, const int32_t* seeds_host, int32_t n_seeds,
                                int32_t b_total, int64_t epoch, int64_t g,
                                const int32_t* next_seeds_host, int32_t next_n, int32_t next_b_total,
                                int64_t next_g, float* loss_out_host);

typedef struct { double seconds; int64_t steps; int64_t minibatches; double mean_loss; } gnn_epoch_stats;
/* All steps of an epoch (collective when world > 1). */
gnn_status gnn_train_epoch(gnn_model* m, int64_t epoch, gnn_epoch_stats* out_host);
gnn_status gnn_synchronize(gnn_model* m);

/* ---------------------------------------------------------------- introspection
 * what: GNN_DBG_LOGITS (b x C of the last step, fp32), GNN_DBG_GRADS (flat, after the
 * all-reduce, before SGD), GNN_DBG_LOSS (1 value: this rank's loss), GNN_DBG_ACT + l
 * (layer l's output H^(l) of the last step, 0-based l, rows x out, fp32; its sign pattern
 * is the ReLU decision the backward pass used).  BUFFER if n is too small. */
enum { GNN_DBG_LOGITS = 0, GNN_DBG_GRADS = 1, GNN_DBG_LOSS = 2, GNN_DBG_PHASES = 8, GNN_DBG_REUSE = 9,
       GNN_DBG_TIMELINE = 10, GNN_DBG_ACT = 16 };
/* GNN_DBG_TIMELINE (diagnostics, when the environment has GS_TIMELINE=1 at model creation): the
 * step timeline since the last read, out[0] = k steps, then per step 4 values in microseconds from
 * the first recorded training start: sampling launch start / end, training start / end (CUDA
 * events on the sampling and training streams).  BUFFER if n < 4k + 1. */
/* GNN_DBG_REUSE: 2 values, the training calls (train_minibatch / train_batch_host / train_epoch
 * steps) whose batch was found already sampled (prefetched while the previous step trained) and
 * those that had to sample it first, since the model was created. */
/* GNN_DBG_PHASES: microseconds of each phase (between grid barriers, the last one until the
 * last block ends) of the last sampling-kernel run; BUFFER if n < phases (<= 32). */
gnn_status gnn_debug_get(gnn_model* m, int32_t what, float* out_host, int64_t n);
/* Sizes of the last trained batch (synchronizes). */
gnn_status gnn_last_sizes(gnn_model* m, gnn_batch_sizes* sizes_host);

/* Per-kernel timing (CUDA events around each launch, eager mode only; for the bench's
 * roofline).  enable=1 turns instrumentation on (and CUDA-graph replay off). */
gnn_status gnn_profile_enable(gnn_model* m, int32_t enable);
/* Accumulated milliseconds and launch count of kernel class `kid` (GNN_K_*). */
enum { GNN_K_SAMPLE = 0, GNN_K_RELABEL = 1, GNN_K_AGG_L1 = 2, GNN_K_AGG = 3, GNN_K_GEMM_FWD = 4,
       GNN_K_GEMM_DGRAD = 5, GNN_K_GEMM_WGRAD = 6, GNN_K_SPMM_BWD = 7, GNN_K_CE = 8,
       GNN_K_SGD = 9, GNN_K_TRANSPOSE = 10, GNN_K_INDUCE = 11, GNN_K_ALLREDUCE = 12,
       GNN_K_SCAN = 13, GNN_K_OTHER = 14, GNN_K_COUNT = 15 };
gnn_status gnn_profile_read(gnn_model* m, int32_t kid, double* ms_out_host, int64_t* launches_out_host);
gnn_status gnn_profile_reset(gnn_model* m);
/* Number of kernels one step launches (for the bench's gpu_launches). */
int64_t gnn_launches_per_step(const gnn_model* m);
/* 1 if every CSR entry v -> u of the graph has its reverse u -> v (checked on the device at
   creation), 0 if not, -1 for NULL.  A symmetric graph induces symmetric ShaDow blocks
   (PAPER.md lines 170-171), which serve as their own transpose in the backward pass. */
int32_t gnn_graph_symmetric(const gnn_graph* g);

#ifdef __cplusplus
}
#endif
#endif /* GNNSTEP_H */
