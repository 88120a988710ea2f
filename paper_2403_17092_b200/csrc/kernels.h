// Host-side launchers of the sm_100a kernels (internal to libgnnstep.so).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "common.cuh"

namespace gs {

// ------------------------------------------------------------------ programmatic dependent launch
// Training-stream kernels are launched with programmatic stream serialization: a kernel's CTAs
// may be scheduled while its predecessor drains (they trigger their dependents on entry), and
// every kernel calls pdl_wait() before its first global-memory access, which waits for the
// predecessor grid's completion and memory flush.  Only prologue work that touches no global
// memory (barrier init, TMEM allocation, descriptor prefetch) precedes pdl_wait().
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// A/B switch GS_CARVEOUT = p (0..100): every training kernel asks for the same L1/shared-memory
// split (cudaFuncAttributePreferredSharedMemoryCarveout), so consecutive or concurrent kernels
// never need an SM reconfiguration.  Unset: the driver's per-kernel choice.
void apply_carveout(const void* kernel);

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
    apply_carveout((const void*)kernel);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ------------------------------------------------------------------ sampling side (sample.cu, sample_step.cu)
#ifndef GS_WARP_GRID_PER_SM
#define GS_WARP_GRID_PER_SM 16
#endif
constexpr int kWarpGrid = 148 * GS_WARP_GRID_PER_SM;   // blocks of 256 threads for warp-per-item kernels

// Epoch permutation keys (Philox tag 1): keys[i] = (w0<<32)|w1 of (train[i], 0, epoch).
void launch_perm_keys(const int32_t* train, int64_t n, uint64_t seed, int64_t epoch,
                      uint64_t* keys, cudaStream_t s);

// Device-side validation of a CSR + labels (synchronous): 0 if valid, else the bit set of
// k_validate (1 row_ptr, 2 column range, 4 row order, 8 label range), -1 on a CUDA error.
int validate_graph(const int64_t* row_ptr, const int32_t* col, int64_t n, const int32_t* y, int C);
// Whether every CSR entry (v -> u) has its reverse (u -> v); synchronous (graph creation).
bool check_symmetric(const int64_t* row_ptr, const int32_t* col, int64_t n, bool* symmetric);

struct GridBarrier {
    unsigned count, gen;
    unsigned nts, pad;            // barriers so far; pad = nts at the last launch's start
    unsigned long long t0;        // kernel start (globaltimer, ns)
    unsigned long long t_end;     // last block's end (atomicMax)
    unsigned long long ts[32];    // ring of barrier-release times
};
// Per block (hop h, or the ShaDow induced block at index `slot`): CSR of the block
// (rowptr over dst, nbr = global source ids, col = local source ids) and, when tcount is
// non-null, its transposed CSR (trowptr over local sources, tdst_s = dst indices ascending).
struct HopIO {
    int k;
    int32_t *rowptr, *nbr, *col;
    int32_t *tcount, *trowptr, *tcursor, *tdst, *tdst_s;
    int32_t* erow;    // destination row of each edge (when tcount is set)
    int count_only;   // only the transposed row pointer (out-degrees) is wanted: no fill, no sort
};
struct SampleParams {
    StepState* st;
    const int64_t* row_ptr;
    const int32_t* col;
    int32_t* nodes;      // the batch's node list: src_h = nodes[0:n_src[h]]
    int32_t* map;        // global -> local id, -1 outside the batch
    uint32_t* bits;      // N-bit set of unseen neighbours (all zero between phases)
    int nwords;
    uint64_t seed;
    int hops, shadow, slot;
    int32_t* icount;     // ShaDow: induced edges per node of S
    int32_t* hubs;       // [3 + cap]: count, next, any, then (block << 27 | row) of transposed rows > 256
    unsigned long long* status;   // look-back words [sample_step_sites(hops) x grid]: tag << 32 | chunk sum
    GridBarrier* bar;
    HopIO hop[kMaxHops + 1];
    // per launch: the batch (the kernel also resets the StepState and writes dst_0)
    const int32_t* seed_src;
    int n_seeds, b_total;
    uint32_t epoch, g, tag;   // tag: step sequence number (unique per launch)
    int full;                 // 1: relabel the last hop too (sampling API, ShaDow, GCN)
};
// One persistent launch: every hop's sampling + relabel, the ShaDow induced block, the
// transposed blocks, the map reset.  Grid = co-resident blocks (occupancy x SMs).
void launch_sample_step(const SampleParams& p, cudaStream_t s);
int sample_step_grid();
int sample_step_sites(int hops);

// ------------------------------------------------------------------ training side (dense.cu)
// Layouts: fp32 activations are row-major with row stride = padded
// width (in_pad = roundup(in, 4); GEMM N padded to 16).  GEMM operands are bf16 split planes
// (hi = bf16(x), lo = bf16(x - hi); lo == nullptr in the bf16-GEMM variant), row-major, and
// rows [M, roundup(M, 64)) of every operand plane are written as zeros (the wgrad reduction
// runs over whole 64-row blocks).  A_l has K_pad = 2*in_pad (SAGE: [H_self | mean]) or in_pad
// (GCN: Â H) columns.
// Operand planes of activations/gradients are stored k-block-tiled: element (r, k) of a plane
// with `rows` rows at ((k / 64) * rows + r) * 64 + k % 64, so that every 64-column x R-row TMA
// box the GEMM loads is one contiguous block of HBM.  rows == 0: plain
// row-major (the weight planes, whose row width is their own).
struct Split { __nv_bfloat16* hi; __nv_bfloat16* lo; int64_t rows; };
__host__ __device__ __forceinline__ int64_t tix(const Split& o, int64_t r, int64_t k) {
    return ((k >> 6) * o.rows + r) * 64 + (k & 63);
}

// Rows of an aggregation input: a local buffer (shards == nullptr), or the feature table
// row-sharded over peers (config 4): row r lives in shard r / rps at local row r % rps; the
// shard pointers are CUDA-IPC mappings of the peers' HBM (NVLink peer loads).  NEXT-2: a
// remote row with a local replica (cache->cmap[r] = slot >= 0) is read from cache->rows
// instead (the GPU feature cache of PAPER.md §3.3, re-aimed at NVLink traffic).
// The cache descriptor lives in device memory at a fixed address, so captured CUDA graphs
// see a cache installed after capture.
// stats (nullable, gnn_cache_stats): row reads by source {local shard, peer, cache replica},
// counted once per warp-level row read (lane 0), so tests and the bench can see the cache work.
struct FeatCache { const int32_t* cmap; const float* rows; unsigned long long* stats; };
struct FeatRows {
    const float* base;
    const float* const* shards;
    int64_t rps;
    const FeatCache* cache;   // sharded tables only (allocated with the graph: never null then)
    int own;                  // this process's shard
    int64_t nrows = 0;        // rows of base (0: unknown)
    __device__ __forceinline__ void count(int which) const {
        unsigned long long* st = cache->stats;
        if (st && (threadIdx.x & 31) == 0) atomicAdd(st + which, 1ull);
    }
    __device__ __forceinline__ const float* row(int r, int ld) const {
        if (!shards) return base + (int64_t)r * ld;
        const int s = (int)(r / rps);
        if (s == own) { count(0); return base + (int64_t)(r - s * rps) * ld; }
        const int32_t* cm = cache->cmap;
        if (cm) {
            const int c = __ldg(cm + r);
            if (c >= 0) { count(2); return cache->rows + (int64_t)c * ld; }
        }
        count(1);
        return shards[s] + (int64_t)(r - s * rps) * ld;
    }
};
// NEXT-2: copy rows ids[0:n) of the (sharded) table into cache rows [0, n) (peer loads).
void launch_cache_fill(FeatRows src, const int32_t* ids, int64_t n, int ld, float* out, cudaStream_t s);

// SAGE-mean aggregation into A = [H_self | mean] for rows i < *rows_ptr.  Neighbour row of
// source c is gmap ? gmap[c] : c, self row smap ? smap[i] : i (layer 1 reads X by global id:
// the fused feature gather).
// fixed_k > 0: the block is fixed-stride (row i's sources at col[i*fixed_k], count in
// blk_rowptr[i]; the training-only last hop of the sampling kernel).  k_max: the block's fanout
// (rows have at most k_max sources); layer 1 on a local table then stages rows by bulk copy.
void launch_agg_sage(const int32_t* rows_ptr, FeatRows H, int in_pad, const int32_t* gmap,
                     const int32_t* smap, const int32_t* blk_rowptr, const int32_t* col, Split A, int fixed_k,
                     int k_max, cudaStream_t s);
// GCN aggregation A = Â H (self loop included) for rows i < *rows_ptr of a block with
// *ndst_ptr destinations; d_out from the transposed row pointer.  col must be local ids.
void launch_agg_gcn(const int32_t* rows_ptr, const int32_t* ndst_ptr, FeatRows H, int in_pad, int lda,
                    const int32_t* gmap, const int32_t* smap, const int32_t* blk_rowptr,
                    const int32_t* col, const int32_t* trowptr, Split A, cudaStream_t s);
// Balanced (merge-path) aggregation over a ShaDow block (dense.cu k_agg_bal): the same
// arithmetic as launch_agg_sage/_gcn (fwd) and launch_spmm_bwd (bwd), with rows split over
// warps by a fixed cut of the merged row+edge sequence, partials combined in a fixed order.
struct BalLaunch {
    bool bwd, gcn;
    const int32_t* n_ptr;      // rows traversed (fwd: output rows; bwd: n_src of the block)
    const int32_t* ndst_ptr;   // n_dst of the block
    const int32_t* dlim_ptr;   // bwd: dA rows < dlim carry gradient
    const int32_t* rowptr;     // traversed CSR (fwd: block; bwd: transposed block)
    const int32_t* col;        // fwd: local sources; bwd: destinations
    const int32_t* orow;       // fwd GCN: transposed row pointer (d_out); bwd: block row pointer (d_in)
    const uint32_t* rmask;     // optional receptive-field mask (== *tag_ptr: in)
    const uint32_t* tag_ptr;
    FeatRows H;                // fwd input rows
    const int32_t* gmap;       // fwd: H row of local node (self and neighbours), nullable
    const float* dA;           // bwd
    const uint32_t* hmask;     // bwd: ReLU decisions of the previous layer (bit per element)
    int mask_ld;               // bwd: words per mask row
    int in_pad;
    Split out;
    int out_w;
    float* part;               // [2 * bal_units_cap()][in_pad] floats
    int32_t* cnt;              // [rows cap] zero-initialised
    // receptive-field compaction (nullable): traverse block rows rlist[0..*n_ptr) with rowptr =
    // their own prefix sum, edges at brow[rlist[r]] + offset, compact output rows; BWD dmap[t] =
    // dA row of destination t or -1 (replaces dlim / rmask)
    const int32_t* rlist = nullptr;
    const int32_t* brow = nullptr;
    const int32_t* dmap = nullptr;
};
int bal_units_cap();   // partial slots needed: 2 * bal_units_cap() rows of in_pad floats
void launch_agg_bal(const BalLaunch& b, cudaStream_t s);
// Receptive-field list of the last layer (after launch_rf_mark): flags / degrees indexed by block
// row, exclusive scans (CUB) over `cap` rows, then rf_list[p] = p-th row in the field (ascending),
// rf_pos[r] = p or -1, sub_rowptr[p] = Σ_{q<p} deg(rf_list[q]) with degrees from `deg_rowptr`
// (the traversed CSR of the backward: the block, or its transpose), *n_rf.  scratch: see
// rf_compact_scratch_bytes(cap).
size_t rf_compact_scratch_bytes(int cap);
void launch_rf_compact(const uint32_t* mask, const uint32_t* tag_ptr, int cap, const int32_t* rowptr,
                       const int32_t* deg_rowptr, void* scratch, int32_t* rf_list, int32_t* rf_pos, int32_t* sub_rowptr,
                       int32_t* sub_rowptr_t, int32_t* n_rf, cudaStream_t s);
// mask[r] = *tag_ptr for the seeds r < *nseed_ptr and their in-neighbours in the block.
void launch_rf_mark(const int32_t* nseed_ptr, const int32_t* rowptr, const int32_t* col, const uint32_t* tag_ptr,
                    uint32_t* mask, cudaStream_t s);
// Per layer: flat fp32 W (rows x out, at params/grads offset poff), its GEMM planes
// W [K_pad x N_pad] (bf16 split), and the wgrad split-K partials.
struct PackLayer {
    int64_t poff;
    int rows, out, in, in_pad, k_pad, n_pad;
    Split Wkn;
    const float* part;
    int splits;
    int64_t split_stride;
};
struct PackAll { PackLayer l[kMaxHops]; int n; bool sage; };
// Deterministic one-shot all-reduce over peer memory (GNN_EXCH_PEER): rank r stores its gradient
// into slot r of every rank's inbox [2 (step parity)][world][pcount] (CUDA-IPC mappings, NVLink
// stores), publishes the step's sequence number in every rank's flag array, and every rank sums
// the world slots of its own inbox in rank order inside the update.  world == 0: not used.
struct PeerX {
    float* const* inbox;              // [world] inbox bases of every rank (device array of peer pointers)
    unsigned long long* const* flags; // [world] flag arrays of every rank ([world] u64 each)
    const float* my_inbox;            // this rank's inbox
    const unsigned long long* my_flags;
    unsigned long long* seq;          // this rank's step sequence number (starts at 1)
    int world, rank, signal;
    int64_t pcount;
    unsigned* done;                   // block counters (zero between launches)
    unsigned* done2;
};
// G[poff + r*out + c] = Σ_z part[z][rpad(r)*n_pad + c] for layers [l0, l1), fixed z order, into
// grads (nullable) and, with x.world, into every rank's inbox (x.signal: then publish the step).
void launch_wgrad_reduce(const PackAll& p, int l0, int l1, float* grads, const PeerX& x, cudaStream_t s);
// Optimizer state: m == nullptr -> SGD; else Adam with moments m, v (flat like params), the
// device step count *t (steps applied so far) and a block counter (zero between launches).
struct OptState { float* m; float* v; int32_t* t; unsigned* done; float beta1, beta2, eps; };
// W <- W - lr*G (SGD) or the Adam update (grads may be nullptr: pack only) and the bf16 planes
// of W, all layers.  reduce: G = the fixed-order sum of the wgrad partials, written to grads
// first (one rank).
// x.world > 0 (peer exchange): G = the rank-order sum of this rank's inbox, after waiting for
// every rank's flag (written to grads, then the update).
void launch_sgd_pack(const PackAll& p, float* params, float* grads, float lr, bool reduce, const OptState& o,
                     cudaStream_t s, const PeerX& x = PeerX{});
// The last layer fused on the CUDA cores (C <= 64): Z = A W, softmax CE (st->loss), dZ split
// planes (+ zero tail rows to a multiple of 64), dA = dZ W^T (fp32 [rows x k_pad]).  Rows
// [0, *m_ptr) of at most m_cap; W = the layer's fp32 parameter block [rows x C].
void launch_last_layer(const int32_t* m_ptr, int m_cap, Split A, int k_pad, int in, int in_pad, bool sage,
                       const float* W, int C, int n_pad, float* Z, Split dz, float* dA, StepState* st,
                       const int32_t* labels, const int32_t* nodes, const float* Hp, const int32_t* rowptr,
                       const int32_t* col, cudaStream_t s);
// (Hp non-null, SAGE: the layer's aggregation A = [H_self | mean] is gathered in the same kernel
// from Hp [rows x in_pad] over the CSR block rowptr/col and written to A's planes.)
bool last_layer_fits(int k_pad, int C);
// Softmax CE over rows [0, batch_n): st->loss = Σ ℓ_i / b_total, dZ = (softmax-onehot)/b_total
// written as split planes [rows x ldz] (+ zero tail rows).
void launch_ce(StepState* st, const float* Z, int ldz, int C, const int32_t* labels,
               const int32_t* nodes, Split dZ, cudaStream_t s);
// Backward aggregation over the transposed block (atomic-free, fixed order), u < n_src[h]:
//   SAGE: dPre_prev[u] = ([u<dlim] dA[u,:in_pad] + Σ_{e in T(u), dst<dlim} dA[dst, in_pad:]/deg(dst)) * [H_prev[u]>0]
//   GCN:  dPre_prev[u] = (Â^T dA)[u] * [H_prev[u] > 0]   (dA rows < dlim)
// [H_prev > 0] is read from the previous layer's forward-GEMM sign mask (hmask, mask_ld words/row).
// dPre_prev is written as split planes [n_src x in_pad] (+ zero tail rows).
void launch_spmm_bwd(bool gcn, int h, const StepState* st, const int32_t* dlim, const float* dA,
                     int in_pad, const int32_t* blk_rowptr, const int32_t* trowptr, const int32_t* tdst,
                     const uint32_t* hmask, int mask_ld, Split dPre_prev, cudaStream_t s);
void launch_init_params(float* p, int64_t cnt, float bound, uint64_t seed, uint32_t layer,
                        cudaStream_t s);

// ------------------------------------------------------------------ tensor-core GEMM (gemm_tc.cu)
// sched: the launch's dynamic tile scheduler {next tile, CTAs done} (2 ints, zero between
// launches; one pair per GEMM launch site: GEMMs that may run concurrently must not share it)
struct TcGemmMaps { CUtensorMap a_hi, a_lo, b_hi, b_lo, c; int* sched = nullptr; };
// 2-D bf16 row-major [rows x cols], box {64 cols, box_rows}, 128B swizzle, OOB reads -> 0.
bool make_tmap_bf16(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows);
// fp32 rows [rows x cols] (cols contiguous, no padding between rows), box {cols, 1}, no swizzle:
// the row-gather (tile::gather4) map of a feature table (cols <= 256, cols * 4 a multiple of 16).
bool make_tmap_rows_f32(CUtensorMap* map, const float* base, int64_t rows, int cols);
// k-block-tiled bf16 plane (Split layout, `rows` rows, `cols` columns): 3-D map {64, rows,
// ceil(cols/64)}, box {64, box_rows, 1}, 128B swizzle.
bool make_tmap_bf16_tiled(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows);
// fp32 C of a GEMM: [depth x rows x cols], row stride ld, depth stride dstride (elements); box
// {32, 32, 1}, 128B swizzle; stores outside [rows x cols] are clipped.
bool make_tmap_f32(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld, int64_t depth,
                   int64_t dstride);
// N tile the GEMM uses for an output width n_pad (TMA box rows of a K-major B operand).
int tc_tile_n(int n_pad);
// mode 0 (dgrad): C[M x n_store] = A[M x k_pad] B^T (B given as [n_pad x k_pad]), M = *m_ptr
//   (rows >= M not stored).  A, B K-major; maps: A box rows 128, B box rows tc_tile_n.
// mode 2 (fwd): as mode 0 but B given as [k_pad x n_pad] (MN-major, W as stored), box rows 64;
//   optional ReLU.
// mode 1 (wgrad): C_z[m_static x n_pad] = Σ_{m in split z} A[m, :]^T B[m, :], reduction length
//   *m_ptr split into `splits` ranges of 64-row blocks; A, B MN-major, maps with box rows 64.
// bf16x3: 3-term split product (fp32 parity); else 1 term (bf16 GEMM variant).
// relu_mask (mode 2 with relu, optional): bit j of word [r * mask_ld + c / 32] = [H[r, c] > 0],
// the ReLU decision the backward pass applies (it then reads 1 bit per element instead of H).
cudaError_t launch_gemm_tc(int mode, bool bf16x3, const TcGemmMaps& maps, const int32_t* m_ptr, int m_static,
                           int m_cap, int n_pad, int k_pad, float* C, int ldc, int n_store, bool relu, int splits,
                           int64_t split_stride, cudaStream_t s, uint32_t* relu_mask = nullptr, int mask_ld = 0);

// Last layer, fused: Z = A W (logits, stored like mode 2) and, in the epilogue, the softmax
// cross-entropy of every row < *m_ptr (= batch_n): st->row_loss, dZ split planes [rows x n_pad]
// (+ zero tail rows to a multiple of 64) and st->loss = Σ ℓ / b_total (per-tile sums, then the last CTA adds the tiles in order).
// n_pad <= 64 (one thread holds a row).
cudaError_t launch_gemm_tc_ce(bool bf16x3, const TcGemmMaps& maps, const int32_t* m_ptr, int m_cap, int n_pad,
                              int k_pad, float* Z, StepState* st, int classes, const int32_t* labels,
                              const int32_t* nodes, Split dz, cudaStream_t s);

}  // namespace gs
