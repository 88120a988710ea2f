// The sampling half of a training step as ONE persistent kernel (sm_100a): neighbour
// sampling of every hop (§2.2), dedup + relabel, the ShaDow induced
// block (lines 170-171), the transposed blocks of the backward pass, and the map reset.
//
// The phases depend on each other through whole-grid results ("all neighbours marked", "all
// new ids assigned"), so they are separated by a software grid barrier instead of kernel
// boundaries: one launch replaces ~20.  Prefix sums inside a
// phase use decoupled look-back between the blocks' contiguous chunks (no extra barrier).
// One block per SM (all co-resident).  Every extent is read from the device StepState, so
// the launch replays inside the step's CUDA graph.
//
// Data produced inside the kernel is read with plain (coherent) loads after a barrier; the
// graph (row_ptr, col) is read through the read-only path.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <climits>

#include <cstdlib>

#include "kernels.h"

namespace gs {
namespace {

constexpr unsigned kFull = 0xffffffffu;
#ifndef GS_SAMPLE_THREADS
#define GS_SAMPLE_THREADS 512
#endif
// one block per SM (a cheaper grid barrier) of 512 threads: at 64 registers it takes half the
// register file, so the training kernels of the previous batch share the SMs while this batch is
// sampled (measured: 1024 threads, the whole register file, serialised sampling and training;
// products 3768 -> 4078 mini-batches/s with 512, 384 and 256 slower)
constexpr int kThreads = GS_SAMPLE_THREADS;
constexpr int kWarps = kThreads / 32;

using BlockScan = cub::BlockScan<int, kThreads>;
using BlockReduce = cub::BlockReduce<int, kThreads>;

struct Smem {
    union {
        typename BlockScan::TempStorage scan;
        typename BlockReduce::TempStorage reduce;
    } cub;
    int carry;
    int excl;
    int total;
};

// Grid barrier (all blocks are resident): one atomic per block; block 0 adds 2^31 - (nb-1),
// the others 1, so the last arrival flips bit 31 of the counter (low bits return to 0).  The
// gpu-scope fences order the phases' global writes and invalidate this SM's L1.
__device__ __forceinline__ void grid_sync(GridBarrier* b) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned nb = gridDim.x;
        const unsigned inc = blockIdx.x == 0 ? (0x80000000u - (nb - 1u)) : 1u;
        __threadfence();
        const unsigned old = atomicAdd(&b->count, inc);
        if (((old ^ (old + inc)) & 0x80000000u) != 0u) {   // last arrival: phase timestamp (debug)
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            b->ts[b->nts & 31u] = t;
            b->nts = b->nts + 1u;
        } else {
            volatile unsigned* vc = &b->count;
            while (((old ^ *vc) & 0x80000000u) == 0u) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ void chunk_of(int n, int& beg, int& end) {
    const int c = (n + gridDim.x - 1) / gridDim.x;
    beg = min(n, (int)blockIdx.x * c);
    end = min(n, beg + c);
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}

// Exclusive scan of f over [0, n), each block owning a contiguous chunk, in ONE phase:
// the block publishes its chunk sum, looks back over its predecessors' published sums
// (status words tagged with the step's sequence number, so no reset is needed), publishes
// its inclusive prefix, then scans its chunk: put(i, excl, v).  Returns the grid total in
// the last block (-1 elsewhere).  Deterministic (integer sums).
template <class F, class PUT>
__device__ int chunk_scan(Smem& sm, int n, F f, PUT put, unsigned long long* status, uint32_t tag) {
    int beg, end;
    chunk_of(n, beg, end);
    // a chunk that fits one pass of the block keeps its values in registers (f evaluated once)
    const bool one = end - beg <= kThreads;
    int s = 0, v1 = 0;
    if (one) {
        if (beg + (int)threadIdx.x < end) v1 = f(beg + threadIdx.x);
        s = v1;
    } else {
        for (int i = beg + threadIdx.x; i < end; i += kThreads) s += f(i);
    }
    const int agg = BlockReduce(sm.cub.reduce).Sum(s);
    const unsigned long long tg = (unsigned long long)tag << 32;   // tag != 0 (status words start at 0)
    if (threadIdx.x == 0) {   // publish this chunk's sum
        __threadfence();
        atomicExch(&status[blockIdx.x], tg | (unsigned)agg);
    }
    // read every predecessor's published sum in parallel (one thread each; grid <= threads)
    int pre = 0;
    for (int j = threadIdx.x; j < (int)blockIdx.x; j += kThreads) {
        unsigned long long w = ld_volatile_u64(&status[j]);
        while ((w & ~0xFFFFFFFFull) != tg) w = ld_volatile_u64(&status[j]);
        pre += (int)(unsigned)(w & 0xFFFFFFFFull);
    }
    __syncthreads();
    const int excl = BlockReduce(sm.cub.reduce).Sum(pre);
    if (threadIdx.x == 0) { sm.excl = excl; sm.carry = excl; sm.total = excl + agg; }
    __syncthreads();
    if (one) {
        const int i = beg + threadIdx.x;
        int ex, tile;
        BlockScan(sm.cub.scan).ExclusiveSum(v1, ex, tile);
        if (i < end) put(i, sm.excl + ex, v1);   // (the reduce result is valid in thread 0 only)
        __syncthreads();
        return blockIdx.x == gridDim.x - 1 ? sm.total : -1;
    }
    for (int base = beg; base < end; base += kThreads) {
        const int i = base + threadIdx.x;
        const int v = i < end ? f(i) : 0;
        int ex, tile;
        BlockScan(sm.cub.scan).ExclusiveSum(v, ex, tile);
        const int carry = sm.carry;
        if (i < end) put(i, carry + ex, v);
        __syncthreads();
        if (threadIdx.x == 0) sm.carry = carry + tile;
        __syncthreads();
    }
    return blockIdx.x == gridDim.x - 1 ? sm.total : -1;
}

constexpr int kWarpSort = 256;                    // ints per warp slice of shared memory
constexpr int kBlockSort = 8192;                  // ints = 32 KB: hub rows sorted in shared memory (keeps most of L1 as cache)
static_assert(kBlockSort >= kWarps * kWarpSort, "warp slices fit the hub-sort buffer");

// In-place ascending bitonic sort of s[0:n2) (n2 a power of two) by `nthr` cooperating
// threads (thread index t), `sync` separating the stages.
template <class SYNC>
__device__ __forceinline__ void bitonic_sort(int* s, int n2, int t, int nthr, SYNC sync) {
    for (int k = 2; k <= n2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = t; i < n2; i += nthr) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const int a = s[i], b = s[ixj];
                    const bool asc = (i & k) == 0;
                    if ((a > b) == asc) { s[i] = b; s[ixj] = a; }
                }
            }
            sync();
        }
    }
}

// Sort len <= 8 ints from src into dst ascending, by one thread (a sorting network on
// registers, INT_MAX padding).
__device__ __forceinline__ void lane_sort8(const int32_t* src, int32_t* dst, int len) {
    if (len <= 1) {
        if (len == 1) dst[0] = src[0];
        return;
    }
    int x[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) x[a] = a < len ? src[a] : INT_MAX;
    constexpr int kNet[19][2] = {{0, 1}, {2, 3}, {4, 5}, {6, 7}, {0, 2}, {1, 3}, {4, 6}, {5, 7}, {1, 2}, {5, 6},
                                 {0, 4}, {3, 7}, {1, 5}, {2, 6}, {1, 4}, {3, 6}, {2, 4}, {3, 5}, {3, 4}};
#pragma unroll
    for (int c = 0; c < 19; ++c) {
        const int a = x[kNet[c][0]], b = x[kNet[c][1]];
        x[kNet[c][0]] = min(a, b);
        x[kNet[c][1]] = max(a, b);
    }
#pragma unroll
    for (int a = 0; a < 8; ++a)
        if (a < len) dst[a] = x[a];
}

__device__ __forceinline__ int min_deg(const int64_t* row_ptr, int v, int k) {
    const int64_t d = __ldg(row_ptr + v + 1) - __ldg(row_ptr + v);
    return d < k ? (int)d : k;
}

// Floyd k-of-d (R4) for 32/GS frontier nodes per warp, one lane group of GS >= k
// lanes per node: lane i draws t_i = floor(r_i (j_i+1) / 2^32), j_i = d-k+i (all draws are
// independent of the picks, so they run in parallel); a k-step ballot resolve replaces a
// taken t_i by j_i; a shuffle rank-sort writes the picks in ascending CSR position.  Rows with
// d <= k are copied whole.  Several nodes per warp keep more dependent loads in flight.
// fixed: the block is written with a fixed stride of k slots per row (row i at nbr[i*k],
// its count in rowptr[i]) instead of CSR — the last hop of a training-only run, whose only
// reader is the layer-1 aggregation; no count scan is needed.
template <int GS>
__device__ __forceinline__ void sample_nodes(const SampleParams& P, int h, int k, int i, bool valid, uint32_t epoch,
                                             uint32_t g, int lane, bool mark, bool fixed) {
    const HopIO& H = P.hop[h];
    const int32_t* dst = h == 0 ? P.seed_src : P.nodes;   // hop 0: the seeds, read at their source
    const int lg = lane & (GS - 1);
    const int gbase = lane & ~(GS - 1);
    int v = 0, d = 0, out = 0;
    int64_t start = 0;
    if (valid) {
        v = dst[i];
        start = __ldg(P.row_ptr + v);
        d = (int)(__ldg(P.row_ptr + v + 1) - start);
        out = fixed ? i * k : H.rowptr[i];
        if (fixed && (lane & (GS - 1)) == 0) H.rowptr[i] = d < k ? d : k;
    }
    const bool floyd = d > k;
    const int j = d - k + lg;
    uint32_t t = 0;
    if (floyd && lg < k) {
        const uint32_t r = method_draw(P.seed, 0u, (uint32_t)v, g, epoch, (uint32_t)h, (uint32_t)lg);
        t = (uint32_t)(((uint64_t)r * (uint64_t)(j + 1)) >> 32);
    }
    int pick = -1;
    for (int q = 0; q < k; ++q) {                 // k is uniform: every lane runs the resolve
        const int tq = (int)__shfl_sync(kFull, t, q, GS);
        const unsigned hit = (__ballot_sync(kFull, lg < q && pick == tq) >> gbase) & ((GS == 32) ? kFull : ((1u << GS) - 1u));
        if (lg == q) pick = hit ? j : tq;
    }
    int rank = 0;
    for (int q = 0; q < k; ++q) rank += (__shfl_sync(kFull, pick, q, GS) < pick) ? 1 : 0;
    if (floyd) {
        if (lg < k) {
            const int u = __ldg(P.col + start + pick);
            H.nbr[out + rank] = u;
            if (H.erow) H.erow[out + rank] = i;
            if (mark) atomicOr(&P.bits[u >> 5], 1u << (u & 31));
        }
    } else {
        for (int q = lg; q < d; q += GS) {
            const int u = __ldg(P.col + start + q);
            H.nbr[out + q] = u;
            if (H.erow) H.erow[out + q] = i;
            if (mark) atomicOr(&P.bits[u >> 5], 1u << (u & 31));
        }
    }
}

template <int GS>
__device__ __forceinline__ void sample_chunk(const SampleParams& P, int h, int k, int beg, int end, uint32_t epoch,
                                             uint32_t g, int lane, int wib, bool mark, bool fixed) {
    constexpr int kPerWarp = 32 / GS;
    for (int i0 = beg + wib * kPerWarp; i0 < end; i0 += kWarps * kPerWarp) {
        const int i = i0 + lane / GS;
        sample_nodes<GS>(P, h, k, i, i < end, epoch, g, lane, mark, fixed);
    }
}

__device__ __forceinline__ void relabel_edges(const SampleParams& P, const HopIO& H, int ne, int gtid, int nthreads) {
    for (int e = gtid; e < ne; e += nthreads) {
        const int c = P.map[H.nbr[e]];
        H.col[e] = c;
        if (H.tcount) atomicAdd(&H.tcount[c], 1);
    }
}

#ifndef GS_SAMPLE_MINB
#define GS_SAMPLE_MINB 4   // register cap 32 / thread (a 48-byte spill): 16K registers per SM
#endif
__global__ void __launch_bounds__(kThreads, GS_SAMPLE_MINB) k_sample_step(SampleParams P) {
    __shared__ Smem sm;
    StepState* st = P.st;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int gtid = blockIdx.x * kThreads + threadIdx.x, nthreads = gridDim.x * kThreads;
    const uint32_t epoch = P.epoch, g = P.g, tag = P.tag;
    const int G = gridDim.x;
    int site = 0;   // scan site index (own status words per scan in the step)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        P.bar->t0 = t;
        P.bar->t_end = 0ull;
        P.bar->pad = P.bar->nts;   // barrier count at launch (phase readout)
        P.hubs[0] = 0;   // hub rows of the transposed sort: count, next, any (read after barriers)
        P.hubs[1] = 0;
        P.hubs[2] = 0;
        // the step's state (dst_0 = the seeds, in batch order)
        for (int h = 0; h <= kMaxHops; ++h) { st->n_dst[h] = 0; st->n_src[h] = 0; st->n_edges[h] = 0; }
        st->n_dst[0] = P.n_seeds;
        st->batch_n = P.n_seeds;
        st->b_total = P.b_total;
        st->epoch = epoch;
        st->g = g;
        st->loss = 0.f;
        st->seq = tag;
    }
    for (int i = gtid; i < P.n_seeds; i += nthreads) {   // nodes[i] = seed_i, map[seed_i] = i
        const int v = P.seed_src[i];
        P.nodes[i] = v;
        P.map[v] = i;
    }

    for (int h = 0; h < P.hops; ++h) {
        const HopIO& H = P.hop[h];
        const int k = H.k;
        // the last hop's new-node list and relabel are needed only by the sampling API, ShaDow
        // and GCN; SAGE layer 1 reads X by the sampled global ids
        const bool mark = P.full || h < P.hops - 1;
        // ---- phase 1: relabel the previous hop (its new ids are all assigned); blk_rowptr =
        //      exclusive scan of min(deg, k); Floyd-sample this block's nodes, mark unseen nbrs
        if (h > 0) relabel_edges(P, P.hop[h - 1], st->n_edges[h - 1], gtid, nthreads);
        const int nd = h == 0 ? P.n_seeds : st->n_dst[h];
        const int32_t* dst = h == 0 ? P.seed_src : P.nodes;
        {
            const bool fixed = !mark;   // training-only last hop: fixed-stride rows, no scan
            if (!fixed) {
                const int tot = chunk_scan(sm, nd, [&](int i) { return min_deg(P.row_ptr, dst[i], k); },
                                           [&](int i, int ex, int) { H.rowptr[i] = ex; }, P.status + (site++) * G, tag);
                if (tot >= 0 && threadIdx.x == 0) { H.rowptr[nd] = tot; st->n_edges[h] = tot; }
            } else {
                ++site;
            }
            int beg, end;
            chunk_of(nd, beg, end);
            if (k <= 8) sample_chunk<8>(P, h, k, beg, end, epoch, g, lane, wib, mark, fixed);
            else if (k <= 16) sample_chunk<16>(P, h, k, beg, end, epoch, g, lane, wib, mark, fixed);
            else sample_chunk<32>(P, h, k, beg, end, epoch, g, lane, wib, mark, fixed);
        }
        grid_sync(P.bar);
        if (!mark) break;
        // ---- phase 2: new nodes in ascending global id (R6): nodes[n_dst + rank], map.
        //      Every sampled neighbour was marked (no map lookup on the sampling path): a marked
        //      node that already has a local id (map >= 0) is not new.
        const bool filt = true;
        {
            auto fresh = [&](int w) {
                uint32_t word = P.bits[w];
                if (!filt || !word) return word;
                uint32_t keep = 0u;
                for (uint32_t x = word; x; x &= x - 1) {
                    const int b = __ffs(x) - 1;
                    if (P.map[w * 32 + b] < 0) keep |= 1u << b;
                }
                return keep;
            };
            const int tot = chunk_scan(sm, P.nwords, [&](int w) { return __popc(fresh(w)); },
                                       [&](int w, int ex, int cnt) {
                                           uint32_t word = fresh(w);
                                           if (filt && P.bits[w]) P.bits[w] = 0u;
                                           if (!cnt) return;
                                           const int base = nd + ex;
                                           int r = 0;
                                           while (word) {
                                               const int b = __ffs(word) - 1;
                                               const int u = w * 32 + b;
                                               P.nodes[base + r] = u;
                                               P.map[u] = base + r;
                                               ++r;
                                               word &= word - 1;
                                           }
                                           P.bits[w] = 0u;
                                       }, P.status + (site++) * G, tag);
            if (tot >= 0 && threadIdx.x == 0) {
                st->n_src[h] = nd + tot;
                st->n_dst[h + 1] = nd + tot;
            }
        }
        grid_sync(P.bar);
    }

    // ---- relabel the last hop; ShaDow: count the induced edges of every node of S
    const int L1 = P.hops - 1;
    if (P.full) relabel_edges(P, P.hop[L1], st->n_edges[L1], gtid, nthreads);
    const int nS = P.full ? st->n_src[L1] : st->n_dst[L1];   // nodes with a map entry
    if (P.shadow) {
        // A warp per node of S walks its CSR row kIndU x 32 entries at a time (all loads of a
        // round issued before any is used), so hub rows take few dependent round trips.
        constexpr int kIndU = 8;
        for (int i = blockIdx.x * kWarps + wib; i < nS; i += G * kWarps) {   // |{u in row v : u in S}|
            const int v = P.nodes[i];
            int c = 0;
            const int64_t rb = __ldg(P.row_ptr + v), re = __ldg(P.row_ptr + v + 1);
            for (int64_t p0 = rb; p0 < re; p0 += 32 * kIndU) {
                int u[kIndU];
#pragma unroll
                for (int r = 0; r < kIndU; ++r) {
                    const int64_t p = p0 + 32 * r + lane;
                    u[r] = p < re ? __ldg(P.col + p) : -1;
                }
#pragma unroll
                for (int r = 0; r < kIndU; ++r) c += (u[r] >= 0 && P.map[u[r]] >= 0) ? 1 : 0;
            }
            for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
            if (lane == 0) P.icount[i] = c;
        }
        grid_sync(P.bar);
        const HopIO& S = P.hop[P.slot];
        const int tot = chunk_scan(sm, nS, [&](int i) { return P.icount[i]; },
                                   [&](int i, int ex, int) { S.rowptr[i] = ex; }, P.status + (site++) * G, tag);
        if (tot >= 0 && threadIdx.x == 0) {
            S.rowptr[nS] = tot;
            st->n_dst[P.slot] = nS; st->n_src[P.slot] = nS; st->n_edges[P.slot] = tot;
        }
        grid_sync(P.bar);   // every row offset visible: the fill below is interleaved over the grid
        // edges (local(u) -> i) in CSR order of row S[i] (R20)
        for (int i = blockIdx.x * kWarps + wib; i < nS; i += G * kWarps) {
            const int v = P.nodes[i];
            int out = S.rowptr[i];
            const int64_t rb = __ldg(P.row_ptr + v), re = __ldg(P.row_ptr + v + 1);
            for (int64_t p0 = rb; p0 < re; p0 += 32 * kIndU) {
                int m[kIndU];
#pragma unroll
                for (int r = 0; r < kIndU; ++r) {
                    const int64_t p = p0 + 32 * r + lane;
                    m[r] = p < re ? __ldg(P.col + p) : -1;
                }
#pragma unroll
                for (int r = 0; r < kIndU; ++r) m[r] = m[r] >= 0 ? P.map[m[r]] : -1;
#pragma unroll
                for (int r = 0; r < kIndU; ++r) {
                    const unsigned bal = __ballot_sync(kFull, m[r] >= 0);
                    if (m[r] >= 0) {
                        const int o = out + __popc(bal & ((1u << lane) - 1u));
                        S.col[o] = m[r];
                        if (S.tcount) {   // transposed block wanted (not when the graph is symmetric)
                            S.erow[o] = i;
                            atomicAdd(&S.tcount[m[r]], 1);
                        }
                    }
                    out += __popc(bal);
                }
            }
        }
    }
    if (P.full) grid_sync(P.bar);

    // ---- transposed blocks (rows = local src ids), all needed blocks together
    for (int h = 0; h <= P.hops; ++h) {
        const HopIO& H = P.hop[h];
        if (!H.tcount) continue;
        const int ns = st->n_src[h];
        const int tot = chunk_scan(sm, ns, [&](int u) { return H.tcount[u]; },
                                   [&](int u, int ex, int cnt) {
                                       H.trowptr[u] = ex; H.tcursor[u] = ex; H.tcount[u] = 0;
                                       if (cnt > kWarpSort && !H.count_only) P.hubs[2] = 1;   // a hub row exists
                                   },
                                   P.status + (site++) * G, tag);
        if (tot >= 0 && threadIdx.x == 0) H.trowptr[ns] = tot;
    }
    grid_sync(P.bar);
    for (int h = 0; h <= P.hops; ++h) {   // edge-parallel fill (erow = each edge's destination row)
        const HopIO& H = P.hop[h];
        if (!H.tcount || H.count_only) continue;
        const int ne = st->n_edges[h];
        for (int e = gtid; e < ne; e += nthreads) H.tdst[atomicAdd(&H.tcursor[H.col[e]], 1)] = H.erow[e];
    }
    grid_sync(P.bar);
    // sort every transposed row ascending (fixed summation order).
    // Pass A: a warp takes 32 consecutive rows; rows of <= 8 entries (almost all) are sorted by
    // their lane alone (sorting network in registers), rows of <= kWarpSort by the warp; longer
    // rows (hubs) go to a global list.  Pass B (after a barrier): blocks take hub rows from the
    // list one at a time (dynamic, so clustered hubs spread over the grid) and sort them
    // block-wide in shared memory.
    extern __shared__ int dyn[];
    __shared__ int s_item;
    const bool any_hub = P.hubs[2] != 0;
    int* wbuf = dyn + wib * kWarpSort;
    for (int h = 0; h <= P.hops; ++h) {
        const HopIO& H = P.hop[h];
        if (!H.tcount || H.count_only) continue;
        const int ns = st->n_src[h];
        for (int u0 = (blockIdx.x * kWarps + wib) * 32; u0 < ns; u0 += G * kWarps * 32) {
            const int ul = u0 + lane;
            const int lb = ul < ns ? H.trowptr[ul] : 0;
            const int ll = ul < ns ? H.trowptr[ul + 1] - lb : 0;
            if (ll <= 8) lane_sort8(H.tdst + lb, H.tdst_s + lb, ll);
            if (ll > kWarpSort) P.hubs[3 + atomicAdd(&P.hubs[0], 1)] = (h << 27) | ul;
            unsigned longm = __ballot_sync(kFull, ll > 8 && ll <= kWarpSort);
            while (longm) {
                const int j = __ffs(longm) - 1;
                longm &= longm - 1;
                const int b0 = __shfl_sync(kFull, lb, j);
                const int len = __shfl_sync(kFull, ll, j);
                if (len <= 32) {
                    const int x = lane < len ? H.tdst[b0 + lane] : INT_MAX;
                    int rank = 0;
                    for (int q = 0; q < len; ++q) rank += (__shfl_sync(kFull, x, q) < x) ? 1 : 0;
                    if (lane < len) H.tdst_s[b0 + rank] = x;
                } else {
                    int n2 = 64;
                    while (n2 < len) n2 <<= 1;
                    for (int a = lane; a < n2; a += 32) wbuf[a] = a < len ? H.tdst[b0 + a] : INT_MAX;
                    __syncwarp();
                    bitonic_sort(wbuf, n2, lane, 32, [] { __syncwarp(); });
                    for (int a = lane; a < len; a += 32) H.tdst_s[b0 + a] = wbuf[a];
                    __syncwarp();
                }
            }
        }
    }
    // pass B only when the transposed scan saw a row longer than kWarpSort (flag read after the
    // fill's barrier, so every block takes the same branch)
    const int nhubs = any_hub ? (grid_sync(P.bar), P.hubs[0]) : 0;
    for (;;) {
        if (threadIdx.x == 0) s_item = atomicAdd(&P.hubs[1], 1);
        __syncthreads();
        const int q = s_item;
        __syncthreads();
        if (q >= nhubs) break;
        const int item = P.hubs[3 + q];
        const HopIO& H = P.hop[item >> 27];
        const int u = item & ((1 << 27) - 1);
        const int b0 = H.trowptr[u];
        const int len = H.trowptr[u + 1] - b0;
        if (len <= kBlockSort) {
            int n2 = 2 * kWarpSort;
            while (n2 < len) n2 <<= 1;
            for (int a = threadIdx.x; a < n2; a += kThreads) dyn[a] = a < len ? H.tdst[b0 + a] : INT_MAX;
            __syncthreads();
            bitonic_sort(dyn, n2, threadIdx.x, kThreads, [] { __syncthreads(); });
            for (int a = threadIdx.x; a < len; a += kThreads) H.tdst_s[b0 + a] = dyn[a];
            __syncthreads();
        } else {                                       // beyond shared memory: rank counting
            for (int a = threadIdx.x; a < len; a += kThreads) {
                const int x = H.tdst[b0 + a];
                int rank = 0;
                for (int b = 0; b < len; ++b) rank += (H.tdst[b0 + b] < x) ? 1 : 0;
                H.tdst_s[b0 + rank] = x;
            }
        }
    }
    for (int i = gtid; i < nS; i += nthreads) P.map[P.nodes[i]] = -1;
    if (threadIdx.x == 0) {   // end of this block (debug phase readout)
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMax(&P.bar->t_end, t);
    }
}

}  // namespace

constexpr int kSortSmem = kBlockSort * (int)sizeof(int);

int sample_step_grid() {
    static int grid = 0;
    if (!grid) {
        int per_sm = 0, dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(k_sample_step, cudaFuncAttributeMaxDynamicSharedMemorySize, kSortSmem);
        // A/B switch GS_SAMPLE_CARVE: the sampling kernel's preferred L1/shared split (unset: driver)
        if (const char* e = std::getenv("GS_SAMPLE_CARVE"))
            cudaFuncSetAttribute(k_sample_step, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(e));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sample_step, kThreads, kSortSmem);
        grid = std::max(1, std::min(per_sm, 1)) * std::max(sms, 1);
        // A/B switch GS_SAMPLE_GRID: fewer sampling blocks (SMs), so that the training kernels it
        // overlaps keep the other SMs to themselves (the persistent GEMMs cannot share an SM with it)
        if (const char* e = std::getenv("GS_SAMPLE_GRID")) grid = std::max(1, std::min(grid, std::atoi(e)));
    }
    return grid;
}

// scan sites per step: 2 per hop + 1 induce + 1 per transposed block
int sample_step_sites(int hops) { return 2 * hops + 1 + (hops + 1); }

// The phases are separated by a software grid barrier and the scans spin on predecessors' words,
// so every block must be resident at once: the launch is cooperative (the driver guarantees
// co-residency, and refuses a grid larger than occupancy x SMs; sample_step_grid() is exactly one
// block per SM).  GS_SAMPLE_COOP=0 launches it as a plain grid (A/B only).
void launch_sample_step(const SampleParams& p, cudaStream_t s) {
    static const bool coop = [] { const char* e = std::getenv("GS_SAMPLE_COOP"); return !(e && e[0] == '0'); }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sample_step_grid());
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSortSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = coop ? 1 : 0;
    apply_carveout((const void*)k_sample_step);
    cudaLaunchKernelEx(&cfg, k_sample_step, p);
}

}  // namespace gs
