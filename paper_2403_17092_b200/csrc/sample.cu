// Sampling side of the step, sm_100a: epoch permutation keys, neighbour sampling
// (§2.2), dedup + relabel, transposed blocks, ShaDow induce
// (§2.2, §5.3).  Every extent is read from the device
// StepState so the whole step can replay as one CUDA graph.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <climits>

#include "kernels.h"

namespace gs {

namespace {
constexpr unsigned kFull = 0xffffffffu;
constexpr int kScanThreads = 256;

__device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }

// ------------------------------------------------------------------ device-wide exclusive scan
// Single pass, decoupled look-back.  Tiles of kScanTile items are claimed in order through a
// ticket counter; a tile publishes its aggregate (flag 1), looks back over its predecessors'
// published values, then publishes its inclusive prefix (flag 2).  n is read on the device,
// the grid is sized for the worst case and surplus blocks exit; the last block to finish
// resets the ticket/status words for the next scan.  Deterministic (integer sums).
constexpr int kScanIPT = 8;
constexpr int kScanTile = kScanThreads * kScanIPT;

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}

template <class F, class W>
__global__ void __launch_bounds__(kScanThreads) k_scan_lookback(F f, W w, ScanScratch sc) {
    using BS = cub::BlockScan<int, kScanThreads>;
    __shared__ typename BS::TempStorage tmp;
    __shared__ int s_vals[kScanTile + kScanTile / 32];
    __shared__ int s_tile, s_excl;
    const int n = f.size();
    const int ntiles = (n + kScanTile - 1) / kScanTile;
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(&sc.ctrl[0], 1u);
    __syncthreads();
    const int tile = s_tile;
    if (tile < ntiles) {
        const int base = tile * kScanTile;
        // striped (coalesced) evaluation into shared memory, blocked read-back
#pragma unroll
        for (int i = 0; i < kScanIPT; ++i) {
            const int li = i * kScanThreads + threadIdx.x;
            const int gi = base + li;
            s_vals[li + li / 32] = gi < n ? f(gi) : 0;
        }
        __syncthreads();
        int v[kScanIPT], tsum = 0;
#pragma unroll
        for (int j = 0; j < kScanIPT; ++j) {
            const int li = threadIdx.x * kScanIPT + j;
            v[j] = s_vals[li + li / 32];
            tsum += v[j];
        }
        int texcl, agg;
        BS(tmp).ExclusiveSum(tsum, texcl, agg);
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            int excl = 0;
            if (tile == 0) {
                if (lane == 0) {
                    __threadfence();
                    atomicExch(&sc.status[0], (2ull << 32) | (unsigned)agg);
                }
            } else {
                if (lane == 0) {
                    __threadfence();
                    atomicExch(&sc.status[tile], (1ull << 32) | (unsigned)agg);
                }
                int j = tile - 1;
                while (true) {
                    const int idx = j - lane;
                    unsigned long long st = idx >= 0 ? ld_volatile_u64(&sc.status[idx]) : (2ull << 32);
                    while (__any_sync(0xffffffffu, (st >> 32) == 0)) {
                        if ((st >> 32) == 0) st = ld_volatile_u64(&sc.status[idx]);
                    }
                    const unsigned pmask = __ballot_sync(0xffffffffu, (st >> 32) == 2);
                    const int last = pmask ? __ffs(pmask) - 1 : 31;
                    int val = lane <= last ? (int)(unsigned)(st & 0xffffffffu) : 0;
                    for (int o = 16; o; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
                    excl += val;
                    if (pmask) break;
                    j -= 32;
                }
                if (lane == 0) {
                    __threadfence();
                    atomicExch(&sc.status[tile], (2ull << 32) | (unsigned)(excl + agg));
                }
            }
            if (lane == 0) s_excl = excl;
        }
        __syncthreads();
        int run = s_excl + texcl;
#pragma unroll
        for (int j = 0; j < kScanIPT; ++j) {
            const int gi = base + threadIdx.x * kScanIPT + j;
            if (gi < n) w(gi, run, v[j]);
            run += v[j];
        }
        if (tile == ntiles - 1 && threadIdx.x == kScanThreads - 1) w.finish(run);
    } else if (ntiles == 0 && tile == 0 && threadIdx.x == 0) {
        w.finish(0);
    }
    // the last block out resets the scan state (all look-backs are complete by then)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned done = atomicAdd(&sc.ctrl[1], 1u);
        s_tile = done == gridDim.x - 1 ? 1 : 0;
    }
    __syncthreads();
    if (s_tile) {
        for (int t = threadIdx.x; t < ntiles; t += kScanThreads) sc.status[t] = 0ull;
        if (threadIdx.x == 0) { sc.ctrl[0] = 0u; sc.ctrl[1] = 0u; }
    }
}

template <class F, class W>
void device_scan(F f, W w, int64_t max_items, ScanScratch sc, cudaStream_t s) {
    int grid = (int)std::min<int64_t>((max_items + kScanTile - 1) / kScanTile, sc.max_tiles);
    if (grid < 1) grid = 1;
    k_scan_lookback<F, W><<<grid, kScanThreads, 0, s>>>(f, w, sc);
}

// ------------------------------------------------------------------ functors
struct RowCountF {           // k_h = min(deg(v), k) for dst node i of hop h
    const StepState* st; int h; int k; const int32_t* nodes; const int64_t* row_ptr;
    __device__ int size() const { return st->n_dst[h]; }
    __device__ int operator()(int i) const {
        const int v = nodes[i];
        const int64_t d = row_ptr[v + 1] - row_ptr[v];
        return d < k ? (int)d : k;
    }
};
struct RowPtrW {
    StepState* st; int h; int32_t* rowptr;
    __device__ void operator()(int i, int excl, int) const { rowptr[i] = excl; }
    __device__ void finish(int total) const { rowptr[st->n_dst[h]] = total; st->n_edges[h] = total; }
};

struct PopF {                // set bits of one bitmap word
    const uint32_t* bits; int nwords;
    __device__ int size() const { return nwords; }
    __device__ int operator()(int w) const { return __popc(bits[w]); }
};
struct AssignW {             // new nodes in ascending global id (R6)
    StepState* st; int h; uint32_t* bits; int32_t* nodes; int32_t* map;
    __device__ void operator()(int w, int excl, int cnt) const {
        if (!cnt) return;
        uint32_t word = bits[w];
        const int base = st->n_dst[h] + excl;
        int r = 0;
        while (word) {
            const int b = __ffs(word) - 1;
            const int u = w * 32 + b;
            nodes[base + r] = u;
            map[u] = base + r;
            ++r;
            word &= word - 1;
        }
        bits[w] = 0;
    }
    __device__ void finish(int total) const {
        const int ns = st->n_dst[h] + total;
        st->n_src[h] = ns;
        if (h + 1 <= kMaxHops) st->n_dst[h + 1] = ns;
    }
};

struct TCountF {
    const StepState* st; int h; const int32_t* tcount;
    __device__ int size() const { return st->n_src[h]; }
    __device__ int operator()(int u) const { return tcount[u]; }
};
struct TRowW {
    const StepState* st; int h; int32_t* tcount; int32_t* trowptr; int32_t* tcursor;
    __device__ void operator()(int u, int excl, int) const {
        trowptr[u] = excl; tcursor[u] = excl; tcount[u] = 0;
    }
    __device__ void finish(int total) const { trowptr[st->n_src[h]] = total; }
};

struct ICountF {
    const StepState* st; int hs; const int32_t* icount;
    __device__ int size() const { return st->n_src[hs]; }
    __device__ int operator()(int i) const { return icount[i]; }
};
struct IRowW {             // square induced block: n_dst = n_src = |S|
    StepState* st; int hs; int slot; int32_t* rowptr;
    __device__ void operator()(int i, int excl, int) const { rowptr[i] = excl; }
    __device__ void finish(int total) const {
        const int n = st->n_src[hs];
        rowptr[n] = total;
        st->n_dst[slot] = n; st->n_src[slot] = n; st->n_edges[slot] = total;
    }
};

// ------------------------------------------------------------------ kernels
__global__ void k_perm_keys(const int32_t* train, int64_t n, uint64_t seed, uint32_t epoch,
                            uint64_t* keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = (uint32_t)train[i];
        const uint4 o = philox4x32_10(make_uint4(v, 0u, (1u << 28) | ((epoch & 0xFFFFFu) << 8), 0u),
                                      make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
        keys[i] = ((uint64_t)o.x << 32) | o.y;
    }
}

__global__ void k_begin_step(StepState* st, const int32_t* seed_src, int32_t n, int32_t b_total,
                             uint32_t epoch, uint32_t g, int32_t* nodes, int32_t* map) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int v = seed_src[i];
        nodes[i] = v;
        map[v] = i;
    }
    if (threadIdx.x == 0) {
        for (int h = 0; h <= kMaxHops; ++h) { st->n_dst[h] = 0; st->n_src[h] = 0; st->n_edges[h] = 0; }
        st->n_dst[0] = n;
        st->batch_n = n;
        st->b_total = b_total;
        st->epoch = epoch;
        st->g = g;
        st->loss = 0.f;
    }
}

// Warp per frontier node.  Floyd's algorithm over CSR positions (R4): lane i
// draws t_i = floor(r_i (j_i+1) / 2^32), j_i = d-k+i, all draws independent of the picks;
// a k-step warp-uniform resolve (ballot) replaces a taken t_i by j_i; a shuffle rank-sort
// puts the picks in ascending position.  O(k) per node, independent of the degree.
__global__ void __launch_bounds__(256) k_sample_fill(int h, int k, const StepState* __restrict__ st,
        const int32_t* __restrict__ nodes, const int64_t* __restrict__ row_ptr,
        const int32_t* __restrict__ col, const int32_t* __restrict__ blk_rowptr,
        int32_t* __restrict__ blk_nbr, const int32_t* __restrict__ map, uint32_t* __restrict__ bits,
        uint64_t seed) {
    const int n = st->n_dst[h];
    const uint32_t epoch = st->epoch, g = st->g;
    const int lane = lane_id();
    for (int i = global_warp(); i < n; i += total_warps()) {
        const int v = nodes[i];
        const int64_t start = row_ptr[v];
        const int d = (int)(row_ptr[v + 1] - start);
        const int out = blk_rowptr[i];
        if (d <= k) {
            for (int q = lane; q < d; q += 32) {
                const int u = col[start + q];
                blk_nbr[out + q] = u;
                if (map[u] < 0) atomicOr(&bits[u >> 5], 1u << (u & 31));
            }
            continue;
        }
        const int j = d - k + lane;
        uint32_t t = 0;
        if (lane < k) {
            const uint32_t r = method_draw(seed, 0u, (uint32_t)v, g, epoch, (uint32_t)h, (uint32_t)lane);
            t = (uint32_t)(((uint64_t)r * (uint64_t)(j + 1)) >> 32);
        }
        int pick = -1;
        for (int q = 0; q < k; ++q) {
            const int tq = (int)__shfl_sync(kFull, t, q);
            const unsigned hit = __ballot_sync(kFull, lane < q && pick == tq);
            if (lane == q) pick = hit ? j : tq;
        }
        int rank = 0;
        for (int q = 0; q < k; ++q) rank += (__shfl_sync(kFull, pick, q) < pick) ? 1 : 0;
        if (lane < k) {
            const int u = col[start + pick];
            blk_nbr[out + rank] = u;
            if (map[u] < 0) atomicOr(&bits[u >> 5], 1u << (u & 31));
        }
    }
}

__global__ void k_relabel_edges(int h, const StepState* __restrict__ st,
                                const int32_t* __restrict__ blk_nbr, int32_t* __restrict__ blk_col,
                                const int32_t* __restrict__ map, int32_t* __restrict__ tcount) {
    const int n = st->n_edges[h];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
        const int c = map[blk_nbr[e]];
        blk_col[e] = c;
        if (tcount) atomicAdd(&tcount[c], 1);
    }
}

__global__ void __launch_bounds__(256) k_transpose_fill(int h, const StepState* __restrict__ st,
        const int32_t* __restrict__ blk_rowptr, const int32_t* __restrict__ blk_col,
        int32_t* __restrict__ tcursor, int32_t* __restrict__ tdst) {
    const int n = st->n_dst[h];
    const int lane = lane_id();
    for (int i = global_warp(); i < n; i += total_warps()) {
        for (int e = blk_rowptr[i] + lane; e < blk_rowptr[i + 1]; e += 32) {
            const int pos = atomicAdd(&tcursor[blk_col[e]], 1);
            tdst[pos] = i;
        }
    }
}

// Warp per transposed row: rank-sort its (distinct) dst indices ascending, so the
// backward sum runs in a fixed order.
__global__ void __launch_bounds__(256) k_transpose_sort(int h, const StepState* __restrict__ st,
        const int32_t* __restrict__ trowptr, const int32_t* __restrict__ tdst,
        int32_t* __restrict__ tdst_sorted) {
    const int n = st->n_src[h];
    const int lane = lane_id();
    for (int u = global_warp(); u < n; u += total_warps()) {
        const int beg = trowptr[u];
        const int len = trowptr[u + 1] - beg;
        if (len <= 32) {
            const int x = lane < len ? tdst[beg + lane] : INT_MAX;
            int rank = 0;
            for (int q = 0; q < len; ++q) rank += (__shfl_sync(kFull, x, q) < x) ? 1 : 0;
            if (lane < len) tdst_sorted[beg + rank] = x;
        } else {
            for (int a = lane; a < len; a += 32) {
                const int x = tdst[beg + a];
                int rank = 0;
                for (int b = 0; b < len; ++b) rank += (tdst[beg + b] < x) ? 1 : 0;
                tdst_sorted[beg + rank] = x;
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_induce_count(int hs, const StepState* __restrict__ st,
        const int32_t* __restrict__ nodes, const int64_t* __restrict__ row_ptr,
        const int32_t* __restrict__ col, const int32_t* __restrict__ map, int32_t* __restrict__ icount) {
    const int n = st->n_src[hs];
    const int lane = lane_id();
    for (int i = global_warp(); i < n; i += total_warps()) {
        const int v = nodes[i];
        int c = 0;
        for (int64_t p = row_ptr[v] + lane; p < row_ptr[v + 1]; p += 32) c += map[col[p]] >= 0;
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
        if (lane == 0) icount[i] = c;
    }
}

// Edge (local(u) -> i) for every u in row S[i] (CSR order) that is in S (R20).
__global__ void __launch_bounds__(256) k_induce_fill(int hs, const StepState* __restrict__ st,
        const int32_t* __restrict__ nodes, const int64_t* __restrict__ row_ptr,
        const int32_t* __restrict__ col, const int32_t* __restrict__ map,
        const int32_t* __restrict__ ind_rowptr, int32_t* __restrict__ ind_col, int32_t* __restrict__ tcount) {
    const int n = st->n_src[hs];
    const int lane = lane_id();
    for (int i = global_warp(); i < n; i += total_warps()) {
        const int v = nodes[i];
        int out = ind_rowptr[i];
        const int64_t beg = row_ptr[v], end = row_ptr[v + 1];
        for (int64_t p0 = beg; p0 < end; p0 += 32) {
            const int64_t p = p0 + lane;
            const int m = p < end ? map[col[p]] : -1;
            const unsigned bal = __ballot_sync(kFull, m >= 0);
            if (m >= 0) {
                ind_col[out + __popc(bal & ((1u << lane) - 1u))] = m;
                atomicAdd(&tcount[m], 1);
            }
            out += __popc(bal);
        }
    }
}

__global__ void k_reset_map(int h, const StepState* __restrict__ st, const int32_t* __restrict__ nodes,
                            int32_t* __restrict__ map) {
    const int n = st->n_src[h];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        map[nodes[i]] = -1;
}
}  // namespace

// ------------------------------------------------------------------ launchers
void launch_perm_keys(const int32_t* train, int64_t n, uint64_t seed, int64_t epoch, uint64_t* keys,
                      cudaStream_t s) {
    if (n <= 0) return;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    k_perm_keys<<<blocks, 256, 0, s>>>(train, n, seed, (uint32_t)epoch, keys);
}

void launch_begin_step(StepState* st, const int32_t* seed_src, int32_t n, int32_t b_total,
                       uint32_t epoch, uint32_t g, int32_t* nodes, int32_t* map, cudaStream_t s) {
    k_begin_step<<<1, 1024, 0, s>>>(st, seed_src, n, b_total, epoch, g, nodes, map);
}

void launch_hop_rowptr(int h, int k, StepState* st, const int32_t* nodes, const int64_t* row_ptr,
                       int32_t* blk_rowptr, int64_t max_dst, ScanScratch sc, cudaStream_t s) {
    device_scan(RowCountF{st, h, k, nodes, row_ptr}, RowPtrW{st, h, blk_rowptr}, max_dst, sc, s);
}

void launch_sample_fill(int h, int k, const StepState* st, const int32_t* nodes, const int64_t* row_ptr,
                        const int32_t* col, const int32_t* blk_rowptr, int32_t* blk_nbr,
                        const int32_t* map, uint32_t* bits, uint64_t seed, cudaStream_t s) {
    k_sample_fill<<<kWarpGrid, 256, 0, s>>>(h, k, st, nodes, row_ptr, col, blk_rowptr, blk_nbr, map,
                                            bits, seed);
}

void launch_assign_new(int h, StepState* st, uint32_t* bits, int64_t nwords, int32_t* nodes,
                       int32_t* map, ScanScratch sc, cudaStream_t s) {
    device_scan(PopF{bits, (int)nwords}, AssignW{st, h, bits, nodes, map}, nwords, sc, s);
}

void launch_relabel_edges(int h, const StepState* st, const int32_t* blk_nbr, int32_t* blk_col,
                          const int32_t* map, int32_t* tcount, cudaStream_t s) {
    k_relabel_edges<<<148 * 8, 256, 0, s>>>(h, st, blk_nbr, blk_col, map, tcount);
}

void launch_transpose(int h, StepState* st, const int32_t* blk_rowptr, const int32_t* blk_col,
                      int32_t* tcount, int32_t* trowptr, int32_t* tcursor, int32_t* tdst,
                      int32_t* tdst_sorted, int64_t max_src, ScanScratch sc, cudaStream_t s) {
    device_scan(TCountF{st, h, tcount}, TRowW{st, h, tcount, trowptr, tcursor}, max_src, sc, s);
    k_transpose_fill<<<kWarpGrid, 256, 0, s>>>(h, st, blk_rowptr, blk_col, tcursor, tdst);
    k_transpose_sort<<<kWarpGrid, 256, 0, s>>>(h, st, trowptr, tdst, tdst_sorted);
}

void launch_induce(int hs, int slot, StepState* st, const int32_t* nodes, const int64_t* row_ptr,
                   const int32_t* col, const int32_t* map, int32_t* icount, int32_t* ind_rowptr,
                   int32_t* ind_col, int32_t* tcount, int64_t max_src, ScanScratch sc, cudaStream_t s) {
    k_induce_count<<<kWarpGrid, 256, 0, s>>>(hs, st, nodes, row_ptr, col, map, icount);
    device_scan(ICountF{st, hs, icount}, IRowW{st, hs, slot, ind_rowptr}, max_src, sc, s);
    k_induce_fill<<<kWarpGrid, 256, 0, s>>>(hs, st, nodes, row_ptr, col, map, ind_rowptr, ind_col, tcount);
}

void launch_reset_map(int h, const StepState* st, const int32_t* nodes, int32_t* map, cudaStream_t s) {
    k_reset_map<<<148 * 4, 256, 0, s>>>(h, st, nodes, map);
}

}  // namespace gs
