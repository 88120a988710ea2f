// Training side of the step, sm_100a: Â·H aggregation forward/backward (Eq. 1-2,
// lines 131-142), softmax cross-entropy + the Eq. (3) gradient (lines 161-165), weight
// packing for the tensor-core GEMMs (gemm_tc.cu), SGD.  All extents come from the device
// StepState (graph-replayable).  GEMM operands are written as bf16 split planes.
#include <cub/block/block_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cstdlib>
#include <map>
#include <tuple>

#include "kernels.h"
#include "tma.cuh"

// k_agg_sage register cap (experiments only): GS_AGG_MINB = n -> __launch_bounds__(256, n).  The
// default (no minimum-blocks hint) compiles to 48 registers and was measured fastest (A/B:
// minBlocks 1 -> 70 registers, products gather 57 -> 76 us; 4 -> 61.5 us; 6 -> Reddit 100 -> 145 us)
#ifdef GS_AGG_MINB
#define GS_AGG_BOUNDS __launch_bounds__(256, GS_AGG_MINB)
#else
#define GS_AGG_BOUNDS __launch_bounds__(256)
#endif
#ifndef GS_AGGU2
#define GS_AGGU2 4   // the same for rows of 129..256 floats
#endif
#ifndef GS_AGGU1
#define GS_AGGU1 4   // neighbour rows in flight per warp for rows of <= 128 floats (k_agg_sage)
#endif

namespace gs {
namespace {
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
    return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float4 f4fma(float w, float4 v, float4 a) {   // a + w*v
    return make_float4(a.x + w * v.x, a.y + w * v.y, a.z + w * v.z, a.w + w * v.w);
}
__device__ __forceinline__ float4 f4scale(float4 a, float w) {
    return make_float4(a.x * w, a.y * w, a.z * w, a.w * w);
}
__device__ __forceinline__ uint32_t pack2(__nv_bfloat16 a, __nv_bfloat16 b) {
    return (uint32_t)__bfloat16_as_ushort(a) | ((uint32_t)__bfloat16_as_ushort(b) << 16);
}
// x = hi + lo + O(2^-16 |x|):  hi = bf16_rn(x), lo = bf16_rn(x - hi)
__device__ __forceinline__ void store_split4(const Split& o, int64_t idx, float4 v) {
    const __nv_bfloat16 h0 = __float2bfloat16_rn(v.x), h1 = __float2bfloat16_rn(v.y);
    const __nv_bfloat16 h2 = __float2bfloat16_rn(v.z), h3 = __float2bfloat16_rn(v.w);
    *reinterpret_cast<uint2*>(o.hi + idx) = make_uint2(pack2(h0, h1), pack2(h2, h3));
    if (o.lo) {
        const __nv_bfloat16 l0 = __float2bfloat16_rn(v.x - __bfloat162float(h0));
        const __nv_bfloat16 l1 = __float2bfloat16_rn(v.y - __bfloat162float(h1));
        const __nv_bfloat16 l2 = __float2bfloat16_rn(v.z - __bfloat162float(h2));
        const __nv_bfloat16 l3 = __float2bfloat16_rn(v.w - __bfloat162float(h3));
        *reinterpret_cast<uint2*>(o.lo + idx) = make_uint2(pack2(l0, l1), pack2(l2, l3));
    }
}
// store_split4 with an L2 eviction policy on the stores (createpolicy)
__device__ __forceinline__ void st_v2_hint(void* p, uint32_t a, uint32_t b, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;" ::"l"(p), "r"(a), "r"(b), "l"(pol) : "memory");
}
__device__ __forceinline__ void store_split4_pol(const Split& o, int64_t idx, float4 v, uint64_t pol) {
    const __nv_bfloat16 h0 = __float2bfloat16_rn(v.x), h1 = __float2bfloat16_rn(v.y);
    const __nv_bfloat16 h2 = __float2bfloat16_rn(v.z), h3 = __float2bfloat16_rn(v.w);
    st_v2_hint(o.hi + idx, pack2(h0, h1), pack2(h2, h3), pol);
    if (o.lo) {
        const __nv_bfloat16 l0 = __float2bfloat16_rn(v.x - __bfloat162float(h0));
        const __nv_bfloat16 l1 = __float2bfloat16_rn(v.y - __bfloat162float(h1));
        const __nv_bfloat16 l2 = __float2bfloat16_rn(v.z - __bfloat162float(h2));
        const __nv_bfloat16 l3 = __float2bfloat16_rn(v.w - __bfloat162float(h3));
        st_v2_hint(o.lo + idx, pack2(l0, l1), pack2(l2, l3), pol);
    }
}
__device__ __forceinline__ void store_split1(const Split& o, int64_t idx, float v) {
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    o.hi[idx] = h;
    if (o.lo) o.lo[idx] = __float2bfloat16_rn(v - __bfloat162float(h));
}
__device__ __forceinline__ int round64(int n) { return (n + 63) & ~63; }
// L2 prefetch of two rows of `width` floats (b may be null): one 128-byte line per lane.
__device__ __forceinline__ void prefetch_rows_l2(const float* a, const float* b, int width, int lane) {
    const int nl = (width * 4 + 127) >> 7;
    for (int l = lane; l < 2 * nl; l += 32) {
        const float* p = l < nl ? a + l * 32 : (b ? b + (l - nl) * 32 : nullptr);
        if (p) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
    }
}
constexpr float4 kZero4 = {0.f, 0.f, 0.f, 0.f};
// Row r of an aggregation input.  SH: the row-sharded table (FeatRows::row picks local shard /
// cache replica / peer, with the optional read counters); else plain pointer arithmetic.  The
// kernels are instantiated per case so the local-table gathers carry no shard branches or atomics
// (with them inlined the compiler serialised the in-flight row loads: Reddit gather 96 -> 111 µs).
template <bool SH>
__device__ __forceinline__ const float4* frow(const FeatRows& H, int r, int ld) {
    if constexpr (SH) return reinterpret_cast<const float4*>(H.row(r, ld));
    else return reinterpret_cast<const float4*>(H.base + (int64_t)r * ld);
}

// ------------------------------------------------------------------ forward aggregation
// Warp per destination row; lanes own 16-byte chunks of the feature row (CPL chunks each).
// Neighbour indices are fetched 32 at a time by the warp and broadcast with shuffles; the
// sum runs in CSR row order with plain fp32 adds, then a true division by the degree.
template <int CPL, bool SH>
__global__ void GS_AGG_BOUNDS k_agg_sage(const int32_t* __restrict__ rows_ptr,
        FeatRows H, int in_pad, const int32_t* __restrict__ gmap,
        const int32_t* __restrict__ smap, const int32_t* __restrict__ rowptr,
        const int32_t* __restrict__ col, Split A, int fixed_k) {
    pdl_trigger();
    pdl_wait();
    const int n = *rows_ptr;
    const int nr = round64(n);
    const int lane = lane_id();
    const int nch = in_pad >> 2;
    const int64_t lda = 2 * (int64_t)in_pad;
    for (int i = global_warp(); i < nr; i += total_warps()) {
        if (i >= n) {                                   // zero tail rows of the operand planes
            for (int ch = lane; ch < 2 * nch; ch += 32) store_split4(A, tix(A, i, 4 * ch), kZero4);
            continue;
        }
        // the self row does not depend on the edge chain: issue its loads first
        const float4* ps = frow<SH>(H, smap ? smap[i] : i, in_pad);
        float4 sv[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) sv[c] = (lane + 32 * c) < nch ? __ldg(ps + lane + 32 * c) : kZero4;
        // CSR rows, or fixed-stride rows (row i at col[i*k], count in rowptr[i])
        const int beg = fixed_k ? i * fixed_k : rowptr[i];
        const int end = fixed_k ? beg + rowptr[i] : rowptr[i + 1];
        float4 acc[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) acc[c] = kZero4;
        for (int e0 = beg; e0 < end; e0 += 32) {
            const int m = min(32, end - e0);
            int myidx = 0;
            if (lane < m) { const int c = col[e0 + lane]; myidx = gmap ? gmap[c] : c; }
            int q = 0;
            // kAggU neighbour rows in flight per warp (memory-level parallelism of the gather);
            // the adds stay in CSR order
            constexpr int kAggU = CPL == 1 ? GS_AGGU1 : CPL <= 2 ? GS_AGGU2 : 2;
            for (; q + kAggU <= m; q += kAggU) {
                float4 v[kAggU][CPL];
#pragma unroll
                for (int u = 0; u < kAggU; ++u) {
                    const float4* pu = frow<SH>(H, __shfl_sync(kFull, myidx, q + u), in_pad);
#pragma unroll
                    for (int c = 0; c < CPL; ++c) {
                        const int ch = lane + 32 * c;
                        v[u][c] = ch < nch ? __ldg(pu + ch) : kZero4;
                    }
                }
#pragma unroll
                for (int u = 0; u < kAggU; ++u)
#pragma unroll
                    for (int c = 0; c < CPL; ++c) acc[c] = f4add(acc[c], v[u][c]);
            }
            for (; q + 2 <= m; q += 2) {
                const int r0 = __shfl_sync(kFull, myidx, q), r1 = __shfl_sync(kFull, myidx, q + 1);
                const float4* p0 = frow<SH>(H, r0, in_pad);
                const float4* p1 = frow<SH>(H, r1, in_pad);
                float4 v0[CPL], v1[CPL];
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int ch = lane + 32 * c;
                    v0[c] = ch < nch ? __ldg(p0 + ch) : kZero4;
                    v1[c] = ch < nch ? __ldg(p1 + ch) : kZero4;
                }
#pragma unroll
                for (int c = 0; c < CPL; ++c) { acc[c] = f4add(acc[c], v0[c]); acc[c] = f4add(acc[c], v1[c]); }
            }
            if (q < m) {
                const int r0 = __shfl_sync(kFull, myidx, q);
                const float4* p0 = frow<SH>(H, r0, in_pad);
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int ch = lane + 32 * c;
                    if (ch < nch) acc[c] = f4add(acc[c], __ldg(p0 + ch));
                }
            }
        }
        const int deg = end - beg;
        const float inv = deg ? 1.0f / (float)deg : 0.f;   // one division per row (R23)
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            const int ch = lane + 32 * c;
            if (ch < nch) {
                store_split4(A, tix(A, i, 4 * ch), sv[c]);
                store_split4(A, tix(A, i, 4 * (nch + ch)), f4scale(acc[c], inv));
            }
        }
    }
}

// ------------------------------------------------------------------ layer-1 gather, staged by TMA
// The fused feature gather + mean of layer 1 (S4 + S5: X rows read by global id), with every row
// moved by the bulk-copy engine (cp.async.bulk global -> shared, one instruction per row, no
// registers held while it is in flight) instead of per-lane vector loads.  Each warp owns NB
// row buffers of `slots` = 1 + k_max row slots (self row + the sampled neighbours of one
// destination row) and an mbarrier per buffer.  For its t-th destination row the warp's lanes
// issue the row copies in parallel (lane 0: self row, lane j: neighbour j-1) after lane 0 armed
// the buffer's barrier with the row bytes; while rows t+1 .. t+NB-1 are in flight the warp waits
// for row t's barrier, sums the neighbour rows from shared memory in CSR order (plain fp32 adds,
// then times the correctly rounded 1/deg: the same arithmetic as k_agg_sage), writes [self | mean]
// as split planes, and re-arms the buffer with row t+NB.
// Memory-level parallelism: NB x (1 + k) rows per warp in flight (products: 2 x 16 rows of 400 B
// = 12.8 KB per warp, ~200 KB per SM) against ~4 rows per warp for register loads.
// G4 (the default; GS_L1_G4=0 for one bulk copy per row): the neighbour rows move four at a
// time by the tensor engine's row gather (cp.async.bulk.tensor.2d...tile::gather4 over a
// {in_pad x 1}-box map of X, SASS UTMALDG.2D.GATHER4), so a row of 15 neighbours costs 4 copy
// instructions instead of 15; a buffer is then the self row (padded to 128 B) and groups of 4
// rows (each 128-B aligned).  Products: 49 -> 43 µs per launch, 4210-4255 -> 4410-4630
// mini-batches/s: the copy-issue rate, not the bytes, was part of the per-row latency.
constexpr int kL1Warps = 4;   // warps per block
__device__ __forceinline__ void gather4_g2s(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int r0, int r1,
                                            int r2, int r3, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "l"(pol)
        : "memory");
}
template <int NB, bool G4>
__global__ void __launch_bounds__(kL1Warps * 32) k_agg_l1_bulk(const int32_t* __restrict__ rows_ptr,
        const float* __restrict__ X, int in_pad, const int32_t* __restrict__ smap,
        const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col, Split A, int fixed_k, int slots,
        int xpol, int apol, const __grid_constant__ CUtensorMap xmap) {
    extern __shared__ __align__(128) unsigned char l1_smem[];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    uint64_t* bar = reinterpret_cast<uint64_t*>(l1_smem) + warp * NB;
    const uint32_t row_bytes = (uint32_t)in_pad * 4u;
    // buffer geometry: G4: self row (sb bytes) + groups of 4 rows (gs bytes each); else slots rows
    const uint32_t sb = (row_bytes + 127u) & ~127u, gs = (4u * row_bytes + 127u) & ~127u;
    const uint32_t buf_bytes = G4 ? sb + (uint32_t)((slots - 1 + 3) / 4) * gs : (uint32_t)slots * row_bytes;
    float* ring = reinterpret_cast<float*>(l1_smem + 128 + (size_t)warp * NB * buf_bytes);
    auto nbr_row = [&](const float* buf, int j) -> const float4* {   // neighbour j (0-based) of a buffer
        if constexpr (G4) return reinterpret_cast<const float4*>(reinterpret_cast<const char*>(buf) + sb + (j >> 2) * gs + (j & 3) * row_bytes);
        else return reinterpret_cast<const float4*>(buf + (size_t)(j + 1) * in_pad);
    };
    if (lane == 0) {
#pragma unroll
        for (int b = 0; b < NB; ++b) mbar_init(&bar[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_async_smem();
    }
    __syncwarp();
    pdl_trigger();
    pdl_wait();
    const int n = *rows_ptr;
    const int nch = in_pad >> 2;
    const int64_t W = total_warps();
    const int64_t gw = global_warp();
    // zero tail rows [n, round64(n)) of the operand planes
    for (int64_t i = n + gw; i < round64(n); i += W)
        for (int ch = lane; ch < 2 * nch; ch += 32) store_split4(A, tix(A, i, 4 * ch), kZero4);
    // L2 policies (A/B switches GS_L1_XPOL / GS_L1_APOL): feature rows 0 normal, 1 evict_last,
    // 2 evict_first; operand-plane stores 0 plain, 1 evict_first, 2 evict_last
    const uint64_t pol = xpol == 1 ? policy_evict_last() : xpol == 2 ? policy_evict_first() : policy_evict_normal();
    const uint64_t spol = apol == 2 ? policy_evict_last() : policy_evict_first();
    // A destination row's indices: this lane's row to copy (lane 0: the self row, lane j: the
    // neighbour j-1) and the row's degree.  Fetched one row ahead of their use, so the index loads
    // overlap the wait for the rows in flight instead of stalling the copy issue.
    struct Idx { int nb, self, c; };
    auto fetch = [&](int64_t i) {
        Idx x{0, 0, 0};
        if (i >= n) return x;
        if (fixed_k) {   // fixed-stride rows: the count and the ids load in parallel
            if (lane < fixed_k) x.nb = col[(int)i * fixed_k + lane];
            x.c = rowptr[i];
        } else {
            const int beg = rowptr[i];
            x.c = rowptr[i + 1] - beg;
            if (lane < x.c) x.nb = col[beg + lane];
        }
        x.self = smap ? smap[i] : i;
        return x;
    };
    // arm buffer b with a row: self row -> slot 0, neighbour j -> slot 1 + j (G4: group j / 4)
    auto issue = [&](int b, const Idx& x) {
        float* buf = reinterpret_cast<float*>(reinterpret_cast<char*>(ring) + (size_t)b * buf_bytes);
        if constexpr (G4) {
            const int ng = (x.c + 3) >> 2;
            const int gl = max(lane - 1, 0);   // lane 1 + g issues group g: neighbours 4g .. 4g+3
            const int lim = max(x.c - 1, 0);   // a short last group repeats its last row (not summed)
            const int r0 = __shfl_sync(0xffffffffu, x.nb, min(4 * gl + 0, lim) & 31);
            const int r1 = __shfl_sync(0xffffffffu, x.nb, min(4 * gl + 1, lim) & 31);
            const int r2 = __shfl_sync(0xffffffffu, x.nb, min(4 * gl + 2, lim) & 31);
            const int r3 = __shfl_sync(0xffffffffu, x.nb, min(4 * gl + 3, lim) & 31);
            if (lane == 0) mbar_expect_tx(&bar[b], row_bytes + (uint32_t)ng * 4u * row_bytes);
            __syncwarp();
            if (lane == 0) bulk_g2s(buf, X + (int64_t)x.self * in_pad, row_bytes, &bar[b], pol);
            else if (lane <= ng)
                gather4_g2s(reinterpret_cast<char*>(buf) + sb + gl * gs, &xmap, &bar[b], 0, r0, r1, r2, r3, pol);
        } else {
            if (lane == 0) mbar_expect_tx(&bar[b], (uint32_t)(x.c + 1) * row_bytes);
            __syncwarp();
            const int src = __shfl_up_sync(0xffffffffu, x.nb, 1);   // lane j (>= 1) takes neighbour j-1
            if (lane <= x.c) {
                const int r = lane == 0 ? x.self : src;
                bulk_g2s(buf + (size_t)lane * in_pad, X + (int64_t)r * in_pad, row_bytes, &bar[b], pol);
            }
        }
    };
    int cnt[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int64_t i = gw + b * W;
        const Idx x = fetch(i);
        cnt[b] = x.c;
        if (i < n) issue(b, x);
    }
    Idx pend = fetch(gw + (int64_t)NB * W);   // the row that re-arms the first freed buffer
    uint32_t phase = 0;   // parity bit of every buffer's current use (buffers are used round-robin)
    int b = 0;
    for (int64_t i = gw; i < n; i += W) {
        const Idx nxt = fetch(i + (int64_t)(NB + 1) * W);   // loads in flight during this row
        mbar_wait(&bar[b], phase);
        const float* buf = reinterpret_cast<const float*>(reinterpret_cast<const char*>(ring) + (size_t)b * buf_bytes);
        int c = cnt[0];
#pragma unroll
        for (int q = 1; q < NB; ++q) if (b == q) c = cnt[q];
        float4 sv = kZero4, acc = kZero4;
        if (lane < nch) {
            sv = reinterpret_cast<const float4*>(buf)[lane];
            for (int j = 0; j < c; ++j) acc = f4add(acc, nbr_row(buf, j)[lane]);
        }
        // rows of more than 128 floats: lanes take further chunks
        float4 sv2 = kZero4, acc2 = kZero4;
        const bool wide = nch > 32;
        if (wide && lane + 32 < nch) {
            sv2 = reinterpret_cast<const float4*>(buf)[lane + 32];
            for (int j = 0; j < c; ++j) acc2 = f4add(acc2, nbr_row(buf, j)[lane + 32]);
        }
        // the buffer is read: re-arm it with this warp's row i + NB*W (async-proxy writes after
        // generic-proxy reads of the same shared memory need the proxy fence)
        fence_async_smem();
        __syncwarp();
        const bool more = i + (int64_t)NB * W < n;
        if (more) issue(b, pend);
#pragma unroll
        for (int q = 0; q < NB; ++q) if (b == q) cnt[q] = more ? pend.c : 0;
        pend = nxt;
        const float inv = c ? 1.0f / (float)c : 0.f;   // one division per row (R23)
        if (apol) {
            if (lane < nch) {
                store_split4_pol(A, tix(A, i, 4 * lane), sv, spol);
                store_split4_pol(A, tix(A, i, 4 * (nch + lane)), f4scale(acc, inv), spol);
            }
            if (wide && lane + 32 < nch) {
                store_split4_pol(A, tix(A, i, 4 * (lane + 32)), sv2, spol);
                store_split4_pol(A, tix(A, i, 4 * (nch + lane + 32)), f4scale(acc2, inv), spol);
            }
        } else {
            if (lane < nch) {
                store_split4(A, tix(A, i, 4 * lane), sv);
                store_split4(A, tix(A, i, 4 * (nch + lane)), f4scale(acc, inv));
            }
            if (wide && lane + 32 < nch) {
                store_split4(A, tix(A, i, 4 * (lane + 32)), sv2);
                store_split4(A, tix(A, i, 4 * (nch + lane + 32)), f4scale(acc2, inv));
            }
        }
        if (++b == NB) { b = 0; phase ^= 1u; }
    }
}

// ------------------------------------------------------------------ layer-1 gather, wide rows
// k_agg_l1_bulk for rows wider than 1 KB (Reddit: 604 floats = 2.4 KB): a destination row's items
// (self row, then its c neighbours in CSR order) are streamed through the warp's NB buffers in
// chunks of G rows (G sized so the buffers of 4 warps fit one block per SM, 7 for Reddit); the
// warp accumulates a row over its chunks and writes [self | mean] after the last one.  Same
// arithmetic and order as k_agg_sage (bit-identical operand planes).
template <int NB, int CPL>
__global__ void __launch_bounds__(kL1Warps * 32) k_agg_l1_stream(const int32_t* __restrict__ rows_ptr,
        const float* __restrict__ X, int in_pad, const int32_t* __restrict__ smap,
        const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col, Split A, int fixed_k, int G) {
    extern __shared__ __align__(128) unsigned char l1_smem[];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    uint64_t* bar = reinterpret_cast<uint64_t*>(l1_smem) + warp * NB;
    const uint32_t row_bytes = (uint32_t)in_pad * 4u;
    float* ring = reinterpret_cast<float*>(l1_smem + 128 + (size_t)warp * NB * G * row_bytes);
    if (lane == 0) {
#pragma unroll
        for (int b = 0; b < NB; ++b) mbar_init(&bar[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_async_smem();
    }
    __syncwarp();
    pdl_trigger();
    pdl_wait();
    const int n = *rows_ptr;
    const int nch = in_pad >> 2;
    const int W = total_warps();
    const int gw = global_warp();
    for (int i = n + gw; i < round64(n); i += W)
        for (int ch = lane; ch < 2 * nch; ch += 32) store_split4(A, tix(A, i, 4 * ch), kZero4);
    const uint64_t pol = policy_evict_normal();
    struct Idx { int nb, self, c; };
    auto fetch = [&](int i) {
        Idx x{0, 0, 0};
        if (i >= n) return x;
        if (fixed_k) {
            if (lane < fixed_k) x.nb = col[i * fixed_k + lane];
            x.c = rowptr[i];
        } else {
            const int beg = rowptr[i];
            x.c = rowptr[i + 1] - beg;
            if (lane < x.c) x.nb = col[beg + lane];
        }
        x.self = smap ? smap[i] : i;
        return x;
    };
    // producer state: the row being issued (its indices), the chunk within it, the next row
    int prow = gw, pq = 0;
    Idx px = fetch(prow);
    int nrow = gw + W;
    Idx nx = fetch(nrow);
    int mrow[NB], mq[NB], mitems[NB], mlast[NB];   // what each buffer holds
    auto issue = [&](int b) {
        if (prow >= n) { mrow[b] = n; return; }
        const int tot = px.c + 1;                    // items of the row: self + neighbours
        const int items = min(G, tot - pq * G);
        float* buf = ring + (size_t)b * G * in_pad;
        if (lane == 0) mbar_expect_tx(&bar[b], (uint32_t)items * row_bytes);
        __syncwarp();
        const int it = pq * G + lane;                // this lane's item
        const int nbv = __shfl_sync(0xffffffffu, px.nb, max(it - 1, 0) & 31);
        if (lane < items) {
            const int r = it == 0 ? px.self : nbv;
            bulk_g2s(buf + (size_t)lane * in_pad, X + (int64_t)r * in_pad, row_bytes, &bar[b], pol);
        }
        mrow[b] = prow; mq[b] = pq; mitems[b] = items; mlast[b] = (pq + 1) * G >= tot;
        if (mlast[b]) { prow = nrow; px = nx; pq = 0; nrow += W; nx = fetch(nrow); }
        else ++pq;
    };
#pragma unroll
    for (int b = 0; b < NB; ++b) issue(b);
    uint32_t phase = 0;
    float4 sv[CPL], acc[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) { sv[c] = kZero4; acc[c] = kZero4; }
    bool done = false;
    while (!done) {
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            if (done) break;
            const int i = mrow[b];
            if (i >= n) { done = true; break; }
            const int q = mq[b], items = mitems[b], last = mlast[b];
            mbar_wait(&bar[b], phase);
            const float* buf = ring + (size_t)b * G * in_pad;
            int j0 = 0;
            if (q == 0) {   // a new row: its self row opens the chunk
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int ch = lane + 32 * c;
                    sv[c] = ch < nch ? reinterpret_cast<const float4*>(buf)[ch] : kZero4;
                    acc[c] = kZero4;
                }
                j0 = 1;
            }
            for (int j = j0; j < items; ++j) {
                const float4* rowp = reinterpret_cast<const float4*>(buf + (size_t)j * in_pad);
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int ch = lane + 32 * c;
                    if (ch < nch) acc[c] = f4add(acc[c], rowp[ch]);
                }
            }
            fence_async_smem();
            __syncwarp();
            issue(b);   // re-arm with the next chunk of the stream
            if (last) {
                const int c_tot = q * G + items - 1;   // neighbours of row i
                const float inv = c_tot ? 1.0f / (float)c_tot : 0.f;   // one division per row (R23)
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int ch = lane + 32 * c;
                    if (ch < nch) {
                        store_split4(A, tix(A, i, 4 * ch), sv[c]);
                        store_split4(A, tix(A, i, 4 * (nch + ch)), f4scale(acc[c], inv));
                    }
                }
            }
        }
        phase ^= 1u;
    }
}

// GCN: A[i] = Σ_e H[c_e] / sqrt(d_in(i) d_out(c_e)) + H[i] / sqrt(d_in(i) d_out(i)),
// d_in(i) = deg(i) + 1, d_out(c) = outdeg_blk(c) + [c < n_dst]  (R12).
template <int CPL, bool SH>
__global__ void __launch_bounds__(256) k_agg_gcn(const int32_t* __restrict__ rows_ptr,
        const int32_t* __restrict__ ndst_ptr, FeatRows H, int in_pad, int lda,
        const int32_t* __restrict__ gmap, const int32_t* __restrict__ smap,
        const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
        const int32_t* __restrict__ trowptr, Split A) {
    pdl_trigger();
    pdl_wait();
    const int n = *rows_ptr;
    const int nr = round64(n);
    const int ndst = *ndst_ptr;
    const int lane = lane_id();
    const int nch = in_pad >> 2;
    for (int i = global_warp(); i < nr; i += total_warps()) {
        if (i >= n) {
            for (int ch = lane; ch < (lda >> 2); ch += 32) store_split4(A, tix(A, i, 4 * ch), kZero4);
            continue;
        }
        const int beg = rowptr[i], end = rowptr[i + 1];
        const float din = (float)(end - beg + 1);
        float4 acc[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) acc[c] = kZero4;
        for (int e0 = beg; e0 < end; e0 += 32) {
            const int m = min(32, end - e0);
            int myrow = 0;
            float myw = 0.f;
            if (lane < m) {
                const int c = col[e0 + lane];
                myrow = gmap ? gmap[c] : c;
                const float dout = (float)(trowptr[c + 1] - trowptr[c] + (c < ndst ? 1 : 0));
                myw = 1.0f / sqrtf(din * dout);
            }
            for (int q = 0; q < m; ++q) {
                const int r = __shfl_sync(kFull, myrow, q);
                const float w = __shfl_sync(kFull, myw, q);
                const float4* p = frow<SH>(H, r, in_pad);
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int ch = lane + 32 * c;
                    if (ch < nch) acc[c] = f4fma(w, __ldg(p + ch), acc[c]);
                }
            }
        }
        const float dself = (float)(trowptr[i + 1] - trowptr[i] + 1);
        const float ws = 1.0f / sqrtf(din * dself);
        const int self = smap ? smap[i] : i;
        const float4* ps = frow<SH>(H, self, in_pad);
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            const int ch = lane + 32 * c;
            if (ch < nch) store_split4(A, tix(A, i, 4 * ch), f4fma(ws, __ldg(ps + ch), acc[c]));
        }
    }
}

// ------------------------------------------------------------------ backward aggregation
// dA rows >= dlim are not computed (ShaDow last layer: only the seeds' rows carry loss,
// the exact receptive-field pruning of DESIGN.md R19) and contribute nothing.
// Software-pipelined over the warp's rows u, u+W, u+2W, ...: the next row's transposed-CSR
// range and its first 32 destinations are loaded while the current row's dA rows are in flight,
// so a row costs about one dependent memory round trip instead of three.
template <int CPL, bool GCN>
__global__ void __launch_bounds__(256, 4) k_spmm_bwd(int h, const StepState* __restrict__ st,
        const int32_t* __restrict__ dlim_ptr, const float* __restrict__ dA, int in_pad,
        const int32_t* __restrict__ rowptr, const int32_t* __restrict__ trowptr,
        const int32_t* __restrict__ tdst, const uint32_t* __restrict__ hmask, int mask_ld, Split dPre) {
    pdl_trigger();
    pdl_wait();
    const int nsrc = st->n_src[h];
    const int nr = round64(nsrc);
    const int ndst = st->n_dst[h];
    const int dlim = *dlim_ptr;
    const int lane = lane_id();
    const int nch = in_pad >> 2;
    const int64_t lda = GCN ? in_pad : 2 * (int64_t)in_pad;
    const int moff = GCN ? 0 : nch;   // dM half of [dSelf | dM]
    const int W = total_warps();
    int u = global_warp();
    // prologue: row u's edge range and first chunk of destinations
    int cb = 0, ce = 0, ci = -1;
    if (u < nsrc) {
        cb = trowptr[u];
        ce = trowptr[u + 1];
        if (u < dlim) prefetch_rows_l2(dA + (int64_t)u * lda, nullptr, in_pad, lane);
    }
    if (lane < ce - cb) ci = tdst[cb + lane];
    for (; u < nr; u += W) {
        if (u >= nsrc) {
            for (int ch = lane; ch < nch; ch += 32) store_split4(dPre, tix(dPre, u, 4 * ch), kZero4);
            continue;
        }
        const int un = u + W;
        int nb = 0, ne = 0;
        if (un < nsrc) { nb = trowptr[un]; ne = trowptr[un + 1]; }
        // the next row's dA-self row goes to L2 now (it is read at the end of that row: no
        // registers held across its edge loop)
        if (un < dlim) prefetch_rows_l2(dA + (int64_t)un * lda, nullptr, in_pad, lane);
        const float dout = (float)(ce - cb + (u < ndst ? 1 : 0));
        // this row's ReLU bits and dA-self row do not depend on the edge loop: in flight with it
        const uint32_t* mp = hmask + (int64_t)u * mask_ld;
        const float4* sp = reinterpret_cast<const float4*>(dA + (int64_t)u * lda);
        uint32_t hv[CPL];
        float4 sv[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            const int ch = lane + 32 * c;
            hv[c] = ch < nch ? __ldg(mp + (ch >> 3)) >> ((4 * ch) & 31) : 0u;
            sv[c] = (ch < nch && u < dlim) ? __ldg(sp + ch) : kZero4;
        }
        float4 acc[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) acc[c] = kZero4;
        for (int e0 = cb; e0 < ce; e0 += 32) {
            const int m = min(32, ce - e0);
            const int t = e0 == cb ? ci : (lane < m ? tdst[e0 + lane] : -1);
            int myi = -1;
            float myd = 1.f;
            if (lane < m && t < dlim) {
                myi = t;
                const float din = (float)(rowptr[t + 1] - rowptr[t] + (GCN ? 1 : 0));
                // edge weight: GCN 1/sqrt(d_in d_out), SAGE 1/deg(dst) (one division per edge, not
                // per element: the backward of the mean is fma(1/deg, dM, acc))
                myd = GCN ? 1.0f / sqrtf(din * dout) : 1.0f / din;
            }
            int q = 0;
            for (; q + 2 <= m; q += 2) {   // two dA rows in flight; accumulation in edge order
                const int i0 = __shfl_sync(kFull, myi, q), i1 = __shfl_sync(kFull, myi, q + 1);
                const float d0 = __shfl_sync(kFull, myd, q), d1 = __shfl_sync(kFull, myd, q + 1);
                const float4* p0 = reinterpret_cast<const float4*>(dA + (int64_t)max(i0, 0) * lda) + moff;
                const float4* p1 = reinterpret_cast<const float4*>(dA + (int64_t)max(i1, 0) * lda) + moff;
                float4 v0[CPL], v1[CPL];
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int ch = lane + 32 * c;
                    v0[c] = (ch < nch && i0 >= 0) ? __ldg(p0 + ch) : kZero4;
                    v1[c] = (ch < nch && i1 >= 0) ? __ldg(p1 + ch) : kZero4;
                }
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    if (i0 >= 0) acc[c] = f4fma(d0, v0[c], acc[c]);
                    if (i1 >= 0) acc[c] = f4fma(d1, v1[c], acc[c]);
                }
            }
            if (q < m) {
                const int i0 = __shfl_sync(kFull, myi, q);
                const float d0 = __shfl_sync(kFull, myd, q);
                if (i0 >= 0) {
                    const float4* p0 = reinterpret_cast<const float4*>(dA + (int64_t)i0 * lda) + moff;
#pragma unroll
                    for (int c = 0; c < CPL; ++c) {
                        const int ch = lane + 32 * c;
                        if (ch < nch) {
                            const float4 v = __ldg(p0 + ch);
                            acc[c] = f4fma(d0, v, acc[c]);
                        }
                    }
                }
            }
        }
        // next row's first destinations (its range has arrived by now)
        ci = -1;
        if (lane < ne - nb) ci = tdst[nb + lane];
        float wself = 0.f;
        if (GCN && u < dlim) {
            const float din = (float)(rowptr[u + 1] - rowptr[u] + 1);
            wself = 1.0f / sqrtf(din * dout);
        }
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            const int ch = lane + 32 * c;
            if (ch < nch) {
                float4 a = acc[c];
                if (u < dlim) a = GCN ? f4fma(wself, sv[c], a) : f4add(a, sv[c]);
                // ReLU'(pre) = [H > 0]  (ReLU'(0) = 0): the forward GEMM's sign bits
                a.x = (hv[c] & 1u) ? a.x : 0.f; a.y = (hv[c] & 2u) ? a.y : 0.f;
                a.z = (hv[c] & 4u) ? a.z : 0.f; a.w = (hv[c] & 8u) ? a.w : 0.f;
                store_split4(dPre, tix(dPre, u, 4 * ch), a);
            }
        }
        cb = nb;
        ce = ne;
    }
}

// ------------------------------------------------------------------ balanced (merge-path) aggregation
// ShaDow blocks (the induced subgraph) have power-law rows (thousands of entries at
// the hubs): a warp per row leaves the grid waiting on the hub rows.  Here the rows and edges of
// the traversed CSR form one merged item sequence (row r owns items [rowptr[r]+r, rowptr[r+1]+r],
// its edges then an end marker) cut into units of T = max(16, items / 2^16) items; a warp takes a unit, finds its
// first row by a 32-ary search of rowptr[r]+r, and sums the unit's part of every row it touches.
// A row inside one unit is finished by that warp.  A row spread over units ua..ub leaves one
// partial per unit (ua: slot 2ua+1 "out", later units: slot 2u "in"); the warp whose piece
// completes the per-row count sums the partials in unit order (fixed order: deterministic) and
// finishes the row.  Counters are reset by the finishing warp.
//   FWD (SAGE/GCN): traversed CSR = the block, rows = output rows, edges = local sources.
//   BWD (SAGE/GCN): traversed CSR = the transposed block, rows = sources u, edges = dst rows t.
// rmask (receptive-field pruning, R19): rows r with rmask[r] != *tag are not computed
// (FWD), dst rows t with rmask[t] != *tag carry no gradient (BWD).
constexpr int kBalTmin = 16, kBalUnits = 1 << 16;
struct BalArgs {
    const int32_t* n_ptr;      // rows traversed (FWD: output rows; BWD: n_src of the block)
    const int32_t* ndst_ptr;   // n_dst of the block (GCN self loops)
    const int32_t* dlim_ptr;   // BWD: dA rows < dlim carry gradient
    const int32_t* rowptr;     // traversed CSR
    const int32_t* col;        // FWD: local sources; BWD: destinations (ascending per row)
    const int32_t* orow;       // the other direction's row pointer (FWD GCN: d_out; BWD: d_in(dst))
    const uint32_t* rmask;
    const uint32_t* tag_ptr;
    FeatRows H;                // FWD input rows
    const int32_t* gmap;       // FWD: row id of local node c in H (layer 1: global ids)
    const float* dA;           // BWD
    const uint32_t* hmask;     // BWD: ReLU decisions of the previous layer (bit per element)
    int mask_ld;
    int in_pad;
    Split out;                 // FWD: A (SAGE [self | mean], GCN Â H); BWD: dPre
    int out_w;                 // columns of `out` (zero tail rows)
    float* part;               // partial rows [2 * units][in_pad]
    int32_t* cnt;              // per-row piece counters (zero between launches)
    int ch0, nchp;             // column panel: float4 chunks [ch0, ch0 + nchp) of every row
    // ShaDow receptive-field compaction (R19): traverse only the listed block rows
    // rlist[0..n) (rowptr is then the listed rows' own prefix sum and edges are read at
    // brow[rlist[r]] + offset; output row r is compact); BWD dmap[t] = dA row of destination t
    // (-1: no gradient), replacing dlim / rmask.
    const int32_t* rlist;
    const int32_t* brow;
    const int32_t* dmap;
};

template <int CPL, int MODE, bool SH = false>   // MODE: 0 FWD SAGE, 1 FWD GCN, 2 BWD SAGE, 3 BWD GCN
__device__ __forceinline__ void agg_bal_body(const BalArgs& a) {
    constexpr bool BWD = MODE >= 2, GCN = (MODE & 1) != 0;
    pdl_trigger();
    pdl_wait();
    const int n = *a.n_ptr;
    const int lane = lane_id();
    const int nch = a.in_pad >> 2;
    // column panel of this launch: chunks [c0, c0 + pch) of every row (the launcher splits wide
    // rows into panels whose working set fits in L2; partial slots and counters are per launch)
    const int c0 = a.ch0, pch = a.nchp;
    const int W = total_warps();
    if (c0 == 0)
        for (int i = n + global_warp(); i < round64(n); i += W)
            for (int ch = lane; ch < (a.out_w >> 2); ch += 32) store_split4(a.out, tix(a.out, i, 4 * ch), kZero4);
    const int ndst = *a.ndst_ptr;
    const int dlim = BWD ? *a.dlim_ptr : 0;
    const uint32_t tag = a.rmask ? *a.tag_ptr : 0u;
    const int64_t items = (int64_t)n + a.rowptr[n];
    // unit size: at least kBalTmin items, at most kBalUnits units (the partial-slot capacity)
    const int T = (int)max((int64_t)kBalTmin, (items + kBalUnits - 1) / kBalUnits);
    const int nunits = (int)((items + T - 1) / T);
    const int64_t ldd = GCN ? a.in_pad : 2 * a.in_pad;   // BWD dA row (SAGE: [dSelf | dM])
    auto put = [&](int64_t idx, float4 v) { store_split4(a.out, idx, v); };

    // finish row r from its full sum `acc` (fwd: normalise + self term; bwd: self term + ReLU')
    auto finish = [&](int r, int R, int rb, int re, float4 (&acc)[CPL], bool any) {
        if constexpr (!BWD) {
            const int self = a.gmap ? a.gmap[R] : R;
            const float4* ps = frow<SH>(a.H, self, a.in_pad);
            if constexpr (GCN) {
                const float din = (float)(re - rb + 1);
                const float dself = (float)(a.orow[R + 1] - a.orow[R] + (R < ndst ? 1 : 0));
                const float ws = 1.0f / sqrtf(din * dself);
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int ch = lane + 32 * c;
                    if (ch < pch) put(tix(a.out, r, 4 * (c0 + ch)), f4fma(ws, __ldg(ps + c0 + ch), acc[c]));
                }
            } else {
                const int deg = re - rb;
                const float inv = deg ? 1.0f / (float)deg : 0.f;
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int ch = lane + 32 * c;
                    if (ch < pch) {
                        put(tix(a.out, r, 4 * (c0 + ch)), __ldg(ps + c0 + ch));
                        put(tix(a.out, r, 4 * (nch + c0 + ch)), f4scale(acc[c], inv));
                    }
                }
            }
        } else {
            const int sr = a.dmap ? a.dmap[R] : ((R < dlim && (!a.rmask || a.rmask[R] == tag)) ? R : -1);
            const bool self_on = sr >= 0;
            float wself = 1.f;
            if (GCN && self_on) {
                const float din = (float)(a.orow[R + 1] - a.orow[R] + 1);
                const float dout = (float)(re - rb + (R < ndst ? 1 : 0));
                wself = 1.0f / sqrtf(din * dout);
            }
            const uint32_t* mp = a.hmask + (int64_t)r * a.mask_ld;
            const float4* sp = reinterpret_cast<const float4*>(a.dA + (int64_t)max(sr, 0) * ldd);
            if (!any && !self_on) {   // no gradient reaches row r: dPre = 0 (no reads)
                for (int ch = lane; ch < pch; ch += 32) store_split4(a.out, tix(a.out, r, 4 * (c0 + ch)), kZero4);
                return;
            }
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                const int ch = lane + 32 * c;
                if (ch < pch) {
                    const int cc = c0 + ch;
                    float4 v = acc[c];
                    if (self_on) v = GCN ? f4fma(wself, __ldg(sp + cc), v) : f4add(v, __ldg(sp + cc));
                    const uint32_t h = __ldg(mp + (cc >> 3)) >> ((4 * cc) & 31);   // ReLU decisions
                    v.x = (h & 1u) ? v.x : 0.f; v.y = (h & 2u) ? v.y : 0.f;
                    v.z = (h & 4u) ? v.z : 0.f; v.w = (h & 8u) ? v.w : 0.f;
                    put(tix(a.out, r, 4 * cc), v);
                }
            }
        }
    };

    for (int u = global_warp(); u < nunits; u += W) {
        const int64_t d0 = (int64_t)u * T, d1 = min(d0 + (int64_t)T, items);
        // r0 = max r in [0, n] with rowptr[r] + r <= d0 (32-ary search; f(r) = rowptr[r]+r increases)
        int lo = 0, hi = n;
        while (hi > lo) {
            const int step = (hi - lo + 31) / 32;
            const int c = lo + (lane + 1) * step;
            const bool ok = c <= hi && (int64_t)a.rowptr[c] + c <= d0;
            const int k = __popc(__ballot_sync(kFull, ok));
            lo += k * step;
            hi = min(hi, lo + step - 1);
        }
        int wb = lo;                                   // window of 32 row pointers from wb
        int rpw = a.rowptr[min(wb + lane, n)];
        for (int r = lo;; ++r) {
            if (r - wb >= 31) { wb = r; rpw = a.rowptr[min(wb + lane, n)]; }
            const int rb = __shfl_sync(kFull, rpw, r - wb), re = __shfl_sync(kFull, rpw, r - wb + 1);
            const int64_t fr = (int64_t)rb + r, fr1 = (int64_t)re + r + 1;
            if (r >= n || fr >= d1) break;
            const int R = a.rlist ? a.rlist[r] : r;          // block row
            const int eoff = a.rlist ? a.brow[R] - rb : 0;   // edge e of row r is block entry e + eoff
            if constexpr (!BWD) {
                if (a.rmask && a.rmask[R] != tag) continue;   // row outside the receptive field
            }
            const int eb = max(rb, (int)(d0 - r)), ee = min(re, (int)(d1 - r));
            float4 acc[CPL];
#pragma unroll
            for (int c = 0; c < CPL; ++c) acc[c] = kZero4;
            const float din_r = (float)(re - rb + 1);                       // FWD GCN: d_in(r)
            const float dout_r = (float)(re - rb + (R < ndst ? 1 : 0));     // BWD GCN: d_out(u)
            bool any = false;   // a contributing edge was seen (else the row sum is exactly 0)
            for (int e0 = eb; e0 < ee; e0 += 32) {
                const int m = min(32, ee - e0);
                int myrow = -1;
                float myw = 0.f;
                if (lane < m) {
                    const int c = a.col[e0 + lane + eoff];
                    if constexpr (!BWD) {
                        myrow = a.gmap ? a.gmap[c] : c;
                        if (GCN) {
                            const float dout = (float)(a.orow[c + 1] - a.orow[c] + (c < ndst ? 1 : 0));
                            myw = 1.0f / sqrtf(din_r * dout);
                        }
                    } else {
                        const int dr = a.dmap ? a.dmap[c] : ((c < dlim && (!a.rmask || a.rmask[c] == tag)) ? c : -1);
                        if (dr >= 0) {
                            myrow = dr;
                            const float din = (float)(a.orow[c + 1] - a.orow[c] + (GCN ? 1 : 0));
                            myw = GCN ? 1.0f / sqrtf(din * dout_r) : 1.0f / din;
                        }
                    }
                }
                int mv = m;
                if constexpr (BWD) {   // compact the contributing edges (order kept) to the low lanes
                    const unsigned vb = __ballot_sync(kFull, myrow >= 0);
                    mv = __popc(vb);
                    if (mv == 0) continue;
                    const int src = (int)(__fns(vb, 0, lane + 1) & 31u);
                    myrow = __shfl_sync(kFull, myrow, src);
                    myw = __shfl_sync(kFull, myw, src);
                }
                any = true;
                // kU rows in flight; accumulation in edge order
                constexpr int kU = CPL <= 2 ? 4 : 2;
                for (int q = 0; q < mv; q += kU) {
                    float4 v[kU][CPL];
                    int rr[kU];
                    float ww[kU];
#pragma unroll
                    for (int j = 0; j < kU; ++j) {
                        rr[j] = __shfl_sync(kFull, myrow, min(q + j, 31));
                        ww[j] = __shfl_sync(kFull, myw, min(q + j, 31));
                        if (q + j >= mv) rr[j] = -1;
                        const float4* p;
                        if constexpr (!BWD) p = frow<SH>(a.H, max(rr[j], 0), a.in_pad) + c0;
                        else p = reinterpret_cast<const float4*>(a.dA + (int64_t)max(rr[j], 0) * ldd) + (GCN ? 0 : nch) + c0;
#pragma unroll
                        for (int c = 0; c < CPL; ++c) {
                            const int ch = lane + 32 * c;
                            v[j][c] = (ch < pch && rr[j] >= 0) ? __ldg(p + ch) : kZero4;
                        }
                    }
#pragma unroll
                    for (int j = 0; j < kU; ++j) {
                        if (rr[j] < 0) continue;
#pragma unroll
                        for (int c = 0; c < CPL; ++c)
                            acc[c] = (GCN || BWD) ? f4fma(ww[j], v[j][c], acc[c]) : f4add(acc[c], v[j][c]);
                    }
                }
            }
            const bool started = fr >= d0, completed = fr1 <= d1;
            if (started && completed) { finish(r, R, rb, re, acc, any); continue; }
            // a piece of a row spread over several units
            float* slot = a.part + (int64_t)(started ? 2 * u + 1 : 2 * u) * a.in_pad;
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                const int ch = lane + 32 * c;
                if (ch < pch) __stcg(reinterpret_cast<float4*>(slot) + ch, acc[c]);
            }
            __threadfence();
            __syncwarp();
            int prev = 0;
            if (lane == 0) prev = atomicAdd(a.cnt + r, 1);
            prev = __shfl_sync(kFull, prev, 0);
            const int ua = (int)(fr / T), ub = (int)((fr1 - 1) / T);
            if (prev != ub - ua) continue;
            __threadfence();
#pragma unroll
            for (int c = 0; c < CPL; ++c) acc[c] = kZero4;
            for (int uu = ua; uu <= ub; ++uu) {   // unit order
                const float4* ps = reinterpret_cast<const float4*>(a.part + (int64_t)(uu == ua ? 2 * uu + 1 : 2 * uu) * a.in_pad);
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int ch = lane + 32 * c;
                    if (ch < pch) acc[c] = f4add(acc[c], __ldcg(ps + ch));
                }
            }
            if (lane == 0) a.cnt[r] = 0;
            finish(r, R, rb, re, acc, true);
        }
    }
}

// Forward and backward instantiations differ in register demand: the backward ones are capped
// at 3 blocks/SM (<= 85 registers; uncapped the GCN backward compiles to 101, 2 blocks/SM),
// the forward ones keep the compiler's choice (a cap measured slower).
template <int CPL, int MODE, bool SH>
__global__ void __launch_bounds__(256) k_agg_bal(BalArgs a) { agg_bal_body<CPL, MODE, SH>(a); }
template <int CPL, int MODE>
__global__ void __launch_bounds__(256, 3) k_agg_bal_bwd(BalArgs a) { agg_bal_body<CPL, MODE>(a); }

// mask[r] = tag for the rows the last layer reads: the seeds r < *nseed_ptr and their
// in-neighbours in the block (ShaDow receptive field of the last layer, R19).
__global__ void __launch_bounds__(256) k_rf_mark(const int32_t* __restrict__ nseed_ptr, const int32_t* __restrict__ rowptr,
                                                 const int32_t* __restrict__ col, const uint32_t* __restrict__ tag_ptr,
                                                 uint32_t* __restrict__ mask) {
    pdl_trigger();
    pdl_wait();
    const int b = *nseed_ptr;
    const uint32_t tag = *tag_ptr;
    const int ne = rowptr[b];   // the seeds are the block's first rows: their edges are [0, rowptr[b])
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    for (int i = tid; i < b; i += nth) mask[i] = tag;
    for (int e = tid; e < ne; e += nth) mask[col[e]] = tag;
}

// Receptive-field compaction (launch_rf_compact): per block row r < cap, in = [mask[r] == tag].
__global__ void k_rf_prep(const uint32_t* __restrict__ mask, const uint32_t* __restrict__ tag_ptr, int cap,
                          const int32_t* __restrict__ rowptr, const int32_t* __restrict__ trow,
                          int32_t* __restrict__ flags, int32_t* __restrict__ degf, int32_t* __restrict__ degt) {
    pdl_trigger();
    pdl_wait();
    const uint32_t tag = *tag_ptr;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < cap; r += gridDim.x * blockDim.x) {
        const bool in = mask[r] == tag;
        flags[r] = in ? 1 : 0;
        degf[r] = in ? rowptr[r + 1] - rowptr[r] : 0;
        degt[r] = in ? trow[r + 1] - trow[r] : 0;
    }
}
__global__ void k_rf_scatter(int cap, const int32_t* __restrict__ flags, const int32_t* __restrict__ degf,
                             const int32_t* __restrict__ degt, const int32_t* __restrict__ pos,
                             const int32_t* __restrict__ scf, const int32_t* __restrict__ sct, int32_t* __restrict__ rf_list,
                             int32_t* __restrict__ rf_pos, int32_t* __restrict__ sub, int32_t* __restrict__ subt,
                             int32_t* __restrict__ n_rf) {
    pdl_trigger();
    pdl_wait();
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < cap; r += gridDim.x * blockDim.x) {
        if (flags[r]) {
            const int p = pos[r];
            rf_list[p] = r;
            rf_pos[r] = p;
            sub[p] = scf[r];
            if (subt != sub) subt[p] = sct[r];
        } else {
            rf_pos[r] = -1;
        }
        if (r == cap - 1) {
            const int n = pos[r] + flags[r];
            *n_rf = n;
            sub[n] = scf[r] + degf[r];
            if (subt != sub) subt[n] = sct[r] + degt[r];
        }
    }
}

// ------------------------------------------------------------------ weights, reduce, SGD
// dW of layers [l0, l1) in one launch: G[off_l + r*out + c] = Σ_z part_l[z][rpad(r)*n_pad + c]
// (split order fixed: deterministic), stored to `grads` (when non-null) and, for the peer exchange
// (x.world > 0), to slot `rank` of every rank's inbox (NVLink stores to CUDA-IPC mappings).  With
// x.signal the last block then publishes the step's sequence number in every rank's flag array.
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__global__ void k_wgrad_reduce(PackAll P, int l0, int l1, float* __restrict__ grads, PeerX x) {
    pdl_trigger();
    pdl_wait();
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const unsigned long long seq = x.world ? *x.seq : 0ull;
    const int64_t slot = x.world ? ((int64_t)(seq & 1ull) * x.world + x.rank) * x.pcount : 0;
    int64_t base = 0;   // the layers' entries form one index space: one pass of the grid in all
    for (int l = l0; l < l1; ++l) {
        const PackLayer& L = P.l[l];
        const int64_t total = (int64_t)L.rows * L.out;
        const int64_t g0 = base > tid ? tid + ((base - tid + nth - 1) / nth) * nth : tid;
        base += total;
        for (int64_t f = g0 - (base - total); f < total; f += nth) {
            const int r = (int)(f / L.out), c = (int)(f % L.out);
            const int rp = P.sage ? (r / L.in) * L.in_pad + (r % L.in) : r;
            const float* src = L.part + (int64_t)rp * L.n_pad + c;
            float s = 0.f;
            for (int z0 = 0; z0 < L.splits; z0 += 8) {   // fixed split order; 8 partials in flight
                float v[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] = z0 + j < L.splits ? src[(z0 + j) * L.split_stride] : 0.f;
#pragma unroll
                for (int j = 0; j < 8; ++j) if (z0 + j < L.splits) s += v[j];
            }
            if (grads) grads[L.poff + f] = s;
            for (int q = 0; q < x.world; ++q) x.inbox[q][slot + L.poff + f] = s;
        }
    }
    if (!x.world) return;
    __threadfence_system();   // this thread's peer stores before anything it does next
    if (!x.signal) return;
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(x.done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence_system();
        for (int q = 0; q < x.world; ++q) st_release_sys(x.flags[q] + x.rank, seq);
        *x.done = 0u;
    }
}

// SGD (W <- W - lr G, §2.2) or Adam (NEXT-4, the listings' torch.optim.Adam,
// P:L398) fused with the repack of the GEMM weight planes W [K_pad x N_pad] (coalesced in that
// order; padding entries stay the zeros written at creation).  Each parameter is visited exactly
// once.  grads == nullptr: pack only.
// reduce (single rank, no exchange in between): G is first reduced from the wgrad split-K
// partials in the fixed split order (the arithmetic of k_wgrad_reduce_all) and stored.
// Adam: t = *o.t + 1 for every thread; bias corrections in fp64; the last block to finish
// stores t (the next step's kernel starts after this one completes).
// Peer exchange (x.world > 0): every block first waits until each rank r has published this step's
// sequence number in this rank's flag array, then G = Σ_{r = 0..world-1} inbox[r] (rank order: the
// same bits on every rank); the last block advances the sequence number.
__global__ void k_sgd_pack(PackAll P, float* __restrict__ params, float* __restrict__ grads, float lr, int reduce,
                           OptState o, PeerX x) {
    pdl_trigger();
    pdl_wait();
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    unsigned long long seq = 0;
    const float* inbox = nullptr;
    if (x.world && grads) {
        seq = *x.seq;
        if (threadIdx.x < x.world) {
            // a rank that never arrives (crashed peer, mismatched step sequence) aborts the kernel
            // after 30 s instead of hanging the device
            unsigned long long t0, t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            while (ld_acquire_sys(x.my_flags + threadIdx.x) < seq) {
                __nanosleep(256);
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                if (t - t0 > 30000000000ull) __trap();
            }
        }
        __syncthreads();
        inbox = x.my_inbox + (int64_t)(seq & 1ull) * x.world * x.pcount;
    }
    const bool adam = o.m != nullptr && grads != nullptr;
    int t = 0;
    float step = 0.f, inv_sqrt_bc2 = 0.f;
    if (adam) {
        t = *o.t + 1;
        const double bc1 = 1.0 - pow((double)o.beta1, (double)t), bc2 = 1.0 - pow((double)o.beta2, (double)t);
        step = (float)((double)lr / bc1);
        inv_sqrt_bc2 = (float)(1.0 / sqrt(bc2));
    }
    int64_t base = 0;   // the layers' entries form one index space: one pass of the grid in all
    for (int l = 0; l < P.n; ++l) {
        const PackLayer& L = P.l[l];
        const int64_t total = (int64_t)L.k_pad * L.n_pad;
        const int64_t g0 = base > tid ? tid + ((base - tid + nth - 1) / nth) * nth : tid;
        base += total;
        for (int64_t f = g0 - (base - total); f < total; f += nth) {
            const int rp = (int)(f / L.n_pad), c = (int)(f % L.n_pad);
            int r = -1;
            if (P.sage) { const int half = rp / L.in_pad, j = rp % L.in_pad; if (j < L.in && half < 2) r = half * L.in + j; }
            else if (rp < L.in) r = rp;
            if (r < 0 || c >= L.out) continue;
            const int64_t idx = L.poff + (int64_t)r * L.out + c;
            float w = params[idx];
            if (grads) {
                float gr;
                if (reduce) {   // fixed split order; 8 partials in flight per round
                    gr = 0.f;
                    for (int z0 = 0; z0 < L.splits; z0 += 8) {
                        float v[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) v[j] = z0 + j < L.splits ? L.part[(z0 + j) * L.split_stride + f] : 0.f;
#pragma unroll
                        for (int j = 0; j < 8; ++j) if (z0 + j < L.splits) gr += v[j];
                    }
                    grads[idx] = gr;
                } else if (inbox) {   // the peers' gradients, summed in rank order
                    gr = 0.f;
                    for (int q = 0; q < x.world; ++q) gr += __ldcv(inbox + (int64_t)q * x.pcount + idx);
                    grads[idx] = gr;
                } else {
                    gr = grads[idx];
                }
                if (adam) {   // m <- b1 m + (1-b1) g; v <- b2 v + (1-b2) g^2; W -= step m / (sqrt(v)/sqrt(bc2) + eps)
                    const float mm = o.beta1 * o.m[idx] + (1.f - o.beta1) * gr;
                    const float vv = o.beta2 * o.v[idx] + (1.f - o.beta2) * gr * gr;
                    o.m[idx] = mm;
                    o.v[idx] = vv;
                    w = w - step * mm / (sqrtf(vv) * inv_sqrt_bc2 + o.eps);
                } else {
                    w = fmaf(-lr, gr, w);   // one rounding (the host rank's update, gnnhost.h)
                }
                params[idx] = w;
            }
            store_split1(L.Wkn, f, w);
        }
    }
    if (adam || inbox) {
        __shared__ bool last;
        __syncthreads();
        unsigned* done = adam ? o.done : x.done2;
        if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
        __syncthreads();
        if (last && threadIdx.x == 0) {
            if (adam) *o.t = t;
            if (inbox) *x.seq = seq + 1;
            *done = 0u;
        }
    }
}

// ------------------------------------------------------------------ softmax cross-entropy
// Warp per row.  ℓ_i = max + log Σ exp(z - max) - z_y;  dZ = (softmax - onehot) / b_total.
// The last block to finish sums the row losses in row order (deterministic).
__global__ void __launch_bounds__(256) k_ce(StepState* st, const float* __restrict__ Z, int ldz, int C,
                                            const int32_t* __restrict__ labels, const int32_t* __restrict__ nodes,
                                            Split dZ, float* __restrict__ row_loss, uint32_t* __restrict__ done) {
    pdl_trigger();
    pdl_wait();
    using BR = cub::BlockReduce<float, 256>;
    __shared__ typename BR::TempStorage tmp;
    __shared__ bool last;
    const int b = st->batch_n;
    const int br = round64(b);
    const float inv_bt = 1.0f / (float)max(st->b_total, 1);
    const int lane = lane_id();
    for (int r = global_warp(); r < br; r += total_warps()) {
        if (r >= b) {
            for (int c = lane; c < ldz; c += 32) store_split1(dZ, tix(dZ, r, c), 0.f);
            continue;
        }
        const float* z = Z + (int64_t)r * ldz;
        float m = -INFINITY;
        for (int c = lane; c < C; c += 32) m = fmaxf(m, z[c]);
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
        float s = 0.f;
        for (int c = lane; c < C; c += 32) s += expf(z[c] - m);
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
        const int y = labels[nodes[r]];
        for (int c = lane; c < ldz; c += 32) {
            float v = 0.f;
            if (c < C) v = (expf(z[c] - m) / s - (c == y ? 1.f : 0.f)) * inv_bt;
            store_split1(dZ, tix(dZ, r, c), v);
        }
        if (lane == 0) row_loss[r] = (m + logf(s)) - z[y];
    }
    if (lane == 0) __threadfence();   // only the row_loss writers need to publish
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    float part = 0.f;
    for (int r = threadIdx.x; r < b; r += 256) part += row_loss[r];
    const float tot = BR(tmp).Sum(part);
    if (threadIdx.x == 0) {
        st->loss = tot * inv_bt;
        *done = 0u;
    }
}

__global__ void k_init(float* p, int64_t cnt, float bound, uint64_t seed, uint32_t layer) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t r = method_draw(seed, 4u, layer, (uint32_t)(i >> 32), 0u, 0u, (uint32_t)i);
        const float u = (float)(r >> 8) * (1.0f / 16777216.0f);
        p[i] = (2.f * u - 1.f) * bound;
    }
}

int cpl_of(int in_pad) { return (in_pad / 4 + 31) / 32; }
}  // namespace

#define GS_CPL_DISPATCH_SH(cpl, SHV, KERNEL, ...)                                       \
    switch (cpl) {                                                                      \
        case 1: launch_pdl(KERNEL<1, SHV>, kWarpGrid, 256, 0, s, __VA_ARGS__); break;       \
        case 2: launch_pdl(KERNEL<2, SHV>, kWarpGrid, 256, 0, s, __VA_ARGS__); break;       \
        case 3: launch_pdl(KERNEL<3, SHV>, kWarpGrid, 256, 0, s, __VA_ARGS__); break;       \
        case 4: launch_pdl(KERNEL<4, SHV>, kWarpGrid, 256, 0, s, __VA_ARGS__); break;       \
        case 5: launch_pdl(KERNEL<5, SHV>, kWarpGrid, 256, 0, s, __VA_ARGS__); break;       \
        case 6: launch_pdl(KERNEL<6, SHV>, kWarpGrid, 256, 0, s, __VA_ARGS__); break;       \
        case 7: launch_pdl(KERNEL<7, SHV>, kWarpGrid, 256, 0, s, __VA_ARGS__); break;       \
        default: launch_pdl(KERNEL<8, SHV>, kWarpGrid, 256, 0, s, __VA_ARGS__); break;      \
    }
// local table, or the row-sharded one (FeatRows::shards set; GS_AGG_FORCE_SH=1: the sharded
// instantiation for local tables too, A/B of the code generation only)
static bool force_sh() {
    static const bool f = [] { const char* e = std::getenv("GS_AGG_FORCE_SH"); return e && e[0] == '1'; }();
    return f;
}
#define GS_CPL_DISPATCH(cpl, H, KERNEL, ...)                                             \
    if ((H).shards || force_sh()) { GS_CPL_DISPATCH_SH(cpl, true, KERNEL, __VA_ARGS__) }   \
    else { GS_CPL_DISPATCH_SH(cpl, false, KERNEL, __VA_ARGS__) }

template <int NB, bool G4 = false>
static bool launch_l1_bulk(const int32_t* rows_ptr, const float* X, int in_pad, const int32_t* smap,
                           const int32_t* blk_rowptr, const int32_t* col, Split A, int fixed_k, int slots,
                           cudaStream_t s, const CUtensorMap* xmap = nullptr) {
    const size_t rb = (size_t)in_pad * 4, sb = (rb + 127) & ~size_t(127), gsz = (4 * rb + 127) & ~size_t(127);
    const size_t buf = G4 ? sb + (size_t)((slots - 1 + 3) / 4) * gsz : (size_t)slots * rb;
    size_t smem = 128 + (size_t)kL1Warps * NB * buf;
    if (smem > 200 * 1024) return false;
    // GS_L1_BPS = b: pad the request just past the (b+1)-blocks threshold, so that at most b blocks
    // share an SM and the rest of its shared memory stays free for a co-resident sampling block
    static const int bps = [] { const char* e = std::getenv("GS_L1_BPS"); return e ? std::atoi(e) : 3; }();
    if (bps > 0) smem = std::max(smem, (size_t)(233472 / (bps + 1) - 1024 + 16));
    static std::map<size_t, int> grids;   // smem bytes -> co-resident blocks x SMs (occupancy-derived)
    // the function's dynamic shared-memory limit only grows: tables of several widths share the
    // kernel (a smaller request set later must not lower the limit a cached grid relies on)
    static size_t attr_max = 0;
    if (smem > attr_max) {
        cudaFuncSetAttribute(k_agg_l1_bulk<NB, G4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_max = smem;
    }
    int& grid = grids[smem];
    if (!grid) {
        // the SMs this kernel runs on are configured with the whole 228 KB as shared memory, so a
        // block of the next batch's sampling kernel (35 KB) still fits beside the 3 gather blocks
        // (the driver otherwise picks the smallest split that holds them, 200 KB, and the sampling
        // kernel, which overlaps training, cannot co-reside: measured -12 % mini-batches/s)
        static const int carve = [] { const char* e = std::getenv("GS_L1_CARVE"); return e ? std::atoi(e) : 100; }();
        if (carve >= 0) cudaFuncSetAttribute(k_agg_l1_bulk<NB, G4>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
        int per_sm = 0, dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_agg_l1_bulk<NB, G4>, kL1Warps * 32, smem);
        if (per_sm < 1) return false;
        grid = per_sm * sms;
    }
    static const int xpol = [] { const char* e = std::getenv("GS_L1_XPOL"); return e ? std::atoi(e) : 0; }();
    static const int apol = [] { const char* e = std::getenv("GS_L1_APOL"); return e ? std::atoi(e) : 0; }();
    static const int pdl = [] { const char* e = std::getenv("GS_L1_PDL"); return e ? std::atoi(e) : 1; }();
    if (pdl)
        launch_pdl(k_agg_l1_bulk<NB, G4>, grid, kL1Warps * 32, smem, s, rows_ptr, X, in_pad, smap, blk_rowptr, col, A,
                   fixed_k, slots, xpol, apol, xmap ? *xmap : CUtensorMap{});
    else
    {
        apply_carveout((const void*)k_agg_l1_bulk<NB, G4>);
        k_agg_l1_bulk<NB, G4><<<grid, kL1Warps * 32, smem, s>>>(rows_ptr, X, in_pad, smap, blk_rowptr, col, A, fixed_k,
                                                               slots, xpol, apol, xmap ? *xmap : CUtensorMap{});
    }
    return true;
}

template <int CPL>
static bool launch_l1_stream(const int32_t* rows_ptr, const float* X, int in_pad, const int32_t* smap,
                             const int32_t* blk_rowptr, const int32_t* col, Split A, int fixed_k, cudaStream_t s) {
    constexpr int NB = 2;
    const int G = std::max(2, std::min(16, 155000 / (kL1Warps * NB * in_pad * 4)));
    const size_t smem = 128 + (size_t)kL1Warps * NB * G * in_pad * 4;
    static std::map<size_t, int> grids;
    static size_t attr_max = 0;   // only grows (see launch_l1_bulk)
    if (smem > attr_max) {
        cudaFuncSetAttribute(k_agg_l1_stream<NB, CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_max = smem;
    }
    int& grid = grids[smem];
    if (!grid) {
        cudaFuncSetAttribute(k_agg_l1_stream<NB, CPL>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        int per_sm = 0, dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_agg_l1_stream<NB, CPL>, kL1Warps * 32, smem);
        if (per_sm < 1) return false;
        grid = per_sm * sms;
    }
    launch_pdl(k_agg_l1_stream<NB, CPL>, grid, kL1Warps * 32, smem, s, rows_ptr, X, in_pad, smap, blk_rowptr, col, A,
               fixed_k, G);
    return true;
}

void launch_agg_sage(const int32_t* rows_ptr, FeatRows H, int in_pad, const int32_t* gmap,
                     const int32_t* smap, const int32_t* blk_rowptr, const int32_t* col, Split A, int fixed_k,
                     int k_max, cudaStream_t s) {
    // layer 1 of the neighbour sampler on a local table: rows staged by the bulk-copy engine
    // (GS_L1_BULK=0: register loads, for A/B; GS_L1_NB: buffers per warp)
    static const int bulk = [] { const char* e = std::getenv("GS_L1_BULK"); return e ? std::atoi(e) : 1; }();
    static const int nb = [] { const char* e = std::getenv("GS_L1_NB"); return e ? std::atoi(e) : 2; }();
    // GS_AGG_BULK_ALL=1 (A/B): the later layers' aggregations (local H rows, self row = i) too
    static const int bulk_all = [] { const char* e = std::getenv("GS_AGG_BULK_ALL"); return e ? std::atoi(e) : 0; }();
    // the row-gather variant (measured: products gather 49 -> 43 µs, 0.47 -> 0.53 of HBM; papers100M
    // rows of 512 B unchanged); GS_L1_G4=0: one bulk copy per row
    static const int g4 = [] { const char* e = std::getenv("GS_L1_G4"); return e ? std::atoi(e) : 1; }();
    // GS_AGG_G4=1 (A/B): the later layers' aggregations (local H rows, self row = i) by the row gather too
    static const int g4_all = [] { const char* e = std::getenv("GS_AGG_G4"); return e ? std::atoi(e) : 0; }();
    if (g4 && bulk && !H.shards && !gmap && (smap || g4_all) && k_max > 0 && k_max <= 31 && in_pad <= 256 &&
        (in_pad * 4) % 16 == 0) {
        // the tensor map of X (rows of in_pad floats, box {in_pad, 1}), one per table: keyed by base,
        // rows and width (a freed table's address can come back with another shape)
        static std::map<std::tuple<const float*, int64_t, int>, CUtensorMap> maps;
        const auto key = std::make_tuple(H.base, H.nrows, in_pad);
        auto it = maps.find(key);
        if (it == maps.end()) {
            CUtensorMap mp;
            if (H.nrows > 0 && make_tmap_rows_f32(&mp, H.base, H.nrows, in_pad)) it = maps.emplace(key, mp).first;
        }
        if (it != maps.end() &&
            launch_l1_bulk<2, true>(rows_ptr, H.base, in_pad, smap, blk_rowptr, col, A, fixed_k, 1 + k_max, s, &it->second))
            return;
    }
    if (bulk && !H.shards && !gmap && (smap || bulk_all) && k_max > 0 && k_max <= 31 && in_pad * 4 <= 1024) {
        const bool ok = nb == 3 ? launch_l1_bulk<3>(rows_ptr, H.base, in_pad, smap, blk_rowptr, col, A, fixed_k,
                                                     1 + k_max, s)
                                : launch_l1_bulk<2>(rows_ptr, H.base, in_pad, smap, blk_rowptr, col, A, fixed_k,
                                                     1 + k_max, s);
        if (ok) return;
    }
    // wider rows (> 1 KB): streamed in chunks (GS_L1_STREAM=0: register loads)
    static const int stream = [] { const char* e = std::getenv("GS_L1_STREAM"); return e ? std::atoi(e) : 1; }();
    if (stream && bulk && !H.shards && !gmap && (smap || bulk_all) && k_max > 0 && k_max <= 31 && in_pad * 4 > 1024) {
        bool ok = false;
        switch (cpl_of(in_pad)) {
            case 3: ok = launch_l1_stream<3>(rows_ptr, H.base, in_pad, smap, blk_rowptr, col, A, fixed_k, s); break;
            case 4: ok = launch_l1_stream<4>(rows_ptr, H.base, in_pad, smap, blk_rowptr, col, A, fixed_k, s); break;
            case 5: ok = launch_l1_stream<5>(rows_ptr, H.base, in_pad, smap, blk_rowptr, col, A, fixed_k, s); break;
            case 6: ok = launch_l1_stream<6>(rows_ptr, H.base, in_pad, smap, blk_rowptr, col, A, fixed_k, s); break;
            case 7: ok = launch_l1_stream<7>(rows_ptr, H.base, in_pad, smap, blk_rowptr, col, A, fixed_k, s); break;
            case 8: ok = launch_l1_stream<8>(rows_ptr, H.base, in_pad, smap, blk_rowptr, col, A, fixed_k, s); break;
            default: break;
        }
        if (ok) return;
    }
    // A/B diagnostic only: GS_AGG_DUMMY_SMEM = bytes of (unused) dynamic shared memory for the
    // register-load layer-1 gather (does a shared-memory footprint alone change the step?)
    static const int dummy = [] { const char* e = std::getenv("GS_AGG_DUMMY_SMEM"); return e ? std::atoi(e) : 0; }();
    if (dummy && k_max > 0 && !gmap && !H.shards && cpl_of(in_pad) == 1) {
        static bool set = false;
        if (!set) { cudaFuncSetAttribute(k_agg_sage<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dummy); set = true; }
        launch_pdl(k_agg_sage<1, false>, kWarpGrid, 256, (size_t)dummy, s, rows_ptr, H, in_pad, gmap, smap, blk_rowptr, col, A,
                   fixed_k);
        return;
    }
    GS_CPL_DISPATCH(cpl_of(in_pad), H, k_agg_sage, rows_ptr, H, in_pad, gmap, smap, blk_rowptr, col, A, fixed_k);
}

void launch_agg_gcn(const int32_t* rows_ptr, const int32_t* ndst_ptr, FeatRows H, int in_pad, int lda,
                    const int32_t* gmap, const int32_t* smap, const int32_t* blk_rowptr,
                    const int32_t* col, const int32_t* trowptr, Split A, cudaStream_t s) {
    GS_CPL_DISPATCH(cpl_of(in_pad), H, k_agg_gcn, rows_ptr, ndst_ptr, H, in_pad, lda, gmap, smap, blk_rowptr,
                    col, trowptr, A);
}

template <bool GCN>
static void spmm_bwd(int h, const StepState* st, const int32_t* dlim, const float* dA, int in_pad,
                     const int32_t* blk_rowptr, const int32_t* trowptr, const int32_t* tdst,
                     const uint32_t* hmask, int mask_ld, Split dPre_prev, cudaStream_t s) {
    switch (cpl_of(in_pad)) {
        case 1: launch_pdl(k_spmm_bwd<1, GCN>, kWarpGrid, 256, 0, s, h, st, dlim, dA, in_pad, blk_rowptr, trowptr, tdst, hmask, mask_ld, dPre_prev); break;
        case 2: launch_pdl(k_spmm_bwd<2, GCN>, kWarpGrid, 256, 0, s, h, st, dlim, dA, in_pad, blk_rowptr, trowptr, tdst, hmask, mask_ld, dPre_prev); break;
        case 3: launch_pdl(k_spmm_bwd<3, GCN>, kWarpGrid, 256, 0, s, h, st, dlim, dA, in_pad, blk_rowptr, trowptr, tdst, hmask, mask_ld, dPre_prev); break;
        default: launch_pdl(k_spmm_bwd<4, GCN>, kWarpGrid, 256, 0, s, h, st, dlim, dA, in_pad, blk_rowptr, trowptr, tdst, hmask, mask_ld, dPre_prev); break;
    }
}

void launch_spmm_bwd(bool gcn, int h, const StepState* st, const int32_t* dlim, const float* dA,
                     int in_pad, const int32_t* blk_rowptr, const int32_t* trowptr, const int32_t* tdst,
                     const uint32_t* hmask, int mask_ld, Split dPre_prev, cudaStream_t s) {
    if (gcn) spmm_bwd<true>(h, st, dlim, dA, in_pad, blk_rowptr, trowptr, tdst, hmask, mask_ld, dPre_prev, s);
    else spmm_bwd<false>(h, st, dlim, dA, in_pad, blk_rowptr, trowptr, tdst, hmask, mask_ld, dPre_prev, s);
}

int bal_units_cap() { return kBalUnits; }

static void launch_agg_bal_panel(const BalArgs& a, int mode, int nchp, cudaStream_t s) {
    const int cpl = (nchp + 31) / 32;
    const int c = cpl <= 1 ? 1 : cpl <= 2 ? 2 : cpl <= 4 ? 4 : 8;
#define GS_BAL(C, M) if (c == C && mode == M) {                                                  \
        if constexpr (M >= 2) launch_pdl(k_agg_bal_bwd<C, M>, kWarpGrid, 256, 0, s, a);            \
        else if (a.H.shards) launch_pdl(k_agg_bal<C, M, true>, kWarpGrid, 256, 0, s, a);           \
        else launch_pdl(k_agg_bal<C, M, false>, kWarpGrid, 256, 0, s, a);                          \
        return;                                                                                   \
    }
    GS_BAL(1, 0) GS_BAL(1, 1) GS_BAL(1, 2) GS_BAL(1, 3)
    GS_BAL(2, 0) GS_BAL(2, 1) GS_BAL(2, 2) GS_BAL(2, 3)
    GS_BAL(4, 0) GS_BAL(4, 1) GS_BAL(4, 2) GS_BAL(4, 3)
    GS_BAL(8, 0) GS_BAL(8, 1) GS_BAL(8, 2) GS_BAL(8, 3)
#undef GS_BAL
}

// Forward launches over wide rows are split into column panels (GS_BAL_PANEL_CH float4 chunks
// each; 0 = whole rows): the edge-wise row reads of a ShaDow block revisit every row many times,
// and a panel's working set (|S| x panel bytes) fits in L2 where whole rows do not.
void launch_agg_bal(const BalLaunch& b, cudaStream_t s) {
    BalArgs a{b.n_ptr, b.ndst_ptr, b.dlim_ptr, b.rowptr, b.col, b.orow, b.rmask, b.tag_ptr, b.H, b.gmap,
              b.dA, b.hmask, b.mask_ld, b.in_pad, b.out, b.out_w, b.part, b.cnt, 0, b.in_pad >> 2,
              b.rlist, b.brow, b.dmap};
    const int mode = (b.bwd ? 2 : 0) + (b.gcn ? 1 : 0);
    static const int pch = [] { const char* e = std::getenv("GS_BAL_PANEL_CH"); return e ? std::atoi(e) : 0; }();
    const int nch = b.in_pad >> 2;
    if (b.bwd || pch <= 0 || pch >= nch) {
        launch_agg_bal_panel(a, mode, nch, s);
        return;
    }
    for (int c0 = 0; c0 < nch; c0 += pch) {
        a.ch0 = c0;
        a.nchp = std::min(pch, nch - c0);
        launch_agg_bal_panel(a, mode, a.nchp, s);
    }
}

static size_t rf_scan_bytes(int cap) {
    size_t b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b, (const int32_t*)nullptr, (int32_t*)nullptr, cap);
    return b;
}
size_t rf_compact_scratch_bytes(int cap) { return 7 * ((size_t)cap * 4 + 256) + rf_scan_bytes(cap) + 256; }

void launch_rf_compact(const uint32_t* mask, const uint32_t* tag_ptr, int cap, const int32_t* rowptr,
                       const int32_t* deg_rowptr, void* scratch, int32_t* rf_list, int32_t* rf_pos, int32_t* sub_rowptr,
                       int32_t* sub_rowptr_t, int32_t* n_rf, cudaStream_t s) {
    char* p = static_cast<char*>(scratch);
    auto take = [&](size_t bytes) { char* q = p; p += (bytes + 255) & ~size_t(255); return q; };
    int32_t* flags = reinterpret_cast<int32_t*>(take(4 * (size_t)cap));
    int32_t* degf = reinterpret_cast<int32_t*>(take(4 * (size_t)cap));
    int32_t* degt = reinterpret_cast<int32_t*>(take(4 * (size_t)cap));
    int32_t* pos = reinterpret_cast<int32_t*>(take(4 * (size_t)cap));
    int32_t* scf = reinterpret_cast<int32_t*>(take(4 * (size_t)cap));
    int32_t* sct = reinterpret_cast<int32_t*>(take(4 * (size_t)cap));
    size_t tb = rf_scan_bytes(cap);
    void* tmp = take(tb);
    const bool two = sub_rowptr_t != sub_rowptr;
    launch_pdl(k_rf_prep, 148 * 4, 256, 0, s, mask, tag_ptr, cap, rowptr, two ? deg_rowptr : rowptr, flags, degf, degt);
    cub::DeviceScan::ExclusiveSum(tmp, tb, flags, pos, cap, s);
    cub::DeviceScan::ExclusiveSum(tmp, tb, degf, scf, cap, s);
    if (two) cub::DeviceScan::ExclusiveSum(tmp, tb, degt, sct, cap, s);
    launch_pdl(k_rf_scatter, 148 * 4, 256, 0, s, cap, flags, degf, degt, pos, scf, sct, rf_list, rf_pos, sub_rowptr,
               sub_rowptr_t, n_rf);
}

void launch_rf_mark(const int32_t* nseed_ptr, const int32_t* rowptr, const int32_t* col, const uint32_t* tag_ptr,
                    uint32_t* mask, cudaStream_t s) {
    launch_pdl(k_rf_mark, 148 * 4, 256, 0, s, nseed_ptr, rowptr, col, tag_ptr, mask);
}

void launch_wgrad_reduce(const PackAll& p, int l0, int l1, float* grads, const PeerX& x, cudaStream_t s) {
    launch_pdl(k_wgrad_reduce, 148 * 4, 256, 0, s, p, l0, l1, grads, x);
}

void launch_sgd_pack(const PackAll& p, float* params, float* grads, float lr, bool reduce, const OptState& o,
                     cudaStream_t s, const PeerX& x) {
    launch_pdl(k_sgd_pack, reduce ? 148 * 8 : 148 * 2, 256, 0, s, p, params, grads, lr, reduce ? 1 : 0, o, x);
}

// ------------------------------------------------------------------ the last layer, fused
// The last layer of a model with C <= 64 classes, one warp per output row, on the CUDA cores in
// fp32: Z = A W (logits; Eq. 1-2), the softmax cross-entropy of the row (Eq. 3, R15: l = max + log
// Σ exp(z - max) - z_y, dZ = (softmax - onehot) / b_total), and dA = dZ W^T — every quantity of
// the row is local to it, so the three products of the layer share one pass over W, which sits
// in shared memory (k_pad x C fp32, row stride C|1 so both the k-major and the c-major sweeps are
// bank-conflict free).  At M = 1024 rows the tensor-core GEMM + CE epilogue was latency-bound
// (18 µs for 0.15 GFLOP, tensor pipe 9 % active) and its dgrad GEMM another 8 µs; here the layer
// is ~1 wave of 128 blocks.  The weight gradient A^T dZ stays on the tensor cores (forked stream).
// A is read from its split planes (hi + lo); W from the fp32 parameters (rows r of the [rows x C]
// block: SAGE k -> (k / in_pad) * in + k % in_pad, GCN k -> k, zero beyond).
constexpr int kLastRows = 8;    // rows per block
constexpr int kLastSplit = 2;   // warps per row (512 threads: a block fits beside a sampling block, 16K registers each)
struct LastArgs {
    const int32_t* m_ptr;      // rows of the layer (batch rows)
    Split A;                   // operand planes [rows x k_pad]
    int k_pad, in, in_pad, sage;
    const float* W;            // the layer's fp32 parameter block [rows x C]
    int C, n_pad;
    float* Z;                  // logits [rows x n_pad] (debug readout)
    Split dz;                  // dZ planes [rows x n_pad] for the weight-gradient GEMM
    float* dA;                 // [rows x k_pad] fp32 for the backward aggregation
    StepState* st;
    const int32_t* labels;
    const int32_t* nodes;
    // SAGE + neighbour sampler: the layer's aggregation too (Hp = H_{L-1} [rows x in_pad] fp32,
    // rowptr/col = the block of hop 0 over local ids): A = [H_self | mean] is gathered here, as
    // k_agg_sage computes it (CSR-order adds, times 1/deg), and written to A's planes for the
    // weight-gradient GEMM; null Hp: A is read from its planes
    const float* Hp;
    const int32_t* rowptr;
    const int32_t* col;
};
__global__ void __launch_bounds__(kLastRows * 32 * kLastSplit) k_last_layer(LastArgs a) {
    // kLastSplit warps per row: warp q (= warp / kLastRows) takes the q-th part of the k range of
    // the logits and of dA; the parts' logits are added in a fixed order (part 0 + 1 + ...)
    extern __shared__ __align__(128) float lsm[];
    // W's k rows are the parameter rows themselves when in == in_pad (hidden layers): one bulk copy
    // of the contiguous [k_pad x C] block (row stride C; odd C keeps both sweeps conflict-free)
    const bool bulk = a.in == a.in_pad && ((a.k_pad * a.C) & 3) == 0 && (reinterpret_cast<uintptr_t>(a.W) & 15) == 0;
    const int ldw = bulk ? a.C : (a.C | 1);
    float* Ws = lsm + 32;                               // [k_pad][ldw] (lsm[0..1]: the mbarrier)
    float* As = Ws + (((size_t)a.k_pad * ldw + 3) & ~size_t(3));   // [kLastRows][k_pad]
    __shared__ float zpart[kLastSplit][kLastRows][64];
    __shared__ float dzs[kLastRows][64];
    __shared__ float wloss[kLastRows];
    __shared__ int is_last;
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int rl = warp % kLastRows, half = warp / kLastRows;
    uint64_t* wbar = reinterpret_cast<uint64_t*>(lsm);
    if (bulk) {
        if (threadIdx.x == 0) {
            mbar_init(wbar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            fence_async_smem();
            const uint32_t bytes = (uint32_t)(a.k_pad * a.C) * 4u;
            mbar_expect_tx(wbar, bytes);
            for (uint32_t o = 0; o < bytes; o += 65536u)   // bulk copies of up to 64 KB
                bulk_g2s(reinterpret_cast<char*>(Ws) + o, reinterpret_cast<const char*>(a.W) + o,
                         min(65536u, bytes - o), wbar, policy_evict_last());
        }
    } else
    // W -> shared memory by asynchronous 4-byte copies, a warp per k row (its parameter row
    // computed once), lanes over the classes; independent of the predecessor kernel
    for (int k = warp; k < a.k_pad; k += kLastSplit * kLastRows) {
        int r = -1;
        if (a.sage) {
            const int hh = k >= a.in_pad ? 1 : 0, j = k - hh * a.in_pad;
            if (j < a.in) r = hh * a.in + j;
        } else if (k < a.in) {
            r = k;
        }
        for (int c = lane; c < a.C; c += 32) {
            if (r >= 0)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(Ws + k * ldw + c)),
                             "l"(a.W + (int64_t)r * a.C + c) : "memory");
            else
                Ws[k * ldw + c] = 0.f;
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    pdl_trigger();
    pdl_wait();
    const int M = *a.m_ptr;
    const int row = blockIdx.x * kLastRows + rl;
    if (bulk) { __syncthreads(); mbar_wait(wbar, 0); }   // (the barrier is initialised before it is polled)
    float* Ar = As + (size_t)rl * a.k_pad;
    if (a.Hp) {
        if (row < M) {
            const int beg = a.rowptr[row], end = a.rowptr[row + 1];
            const float inv = end > beg ? 1.0f / (float)(end - beg) : 0.f;   // one division per row (R23)
            const int nch = a.in_pad >> 2;
            const float4* H4 = reinterpret_cast<const float4*>(a.Hp);
            for (int ch = lane + 32 * half; ch < nch; ch += 32 * kLastSplit) {   // 16-byte chunks; adds in CSR order
                const float4 sv = H4[(int64_t)row * nch + ch];
                float4 acc = kZero4;
                for (int e = beg; e < end; ++e) acc = f4add(acc, H4[(int64_t)__ldg(a.col + e) * nch + ch]);
                const float4 mv = f4scale(acc, inv);
                *reinterpret_cast<float4*>(Ar + 4 * ch) = sv;
                *reinterpret_cast<float4*>(Ar + a.in_pad + 4 * ch) = mv;
                store_split4(a.A, tix(a.A, row, 4 * ch), sv);
                store_split4(a.A, tix(a.A, row, a.in_pad + 4 * ch), mv);
            }
        } else if (row < ((M + 63) & ~63)) {   // zero tail rows of the operand planes
            for (int k = lane + 32 * half; k < a.k_pad; k += 32 * kLastSplit) store_split1(a.A, tix(a.A, row, k), 0.f);
        }
    } else if (row < M) {
        for (int k = lane + 32 * half; k < a.k_pad; k += 32 * kLastSplit) {
            const int64_t ix = tix(a.A, row, k);
            Ar[k] = __bfloat162float(a.A.hi[ix]) + (a.A.lo ? __bfloat162float(a.A.lo[ix]) : 0.f);
        }
    }
    __syncthreads();
    const int K2 = a.k_pad / kLastSplit;   // k_pad is a multiple of 4 * kLastSplit
    const int kb = half * K2;
    const int c0 = lane, c1 = lane + 32;
    const bool v0 = c0 < a.C, v1 = c1 < a.C;
    float z0 = 0.f, z1 = 0.f;
    if (row < M) {
        // this half's logits: four partial sums per class (k mod 4, k ascending), fixed-order total
        float p0[4] = {0.f, 0.f, 0.f, 0.f}, p1[4] = {0.f, 0.f, 0.f, 0.f};
        const float* w0 = Ws + (v0 ? c0 : 0);
        const float* w1 = Ws + (v1 ? c1 : 0);
#pragma unroll 2
        for (int k = kb; k < kb + K2; k += 4) {
            const float4 x = *reinterpret_cast<const float4*>(Ar + k);
            p0[0] = fmaf(x.x, w0[(k + 0) * ldw], p0[0]); p1[0] = fmaf(x.x, w1[(k + 0) * ldw], p1[0]);
            p0[1] = fmaf(x.y, w0[(k + 1) * ldw], p0[1]); p1[1] = fmaf(x.y, w1[(k + 1) * ldw], p1[1]);
            p0[2] = fmaf(x.z, w0[(k + 2) * ldw], p0[2]); p1[2] = fmaf(x.z, w1[(k + 2) * ldw], p1[2]);
            p0[3] = fmaf(x.w, w0[(k + 3) * ldw], p0[3]); p1[3] = fmaf(x.w, w1[(k + 3) * ldw], p1[3]);
        }
        z0 = (p0[0] + p0[1]) + (p0[2] + p0[3]);
        z1 = (p1[0] + p1[1]) + (p1[2] + p1[3]);
        zpart[half][rl][c0] = z0;
        zpart[half][rl][c1] = z1;
    }
    __syncthreads();
    float l = 0.f;
    if (row < M && half == 0) {
        float t0 = zpart[0][rl][c0], t1 = zpart[0][rl][c1];
#pragma unroll
        for (int q = 1; q < kLastSplit; ++q) { t0 += zpart[q][rl][c0]; t1 += zpart[q][rl][c1]; }
        z0 = v0 ? t0 : 0.f;
        z1 = v1 ? t1 : 0.f;
        if (v0) a.Z[(int64_t)row * a.n_pad + c0] = z0;
        if (v1) a.Z[(int64_t)row * a.n_pad + c1] = z1;
        // softmax cross-entropy of the row
        float mx = fmaxf(v0 ? z0 : -INFINITY, v1 ? z1 : -INFINITY);
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
        const float e0 = v0 ? expf(z0 - mx) : 0.f, e1 = v1 ? expf(z1 - mx) : 0.f;
        float ssum = e0 + e1;
        for (int o = 16; o; o >>= 1) ssum += __shfl_xor_sync(kFull, ssum, o);
        const int y = a.labels[a.nodes[row]];
        const float zy = __shfl_sync(kFull, y < 32 ? z0 : z1, y & 31);
        l = (mx + logf(ssum)) - zy;
        const float inv_s = 1.0f / ssum, inv_bt = 1.0f / (float)max(a.st->b_total, 1);
        const float d0 = v0 ? (e0 * inv_s - (c0 == y ? 1.f : 0.f)) * inv_bt : 0.f;
        const float d1 = v1 ? (e1 * inv_s - (c1 == y ? 1.f : 0.f)) * inv_bt : 0.f;
        dzs[rl][c0] = d0;
        dzs[rl][c1] = d1;
        if (c0 < a.n_pad) store_split1(a.dz, tix(a.dz, row, c0), d0);
        if (c1 < a.n_pad) store_split1(a.dz, tix(a.dz, row, c1), d1);
    } else if (half == 0 && row >= M && row < ((M + 63) & ~63)) {   // zero tail rows of the dZ planes
        for (int c = lane; c < a.n_pad; c += 32) store_split1(a.dz, tix(a.dz, row, c), 0.f);
    }
    __syncthreads();
    if (row < M) {
        // dA[row, k] = Σ_c dZ[row, c] W[k, c]  (c ascending), this half's k = kb + lane + 32 j
        for (int k0 = kb; k0 < kb + K2; k0 += 32 * 8) {
            float acc[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = 0.f;
            for (int c = 0; c < a.C; ++c) {
                const float dc = dzs[rl][c];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int k = k0 + lane + 32 * j;
                    if (k < kb + K2) acc[j] = fmaf(dc, Ws[k * ldw + c], acc[j]);
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int k = k0 + lane + 32 * j;
                if (k < kb + K2) a.dA[(int64_t)row * a.k_pad + k] = acc[j];
            }
        }
    }
    // the loss: the block's rows in order, then the blocks in order by the last block to finish
    if (lane == 0 && half == 0) wloss[rl] = l;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < kLastRows; ++w) t += wloss[w];
        a.st->row_loss[blockIdx.x] = t;
        __threadfence();
        is_last = atomicAdd(&a.st->ce_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (is_last && threadIdx.x == 0) {
        __threadfence();
        float tot = 0.f;
        for (int b = 0; b < (int)gridDim.x; ++b) tot += __ldcg(&a.st->row_loss[b]);
        a.st->loss = tot * (1.0f / (float)max(a.st->b_total, 1));
        a.st->ce_done = 0u;
    }
}

void launch_last_layer(const int32_t* m_ptr, int m_cap, Split A, int k_pad, int in, int in_pad, bool sage,
                       const float* W, int C, int n_pad, float* Z, Split dz, float* dA, StepState* st,
                       const int32_t* labels, const int32_t* nodes, const float* Hp, const int32_t* rowptr,
                       const int32_t* col, cudaStream_t s) {
    const size_t smem = sizeof(float) * (32 + (((size_t)k_pad * (C | 1) + 3) & ~size_t(3)) + (size_t)kLastRows * k_pad);
    static size_t attr = 0;
    if (smem > attr) {
        cudaFuncSetAttribute(k_last_layer, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = smem;
    }
    const int grid = (((m_cap + 63) & ~63) + kLastRows - 1) / kLastRows;
    LastArgs a{m_ptr, A, k_pad, in, in_pad, sage ? 1 : 0, W, C, n_pad, Z, dz, dA, st, labels, nodes, Hp, rowptr, col};
    launch_pdl(k_last_layer, grid, kLastRows * 32 * kLastSplit, smem, s, a);
}

bool last_layer_fits(int k_pad, int C) {
    return C <= 64 && k_pad % (4 * kLastSplit) == 0 &&
           sizeof(float) * (32 + (size_t)k_pad * (C | 1) + 4 + (size_t)kLastRows * k_pad) <= 200 * 1024;
}

void launch_ce(StepState* st, const float* Z, int ldz, int C, const int32_t* labels, const int32_t* nodes,
               Split dZ, cudaStream_t s) {
    launch_pdl(k_ce, 128, 256, 0, s, st, Z, ldz, C, labels, nodes, dZ, st->row_loss, &st->ce_done);
}

void launch_init_params(float* p, int64_t cnt, float bound, uint64_t seed, uint32_t layer, cudaStream_t s) {
    const int blocks = (int)std::min<int64_t>((cnt + 255) / 256, 148 * 4);
    k_init<<<blocks, 256, 0, s>>>(p, cnt, bound, seed, layer);
}

}  // namespace gs
