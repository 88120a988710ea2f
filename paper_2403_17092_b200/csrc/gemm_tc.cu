// Dense update GEMMs of the step on the 5th-generation tensor cores (sm_100a):
// TMA (cp.async.bulk.tensor, 128B swizzle) -> shared memory -> tcgen05.mma (kind::f16, bf16
// operands, fp32 accumulator in TMEM) -> tcgen05.ld -> fp32 epilogue (+ReLU).
//
// fp32 parity (north_star: 1e-4) uses a 3-term bf16 split: x = x_hi + x_lo with
// x_hi = bf16(x), x_lo = bf16(x - x_hi); D = A_hi B_hi + A_hi B_lo + A_lo B_hi accumulated in
// fp32 (relative error ~ 2^-16 per product).  The bf16 variant
// (GNN_BF16_GEMM) issues the A_hi B_hi term only.
//
// Three uses:
//   fwd   Pre = A W         A: [M x K] K-major,   B = W^T [N x K] K-major      (+ReLU)
//   dgrad dA  = dPre W^T    A: [M x N] K-major,   B = W   [K x N] K-major
//   wgrad dW  = A^T dPre    A^T: MN-major,        B = dPre MN-major, split over M (deterministic)
//
// Persistent: one CTA per SM walks a static tile list (t = blockIdx + j * gridDim), or (A/B switch
// GS_GEMM_DYN=1, measured slower) tiles handed out dynamically by an atomic tile counter per launch
// site (GemmArgs::sched), so that a CTA that starts late, because another kernel still holds its
// SM, takes fewer tiles instead of holding a fixed share of them.  Warp 0 = TMA producer and tile scheduler (it publishes each tile index in a
// 4-slot shared ring read by the MMA warp and the 4 epilogue warps), warp 1 = TMEM allocator +
// MMA issuer, warps 2..5 = epilogue (one TMEM lane quarter each).  Two TMEM accumulators: the
// epilogue of tile j overlaps the MMAs of tile j+1.  Every tile's result is independent of
// which CTA computes it (split-K partials go to per-split slots, the CE loss to per-tile
// partials), so the output is bit-identical under any schedule.
#include <cuda.h>
#include <cstdlib>
#include <cuda_bf16.h>

#include "kernels.h"
#include "tma.cuh"

#ifndef GS_TC_STAGES_WIDE
#define GS_TC_STAGES_WIDE 3   // pipeline stages of the 96/128-column tiles
#endif
#ifndef GS_TC_STAGES_NARROW
#define GS_TC_STAGES_NARROW 4   // pipeline stages of the <= 64-column tiles
#endif

namespace gs {
namespace {

constexpr int kBM = 128;     // UMMA M (cta_group::1)
constexpr int kBK = 64;      // bf16 elements per 128-byte swizzle row
constexpr int kThreads = 192;

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

// TMA store of a swizzled shared-memory box (bulk-group completion); C maps are always 3-D.
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// 32 consecutive TMEM columns of this warp's lane quarter (thread = lane = row).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}

// Shared-memory matrix descriptor (tcgen05 "matrix descriptor"): start>>4 [0,14),
// LBO>>4 [16,30), SBO>>4 [32,46), version 1 [46,48), layout SWIZZLE_128B (2) [61,64).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// Instruction descriptor, kind::f16: D f32, A/B bf16, majors, N>>3, M>>4.
template <int BN, bool A_MN, bool B_MN>
__host__ __device__ constexpr uint32_t idesc() {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((A_MN ? 1u : 0u) << 15) | ((B_MN ? 1u : 0u) << 16) |
           ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}

template <int BN>
struct TileCfg {
    static constexpr int kAStage = kBM * kBK * 2;                    // 16 KB per plane
    static constexpr int kBStage = ((BN + 63) / 64) * 64 * kBK * 2;  // whole 64-wide boxes (MN-major)
    static constexpr int kAccCols = BN <= 32 ? 32 : BN <= 64 ? 64 : 128;      // one accumulator
    static constexpr int kTmemCols = 2 * kAccCols;                            // double buffered
    // bytes one stage's TMA boxes deliver (OOB parts are zero-filled but still counted)
    static constexpr int kBBytesK = BN * kBK * 2;                     // K-major: box {64, BN}
    static constexpr int kBBytesMN = ((BN + 63) / 64) * 64 * kBK * 2; // MN-major: boxes {64, 64}
};

constexpr int kEpiCols = 32;                          // epilogue chunk: 32 fp32 = one 128 B swizzle row
constexpr int kEpiBuf = 32 * kEpiCols * 4;           // one warp's 32-row chunk (4 KB)
constexpr int kEpiBytes = 4 * 2 * kEpiBuf;           // 4 epilogue warps x double buffer

struct GemmArgs {
    const int32_t* m_ptr;   // fwd/dgrad: rows of C (dynamic); wgrad: reduction length (dynamic)
    int m_static;           // wgrad: rows of C
    int m_tiles_cap;        // fwd/dgrad: tile rows of the worst case
    int n_tiles;
    int splits;             // wgrad
    int k_blocks;           // fwd/dgrad: reduction in 64-blocks (static)
    int k_len;              // fwd/dgrad: reduction length (the last block's k16 steps past it are skipped)
    int n_store;            // columns of C to store
    float* C;
    int ldc;
    int relu;
    int64_t split_stride;   // wgrad: C + z * split_stride
    // MODE 3 (last layer, fwd + softmax cross-entropy): rows of C are logits
    StepState* st;
    const int32_t* labels;
    const int32_t* nodes;
    Split dz;               // dZ planes [rows x ldc]
    int classes;
    uint32_t* mask;         // MODE 2 with relu: sign bits of the stored H (nullable)
    int mask_ld;
    int diag;               // profiling diagnostics only (env GS_GEMM_DIAG): 1 skip C stores, 2 skip MMAs, 4 skip loads, 8 skip the CE epilogue, 16 skip the loss sum
    int* sched;             // {next tile, CTAs done}: the dynamic tile scheduler (null: static tiles)
    int clc;                // 1: one CTA per tile, idle CTAs steal pending CTAs' tiles (cluster launch control)
};
constexpr int kTileRing = 4;   // tile indices the scheduler may publish ahead of the epilogue

struct TileInfo { int tm, tn, z, kb0, nkb; };

template <int MODE>
__device__ __forceinline__ TileInfo tile_info(const GemmArgs& a, int t, int M) {
    TileInfo ti;
    if (MODE != 1) {
        ti.tm = t / a.n_tiles;
        ti.tn = t % a.n_tiles;
        ti.z = 0;
        ti.kb0 = 0;
        ti.nkb = a.k_blocks;
    } else {
        const int mt = (a.m_static + kBM - 1) / kBM;
        const int per_z = mt * a.n_tiles;
        ti.z = t / per_z;
        const int r = t % per_z;
        ti.tm = r / a.n_tiles;
        ti.tn = r % a.n_tiles;
        const int nkb_all = (M + kBK - 1) / kBK;
        const int per = (nkb_all + a.splits - 1) / a.splits;
        ti.kb0 = min(nkb_all, ti.z * per);
        ti.nkb = min(nkb_all, ti.kb0 + per) - ti.kb0;
    }
    return ti;
}

// Softmax cross-entropy of one logits row held by this thread (zr: fp32 bits, columns >= C
// ignored) (R15): l = max + log sum exp(z - max) - z_y;  dZ = (softmax - onehot) /
// b_total as split planes; rows in [M, round64(M)) get zero dZ (the wgrad reduction pads to 64).
// Returns the row's loss (0 outside [0, M)).
template <int BN>
__device__ __forceinline__ float ce_rows(const GemmArgs& args, uint32_t (&zr)[(BN + 31) / 32][32], int row, int M) {
    constexpr int kZ = (BN + 31) / 32 * 32;
    const int C = args.classes;
    const float inv_bt = 1.0f / (float)max(args.st->b_total, 1);
    if (row < M) {
        const int y = args.labels[args.nodes[row]];
        float mx = -INFINITY, zy = 0.f;
#pragma unroll
        for (int c = 0; c < kZ; ++c) {
            const float z = __uint_as_float(zr[c >> 5][c & 31]);
            if (c < C) mx = fmaxf(mx, z);
            if (c == y) zy = z;
        }
        float s = 0.f;
#pragma unroll
        for (int c = 0; c < kZ; ++c) {   // e_c = exp(z_c - max) kept in place
            const float e = c < C ? expf(__uint_as_float(zr[c >> 5][c & 31]) - mx) : 0.f;
            zr[c >> 5][c & 31] = __float_as_uint(e);
            s += e;
        }
        const float inv_s = 1.0f / s;
#pragma unroll
        for (int c = 0; c < BN; c += 8) {   // dZ = (e/s - onehot)/b_total, 16-byte stores
            uint32_t hw[4], lw[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int c0 = c + 2 * q, c1 = c0 + 1;
                const float d0 = c0 < C ? (__uint_as_float(zr[c0 >> 5][c0 & 31]) * inv_s - (c0 == y ? 1.f : 0.f)) * inv_bt : 0.f;
                const float d1 = c1 < C ? (__uint_as_float(zr[c1 >> 5][c1 & 31]) * inv_s - (c1 == y ? 1.f : 0.f)) * inv_bt : 0.f;
                const __nv_bfloat162 hi = __floats2bfloat162_rn(d0, d1);
                const __nv_bfloat162 lo = __floats2bfloat162_rn(d0 - __low2float(hi), d1 - __high2float(hi));
                hw[q] = *reinterpret_cast<const uint32_t*>(&hi);
                lw[q] = *reinterpret_cast<const uint32_t*>(&lo);
            }
            *reinterpret_cast<uint4*>(args.dz.hi + tix(args.dz, row, c)) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            if (args.dz.lo) *reinterpret_cast<uint4*>(args.dz.lo + tix(args.dz, row, c)) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
        return (mx + logf(s)) - zy;
    } else if (row < ((M + 63) & ~63)) {      // zero tail rows of the dZ planes
#pragma unroll
        for (int c = 0; c < BN; c += 8) {
            *reinterpret_cast<uint4*>(args.dz.hi + tix(args.dz, row, c)) = make_uint4(0u, 0u, 0u, 0u);
            if (args.dz.lo) *reinterpret_cast<uint4*>(args.dz.lo + tix(args.dz, row, c)) = make_uint4(0u, 0u, 0u, 0u);
        }
    }
    return 0.f;
}

// MODE 0 = dgrad (A, B K-major), MODE 1 = wgrad (A, B MN-major, split z), MODE 2 = fwd (A K-major,
// B MN-major: W read as stored, [K x N]), MODE 3 = fwd of the last layer with the softmax
// cross-entropy in the epilogue (a thread holds a whole logits row: BN = n_pad <= 64).
template <int BN, int STAGES, int TERMS, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
k_gemm_tc(const __grid_constant__ CUtensorMap mA_hi, const __grid_constant__ CUtensorMap mA_lo,
          const __grid_constant__ CUtensorMap mB_hi, const __grid_constant__ CUtensorMap mB_lo,
          const __grid_constant__ CUtensorMap mC, GemmArgs args) {
    using Cfg = TileCfg<BN>;
    constexpr bool A_MN = MODE == 1;          // wgrad: A^T read from row-major A
    constexpr bool B_MN = MODE >= 1;          // wgrad (dPre), fwd mode 2 (W [K x N])
    constexpr int kAPlanes = TERMS == 3 ? 2 : 1;
    constexpr int kStageBytes = kAPlanes * (Cfg::kAStage + Cfg::kBStage);
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full_bar[STAGES], empty_bar[STAGES], tfull[2], tempty[2];
    __shared__ uint64_t ring_full[kTileRing], ring_empty[kTileRing];
    __shared__ int ring_tile[kTileRing];
    __shared__ __align__(16) uint4 clc_resp;   // the try_cancel response (16 bytes)
    __shared__ uint64_t clc_bar;
    __shared__ uint32_t tmem_base_sh;
    __shared__ int ce_last;
    __shared__ float ce_warp[2][4];   // MODE 3: per-tile sums of the 4 epilogue warps (double buffered)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    pdl_trigger();
    if (threadIdx.x == 0) {
        for (const CUtensorMap* mp : {&mA_hi, &mA_lo, &mB_hi, &mB_lo, &mC})
            asm volatile("prefetch.tensormap [%0];" ::"l"(mp) : "memory");
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
        for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 4); }
        for (int r = 0; r < kTileRing; ++r) { mbar_init(&ring_full[r], 1); mbar_init(&ring_empty[r], 5); }
        mbar_init(&clc_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(Cfg::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    // everything above is independent of the predecessor kernel (programmatic launch)
    pdl_wait();
    const int M = *args.m_ptr;
    const int ntiles = MODE != 1 ? ((M + kBM - 1) / kBM) * args.n_tiles
                                 : ((args.m_static + kBM - 1) / kBM) * args.n_tiles * args.splits;
    const int t_first = (int)blockIdx.x, t_step = (int)gridDim.x;
    // the j-th tile of this CTA: published by the producer (dynamic) or blockIdx + j * gridDim
    const bool dyn = args.sched != nullptr || args.clc;
    auto next_tile = [&](int j) -> int {   // consumers (MMA thread, epilogue warps)
        if (!dyn) return t_first + j * t_step;
        const int r = j % kTileRing;
        mbar_wait(&ring_full[r], (j / kTileRing) & 1);
        const int t = ring_tile[r];
        return t;
    };
    auto release_tile = [&](int j) {      // one arrival per consumer (MMA thread, 4 epilogue lane-0s)
        if (dyn) mbar_arrive(&ring_empty[j % kTileRing]);
    };

    if (warp == 0) {
        // ================= TMA producer
        if (lane == 0) {
            int it = 0;
            int clc_t = (int)blockIdx.x;      // CLC: this CTA's own tile first, then stolen ones
            uint32_t clc_phase = 0;
            for (int jt = 0;; ++jt) {
                int t;
                if (args.clc) {   // publish the tile; ask for a pending CTA's tile while this one loads
                    const int r = jt % kTileRing;
                    if (jt >= kTileRing) mbar_wait(&ring_empty[r], ((jt / kTileRing) - 1) & 1);
                    t = clc_t;
                    const bool valid = t >= 0 && t < ntiles;
                    ring_tile[r] = valid ? t : -1;
                    mbar_arrive(&ring_full[r]);
                    if (!valid) break;
                    mbar_expect_tx(&clc_bar, 16u);
                    asm volatile("clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];"
                                 ::"r"(smem_u32(&clc_resp)), "r"(smem_u32(&clc_bar)) : "memory");
                } else if (dyn) {   // claim a tile and publish it to the consumers
                    const int r = jt % kTileRing;
                    if (jt >= kTileRing) mbar_wait(&ring_empty[r], ((jt / kTileRing) - 1) & 1);
                    t = atomicAdd(args.sched, 1);
                    ring_tile[r] = t < ntiles ? t : -1;
                    mbar_arrive(&ring_full[r]);   // (release: orders the ring write)
                    if (t >= ntiles) break;
                } else {
                    t = t_first + jt * t_step;
                    if (t >= ntiles) break;
                }
                const TileInfo ti = tile_info<MODE>(args, t, M);
                const int tile_m = ti.tm * kBM, tile_n = ti.tn * BN;
                for (int kb = 0; kb < ti.nkb; ++kb, ++it) {
                    const int s = it % STAGES;
                    if (it >= STAGES) mbar_wait(&empty_bar[s], ((it / STAGES) - 1) & 1);
                    uint8_t* st = smem + s * kStageBytes;
                    uint8_t* a_hi = st;
                    uint8_t* b_hi = st + Cfg::kAStage;
                    uint8_t* a_lo = st + Cfg::kAStage + Cfg::kBStage;
                    uint8_t* b_lo = a_lo + Cfg::kAStage;
                    if (args.diag & 4) { mbar_arrive(&full_bar[s]); continue; }   // diagnostics: no loads
                    mbar_expect_tx(&full_bar[s], kAPlanes * (Cfg::kAStage + (B_MN ? Cfg::kBBytesMN : Cfg::kBBytesK)));
                    const int k0 = (ti.kb0 + kb) * kBK;
                    // A planes are k-block-tiled (3-D maps {64, rows, k-block}): every box is one
                    // contiguous block of HBM
                    if (!A_MN) {          // K-major: box {64 (k), 128 rows} of k-block k0/64
                        tma_load_3d(a_hi, &mA_hi, &full_bar[s], 0, tile_m, k0 >> 6);
                        if (TERMS == 3) tma_load_3d(a_lo, &mA_lo, &full_bar[s], 0, tile_m, k0 >> 6);
                    } else {              // MN-major: boxes {64 (m), 64 (k rows)}, 8 KB apart
#pragma unroll
                        for (int j = 0; j < kBM / 64; ++j) {
                            tma_load_3d(a_hi + j * 8192, &mA_hi, &full_bar[s], 0, k0, (tile_m >> 6) + j);
                            if (TERMS == 3) tma_load_3d(a_lo + j * 8192, &mA_lo, &full_bar[s], 0, k0, (tile_m >> 6) + j);
                        }
                    }
                    if (!B_MN) {
                        tma_load_2d(b_hi, &mB_hi, &full_bar[s], k0, tile_n);
                        if (TERMS == 3) tma_load_2d(b_lo, &mB_lo, &full_bar[s], k0, tile_n);
                    } else if (MODE == 1) {   // dPre planes (tiled), MN-major
#pragma unroll
                        for (int j = 0; j < (BN + 63) / 64; ++j) {
                            tma_load_3d(b_hi + j * 8192, &mB_hi, &full_bar[s], 0, k0, (tile_n >> 6) + j);
                            if (TERMS == 3) tma_load_3d(b_lo + j * 8192, &mB_lo, &full_bar[s], 0, k0, (tile_n >> 6) + j);
                        }
                    } else {                  // W [K x N] as stored, MN-major
#pragma unroll
                        for (int j = 0; j < (BN + 63) / 64; ++j) {
                            tma_load_2d(b_hi + j * 8192, &mB_hi, &full_bar[s], tile_n + 64 * j, k0);
                            if (TERMS == 3) tma_load_2d(b_lo + j * 8192, &mB_lo, &full_bar[s], tile_n + 64 * j, k0);
                        }
                    }
                }
                if (args.clc) {   // the stolen CTA's index is the next tile (none left: stop)
                    mbar_wait(&clc_bar, clc_phase);
                    clc_phase ^= 1u;
                    uint32_t cx = 0, ok = 0;
                    asm volatile(
                        "{\n\t.reg .pred p1;\n\t.reg .b128 r;\n\t"
                        "ld.shared.b128 r, [%2];\n\t"
                        "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p1, r;\n\t"
                        "selp.u32 %1, 1, 0, p1;\n\t"
                        "@p1 clusterlaunchcontrol.query_cancel.get_first_ctaid.v4.b32.b128 {%0, _, _, _}, r;\n\t}"
                        : "=r"(cx), "=r"(ok) : "r"(smem_u32(&clc_resp)) : "memory");
                    clc_t = ok ? (int)cx : -1;
                }
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer (one thread)
        if (lane == 0) {
            constexpr uint32_t id = idesc<BN, A_MN, B_MN>();
            // reduction extent: operands are zero past it, so the k16 steps beyond it are skipped
            const int klen = MODE == 1 ? M : args.k_len;
            int it = 0, j = 0;
            for (int jt = 0;; ++jt) {
                const int t = next_tile(jt);
                release_tile(jt);
                if (t < 0 || t >= ntiles) break;
                const TileInfo ti = tile_info<MODE>(args, t, M);
                if (ti.nkb == 0) continue;
                const int acc = j & 1;
                if (j >= 2) { mbar_wait(&tempty[acc], ((j >> 1) - 1) & 1); tc_fence_after(); }
                const uint32_t d = tmem + (uint32_t)(acc * Cfg::kAccCols);
                for (int kb = 0; kb < ti.nkb; ++kb, ++it) {
                    const int s = it % STAGES;
                    mbar_wait(&full_bar[s], (it / STAGES) & 1);
                    tc_fence_after();
                    uint8_t* st = smem + s * kStageBytes;
                    const uint32_t a_hi = smem_u32(st), b_hi = smem_u32(st + Cfg::kAStage);
                    const uint32_t a_lo = smem_u32(st + Cfg::kAStage + Cfg::kBStage);
                    const uint32_t b_lo = a_lo + Cfg::kAStage;
                    const int nkk = min(kBK / 16, (klen - (ti.kb0 + kb) * kBK + 15) / 16);
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        if (kk > 0 && kk >= nkk) break;
                        // K-major: +32 B per 16-element k step inside the 128 B swizzle row;
                        // MN-major: +16 rows x 128 B per k step.
                        const uint32_t oa = A_MN ? kk * 2048 : kk * 32, ob = B_MN ? kk * 2048 : kk * 32;
                        const uint32_t la = A_MN ? 8192 : 16, lb = B_MN ? 8192 : 16, sbo = 1024;
                        const uint64_t dah = sdesc(a_hi + oa, la, sbo), dbh = sdesc(b_hi + ob, lb, sbo);
                        if ((args.diag & 2) && (kb > 0 || kk > 0)) continue;
                        tc_mma(d, dah, dbh, id, (kb > 0 || kk > 0) ? 1u : 0u);
                        if (TERMS == 3) {
                            const uint64_t dal = sdesc(a_lo + oa, la, sbo), dbl = sdesc(b_lo + ob, lb, sbo);
                            tc_mma(d, dah, dbl, id, 1u);
                            tc_mma(d, dal, dbh, id, 1u);
                        }
                    }
                    tc_commit(&empty_bar[s]);
                }
                tc_commit(&tfull[acc]);
                ++j;
            }
        }
    } else {
        // ================= epilogue: TMEM -> registers (+ReLU) -> swizzled smem -> TMA store
        // Each warp owns one TMEM lane quarter (32 rows of the tile) and moves it out in
        // 32-column chunks: tcgen05.ld 32x32b.x32 (thread = row), 16-byte smem stores in the
        // 128B-swizzle pattern (conflict-free), then one bulk tensor store per chunk; rows/columns
        // outside the tensor map's extent are clipped by the TMA unit.
        const int q = warp & 3;                       // TMEM lane quarter this warp may access
        uint8_t* ebuf = smem + STAGES * kStageBytes + q * 2 * kEpiBuf;
        int j = 0;
        for (int jt = 0;; ++jt) {
            const int t = next_tile(jt);
            __syncwarp();
            if (lane == 0) release_tile(jt);
            if (t < 0 || t >= ntiles) break;
            const TileInfo ti = tile_info<MODE>(args, t, M);
            const int row0 = ti.tm * kBM + q * 32;
            const int tile_n = ti.tn * BN;
            const bool rows_ok = MODE == 1 ? row0 < args.m_static : row0 < M;
            const bool has = ti.nkb > 0;
            const int acc = j & 1;
            if (has) {
                mbar_wait(&tfull[acc], (j >> 1) & 1);
                tc_fence_after();
            }
#pragma unroll
            for (int c0 = 0; c0 < BN; c0 += 2 * kEpiCols) {
                // two 32-column chunks per TMEM wait; each goes out through its own smem buffer
                const bool two = c0 + kEpiCols < BN;
                uint32_t v[2][32];
                if (has) {
                    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * Cfg::kAccCols + c0);
                    tmem_ld32(taddr, v[0]);
                    if (two) tmem_ld32(taddr + kEpiCols, v[1]);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                } else {
#pragma unroll
                    for (int x = 0; x < 32; ++x) { v[0][x] = 0u; v[1][x] = 0u; }
                }
                if (!rows_ok) continue;                 // (warp-uniform) nothing of this quarter is stored
                if (lane == 0) bulk_wait_read<0>();     // the previous stores have read both buffers
                __syncwarp();
#pragma unroll
                for (int hb = 0; hb < 2; ++hb) {
                    if (hb == 1 && !two) break;
                    uint8_t* myrow = ebuf + hb * kEpiBuf + lane * 128;
                    uint32_t mb = 0u;   // ReLU decisions of these 32 columns (MODE 2)
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        float4 f;
                        f.x = __uint_as_float(v[hb][4 * c]); f.y = __uint_as_float(v[hb][4 * c + 1]);
                        f.z = __uint_as_float(v[hb][4 * c + 2]); f.w = __uint_as_float(v[hb][4 * c + 3]);
                        if (args.relu) { f.x = fmaxf(f.x, 0.f); f.y = fmaxf(f.y, 0.f); f.z = fmaxf(f.z, 0.f); f.w = fmaxf(f.w, 0.f); }
                        if (MODE == 2)
                            mb |= ((f.x > 0.f ? 1u : 0u) | (f.y > 0.f ? 2u : 0u) | (f.z > 0.f ? 4u : 0u) | (f.w > 0.f ? 8u : 0u))
                                  << (4 * c);
                        *reinterpret_cast<float4*>(myrow + ((c ^ (lane & 7)) << 4)) = f;
                    }
                    if (MODE == 2 && args.mask && row0 + lane < M)
                        args.mask[(size_t)(row0 + lane) * args.mask_ld + ((tile_n + c0) >> 5) + hb] = mb;
                }
                fence_async_smem();
                __syncwarp();
                if (lane == 0 && !(args.diag & 1)) {
                    tma_store_3d(&mC, ebuf, tile_n + c0, row0, ti.z);
                    if (two) tma_store_3d(&mC, ebuf + kEpiBuf, tile_n + c0 + kEpiCols, row0, ti.z);
                    bulk_commit();
                }
            }
            if (MODE == 3 && has && !(args.diag & 8)) {
                // softmax cross-entropy of this thread's row (R15):
                // l = max + log sum exp(z - max) - z_y;  dZ = (softmax - onehot) / b_total
                constexpr int kZ = (BN + 31) / 32 * 32;
                uint32_t zr[kZ / 32][32];
#pragma unroll
                for (int c0 = 0; c0 < kZ; c0 += 32)
                    tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * Cfg::kAccCols + c0), zr[c0 / 32]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                float l = ce_rows<BN>(args, zr, row0 + lane, M);
                // the tile's loss: lanes (fixed tree), then the 4 warps in order -> row_loss[tile]
                // (one partial per 128-row tile; the last CTA sums the tiles in order)
                for (int o = 16; o; o >>= 1) l += __shfl_down_sync(0xffffffffu, l, o);
                if (lane == 0) ce_warp[j & 1][q] = l;
                asm volatile("bar.sync 1, 128;" ::: "memory");   // the 4 epilogue warps
                if (q == 0 && lane == 0) {
                    args.st->row_loss[ti.tm] = ((ce_warp[j & 1][0] + ce_warp[j & 1][1]) + ce_warp[j & 1][2]) + ce_warp[j & 1][3];
                    __threadfence();
                }
            }
            if (has) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
                ++j;
            }
        }
        if (lane == 0) bulk_wait_all();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cfg::kTmemCols));
    }
    if (args.sched && !args.clc && threadIdx.x == 0) {
        // every CTA has claimed its last (past-the-end) tile: the last one to finish re-arms the
        // counter for the next launch from this site
        __threadfence();   // this CTA's claims precede its "done" in every observer's view
        if (atomicAdd(args.sched + 1, 1) == (int)gridDim.x - 1) {
            args.sched[0] = 0;
            args.sched[1] = 0;
            __threadfence();
        }
    }
    if (MODE == 3 && !(args.diag & 16)) {
        // the last CTA to finish sums the per-tile losses in tile order (deterministic)
        if (threadIdx.x == 0) ce_last = atomicAdd(&args.st->ce_done, 1u) == gridDim.x - 1;
        __syncthreads();
        if (!ce_last) return;
        __threadfence();
        if (threadIdx.x == 0) {   // the tiles' partials in tile order
            float tot = 0.f;
            const int nt = (M + kBM - 1) / kBM;
            for (int t = 0; t < nt; ++t) tot += __ldcg(&args.st->row_loss[t]);
            args.st->loss = tot * (1.0f / (float)max(args.st->b_total, 1));
            args.st->ce_done = 0u;
        }
    }
}

// ------------------------------------------------------------------ host: tensor maps
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
        fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}

}  // namespace

// 2-D bf16 row-major [rows x cols] (cols contiguous), box {64, box_rows}, 128B swizzle, OOB -> 0.
bool make_tmap_bf16(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows) {
    EncodeFn fn = encode_fn();
    if (!fn || !base) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64u, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1u, 1u};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// k-block-tiled bf16 plane: {64, rows, ceil(cols/64)}, box {64, box_rows, 1}, 128B swizzle.
bool make_tmap_bf16_tiled(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows) {
    EncodeFn fn = encode_fn();
    if (!fn || !base) return false;
    cuuint64_t dims[3] = {64u, (cuuint64_t)rows, (cuuint64_t)((cols + 63) / 64)};
    cuuint64_t strides[2] = {128u, (cuuint64_t)rows * 128u};
    cuuint32_t box[3] = {64u, (cuuint32_t)box_rows, 1u};
    cuuint32_t estr[3] = {1u, 1u, 1u};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_tmap_rows_f32(CUtensorMap* map, const float* base, int64_t rows, int cols) {
    EncodeFn fn = encode_fn();
    if (!fn || !base || cols > 256 || (cols * 4) % 16 != 0) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    cuuint32_t box[2] = {(cuuint32_t)cols, 1u};
    cuuint32_t estr[2] = {1u, 1u};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp32 [depth x rows x cols] (cols contiguous, row stride ld elements, depth stride dstride
// elements), box {32, 32, 1}, 128B swizzle: the GEMM epilogue's store target.
bool make_tmap_f32(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld, int64_t depth,
                   int64_t dstride) {
    EncodeFn fn = encode_fn();
    if (!fn || !base) return false;
    cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)depth};
    cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)std::max<int64_t>(dstride, rows * ld) * 4};
    cuuint32_t box[3] = {(cuuint32_t)kEpiCols, 32u, 1u};
    cuuint32_t estr[3] = {1u, 1u, 1u};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box,
              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {
constexpr int kSMs = 148;

template <int BN, int STAGES, int TERMS, int MODE>
cudaError_t launch_tc(int grid, const TcGemmMaps& mp, const GemmArgs& a, cudaStream_t s) {
    using Cfg = TileCfg<BN>;
    constexpr int kAPlanes = TERMS == 3 ? 2 : 1;
    constexpr int smem = STAGES * kAPlanes * (Cfg::kAStage + Cfg::kBStage) + kEpiBytes + 1024;
    static_assert(smem <= 227 * 1024, "shared memory budget");
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_gemm_tc<BN, STAGES, TERMS, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    return launch_pdl(k_gemm_tc<BN, STAGES, TERMS, MODE>, grid, kThreads, smem, s, mp.a_hi, mp.a_lo, mp.b_hi,
                      mp.b_lo, mp.c, a);
}

template <int TERMS, int MODE>
cudaError_t dispatch_bn(int bn, int grid, const TcGemmMaps& mp, const GemmArgs& a, cudaStream_t s) {
    switch (bn) {
        case 16: return launch_tc<16, GS_TC_STAGES_NARROW, TERMS, MODE>(grid, mp, a, s);
        case 32: return launch_tc<32, GS_TC_STAGES_NARROW, TERMS, MODE>(grid, mp, a, s);
        case 48: return launch_tc<48, GS_TC_STAGES_NARROW, TERMS, MODE>(grid, mp, a, s);
        case 64: return launch_tc<64, GS_TC_STAGES_NARROW, TERMS, MODE>(grid, mp, a, s);
        case 96: return launch_tc<96, GS_TC_STAGES_WIDE, TERMS, MODE>(grid, mp, a, s);
        case 128: return launch_tc<128, GS_TC_STAGES_WIDE, TERMS, MODE>(grid, mp, a, s);
        default: return cudaErrorInvalidValue;
    }
}
template <int TERMS>
cudaError_t dispatch_ce(int bn, int grid, const TcGemmMaps& mp, const GemmArgs& a, cudaStream_t s) {
    switch (bn) {
        case 16: return launch_tc<16, GS_TC_STAGES_NARROW, TERMS, 3>(grid, mp, a, s);
        case 32: return launch_tc<32, GS_TC_STAGES_NARROW, TERMS, 3>(grid, mp, a, s);
        case 48: return launch_tc<48, GS_TC_STAGES_NARROW, TERMS, 3>(grid, mp, a, s);
        case 64: return launch_tc<64, GS_TC_STAGES_NARROW, TERMS, 3>(grid, mp, a, s);
        default: return cudaErrorInvalidValue;
    }
}
}  // namespace

int tc_tile_n(int n_pad) {
    if (n_pad <= 128) return n_pad;   // n_pad is a multiple of 16
    return 128;
}

// GS_GEMM_DYN=1 (A/B): the dynamic tile scheduler.  Measured slower than the static tile list
// (tile t on CTA t mod grid): products GEMM classes fwd 63 -> 67, dgrad 27 -> 30, wgrad 54 ->
// 61 µs per step (the claim + ring hand-off per tile costs more than late CTAs lose), so off.
bool dyn_sched() {
    static const bool d = [] { const char* e = getenv("GS_GEMM_DYN"); return e && e[0] == '1'; }();
    return d;
}

// GS_GEMM_CLC=1 (A/B): a grid of one CTA per tile of the worst case; a CTA that finished its tile
// cancels a CTA the hardware has not launched yet (clusterlaunchcontrol.try_cancel) and computes
// that CTA's tile, so the GEMM finishes on the SMs it got (the others may be held by the
// overlapped sampling kernel) instead of waiting for a fixed share of tiles on every SM
bool clc_sched() {
    static const bool d = [] { const char* e = getenv("GS_GEMM_CLC"); return e && e[0] == '1'; }();
    return d;
}

static int gemm_diag() {
    static int d = -1;
    if (d < 0) {
        const char* e = getenv("GS_GEMM_DIAG");
        d = e ? atoi(e) : 0;
    }
    return d;
}

cudaError_t launch_gemm_tc(int mode, bool bf16x3, const TcGemmMaps& maps, const int32_t* m_ptr, int m_static,
                           int m_cap, int n_pad, int k_pad, float* C, int ldc, int n_store, bool relu, int splits,
                           int64_t split_stride, cudaStream_t s, uint32_t* relu_mask, int mask_ld) {
    const int bn = tc_tile_n(n_pad);
    GemmArgs a{};
    a.mask = relu ? relu_mask : nullptr;
    a.mask_ld = mask_ld;
    a.m_ptr = m_ptr;
    a.m_static = m_static;
    a.m_tiles_cap = (m_cap + kBM - 1) / kBM;
    a.n_tiles = (n_pad + bn - 1) / bn;
    a.splits = splits;
    a.k_blocks = (k_pad + kBK - 1) / kBK;
    a.k_len = k_pad;
    a.n_store = n_store;
    a.C = C;
    a.ldc = ldc;
    a.relu = relu ? 1 : 0;
    a.split_stride = split_stride;
    a.diag = gemm_diag();
    a.sched = dyn_sched() ? maps.sched : nullptr;
    a.clc = clc_sched() ? 1 : 0;
    int tiles_cap;
    if (mode != 1) tiles_cap = a.m_tiles_cap * a.n_tiles;
    else tiles_cap = ((m_static + kBM - 1) / kBM) * a.n_tiles * splits;
    const int grid = a.clc ? std::max(1, tiles_cap) : std::max(1, std::min(kSMs, tiles_cap));
    if (mode == 0) return bf16x3 ? dispatch_bn<3, 0>(bn, grid, maps, a, s) : dispatch_bn<1, 0>(bn, grid, maps, a, s);
    if (mode == 2) return bf16x3 ? dispatch_bn<3, 2>(bn, grid, maps, a, s) : dispatch_bn<1, 2>(bn, grid, maps, a, s);
    return bf16x3 ? dispatch_bn<3, 1>(bn, grid, maps, a, s) : dispatch_bn<1, 1>(bn, grid, maps, a, s);
}

}  // namespace gs

namespace gs {
cudaError_t launch_gemm_tc_ce(bool bf16x3, const TcGemmMaps& maps, const int32_t* m_ptr, int m_cap, int n_pad,
                              int k_pad, float* Z, StepState* st, int classes, const int32_t* labels,
                              const int32_t* nodes, Split dz, cudaStream_t s) {
    if (n_pad > 64) return cudaErrorInvalidValue;
    GemmArgs a{};
    a.m_ptr = m_ptr;
    a.m_tiles_cap = (m_cap + kBM - 1) / kBM;
    a.n_tiles = 1;
    a.splits = 1;
    a.k_blocks = (k_pad + kBK - 1) / kBK;
    a.k_len = k_pad;
    a.n_store = n_pad;
    a.C = Z;
    a.ldc = n_pad;
    a.st = st;
    a.labels = labels;
    a.nodes = nodes;
    a.dz = dz;
    a.classes = classes;
    a.diag = gemm_diag();
    a.sched = dyn_sched() ? maps.sched : nullptr;
    const int grid = std::max(1, std::min(kSMs, a.m_tiles_cap));
    return bf16x3 ? dispatch_ce<3>(n_pad, grid, maps, a, s) : dispatch_ce<1>(n_pad, grid, maps, a, s);
}
}  // namespace gs
