// Internal device helpers of the B200 path (sm_100a).  Shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gs {

constexpr int kMaxHops = 8;

// Device-resident sizes of the batch in flight.  Every kernel of a step reads its
// extent from here, so one CUDA graph replays every step.
struct StepState {
    int32_t n_dst[kMaxHops + 1];
    int32_t n_src[kMaxHops + 1];
    int32_t n_edges[kMaxHops + 1];
    int32_t batch_n;      // seeds of this rank's batch
    int32_t b_total;      // seeds of the step over all ranks (Eq. 3 denominator, R9)
    uint32_t epoch;
    uint32_t g;           // global batch index (sampling key, R3)
    float loss;           // this rank's Σ ℓ_i / b_total
    uint32_t ce_done;     // CE blocks finished (reset by the last one)
    uint32_t seq;         // step sequence number (tags the sampling kernel's scan words)
    int32_t n_rf;         // ShaDow: rows of the last layer's receptive field (compacted layer L-1)
    int32_t pad2[2];
    float row_loss[1024]; // ℓ_i of the batch rows (batch_size <= 1024)
};

// Philox4x32-10 (R3): the method's counter-based draws.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) { k.x += 0x9E3779B9u; k.y += 0xBB67AE85u; }
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    }
    return c;
}

// word (draw & 3) of Philox at ctr = (a, b, tag<<28 | (epoch & 0xFFFFF)<<8 | hop, draw>>2)
__device__ __forceinline__ uint32_t method_draw(uint64_t seed, uint32_t tag, uint32_t a, uint32_t b,
                                                uint32_t epoch, uint32_t hop, uint32_t draw) {
    const uint4 o = philox4x32_10(
        make_uint4(a, b, (tag << 28) | ((epoch & 0xFFFFFu) << 8) | (hop & 0xFFu), draw >> 2),
        make_uint2((uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)));
    const uint32_t w = draw & 3u;
    return w == 0 ? o.x : w == 1 ? o.y : w == 2 ? o.z : o.w;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int global_warp() { return (blockIdx.x * blockDim.x + threadIdx.x) >> 5; }
__device__ __forceinline__ int total_warps() { return (gridDim.x * blockDim.x) >> 5; }

}  // namespace gs
