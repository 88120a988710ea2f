// Epoch permutation keys and the per-step preamble (sm_100a).  The sampling phases themselves
// are one persistent kernel in sample_step.cu.
#include "kernels.h"

namespace gs {
namespace {

// key64(v) = (w0 << 32) | w1 of Philox tag 1 at (v, 0, epoch)   (R7)
__global__ void k_perm_keys(const int32_t* train, int64_t n, uint64_t seed, uint32_t epoch, uint64_t* keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = (uint32_t)train[i];
        const uint4 o = philox4x32_10(make_uint4(v, 0u, (1u << 28) | ((epoch & 0xFFFFFu) << 8), 0u),
                                      make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
        keys[i] = ((uint64_t)o.x << 32) | o.y;
    }
}

// dst_0 = seeds (batch order): nodes[i] = seed_i, map[seed_i] = i; reset the step's sizes.
__global__ void k_begin_step(StepState* st, const int32_t* seed_src, int32_t n, int32_t b_total, uint32_t epoch,
                             uint32_t g, int32_t* nodes, int32_t* map, uint32_t* seq) {
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
        st->seq = ++*seq;     // unique across both batch sets (the scan words are shared)
    }
}

}  // namespace

void launch_perm_keys(const int32_t* train, int64_t n, uint64_t seed, int64_t epoch, uint64_t* keys, cudaStream_t s) {
    if (n <= 0) return;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    k_perm_keys<<<blocks, 256, 0, s>>>(train, n, seed, (uint32_t)epoch, keys);
}

void launch_begin_step(StepState* st, const int32_t* seed_src, int32_t n, int32_t b_total, uint32_t epoch,
                       uint32_t g, int32_t* nodes, int32_t* map, uint32_t* seq, cudaStream_t s) {
    k_begin_step<<<1, 1024, 0, s>>>(st, seed_src, n, b_total, epoch, g, nodes, map, seq);
}

}  // namespace gs
