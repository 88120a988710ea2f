// Epoch permutation keys (sm_100a).  The sampling phases themselves
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

}  // namespace

void launch_perm_keys(const int32_t* train, int64_t n, uint64_t seed, int64_t epoch, uint64_t* keys, cudaStream_t s) {
    if (n <= 0) return;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    k_perm_keys<<<blocks, 256, 0, s>>>(train, n, seed, (uint32_t)epoch, keys);
}


}  // namespace gs
