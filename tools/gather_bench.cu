// Random-row gather ceiling (tools/gather_ceiling.py): a warp per output row sums U random
// rows of an [N x F] fp32 table (indices precomputed, no dependent loads), U rows in flight.
#include <cuda_runtime.h>
#include <stdint.h>

template <int U>
__global__ void k_gather(const float4* __restrict__ X, int nch, const int* __restrict__ idx, int R,
                         float4* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int W = (gridDim.x * blockDim.x) >> 5;
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r * U < R; r += W) {
        float4 acc = {0.f, 0.f, 0.f, 0.f};
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = r * U + u;
            const int row = j < R ? __ldg(idx + j) : 0;
            v[u] = lane < nch ? __ldg(X + (int64_t)row * nch + lane) : acc;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
        if (lane < nch) out[(int64_t)r * nch + lane] = acc;
    }
}

extern "C" float gather_bench(const float* X, int F, const int* idx, int R, float* out, int U, int blocks, int reps) {
    const int nch = F / 4;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int i = 0; i < reps; ++i) {
        cudaEventRecord(a);
        switch (U) {
            case 1: k_gather<1><<<blocks, 256>>>((const float4*)X, nch, idx, R, (float4*)out); break;
            case 2: k_gather<2><<<blocks, 256>>>((const float4*)X, nch, idx, R, (float4*)out); break;
            case 4: k_gather<4><<<blocks, 256>>>((const float4*)X, nch, idx, R, (float4*)out); break;
            case 8: k_gather<8><<<blocks, 256>>>((const float4*)X, nch, idx, R, (float4*)out); break;
            default: k_gather<16><<<blocks, 256>>>((const float4*)X, nch, idx, R, (float4*)out); break;
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best * 1e3f;
}
