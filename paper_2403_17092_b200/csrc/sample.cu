// Epoch permutation keys (sm_100a).  The sampling phases themselves
// are one persistent kernel in sample_step.cu.
#include <cstdlib>
#include <mutex>
#include <set>

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

// Symmetry of the CSR: every entry u of row v has v in row u (rows ascending: binary search).
// A warp per row; *asym is set on the first missing reverse entry.
__global__ void k_check_symmetric(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col, int64_t n,
                                  int* __restrict__ asym) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = w0; v < n; v += nw) {
        const int64_t rb = row_ptr[v], re = row_ptr[v + 1];
        for (int64_t p = rb + lane; p < re; p += 32) {
            const int u = col[p];
            int64_t lo = row_ptr[u], hi = row_ptr[u + 1];
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (col[mid] < v) lo = mid + 1; else hi = mid;
            }
            if (lo >= row_ptr[u + 1] || col[lo] != v) atomicOr(asym, 1);
        }
    }
}

// Validation of a graph given in device memory (gnn_graph_create_device): bad[0] |= 1 row_ptr not
// non-decreasing or row_ptr[0] != 0, 2 a column id out of [0, n), 4 a row not strictly
// ascending (duplicate or unsorted), 8 a label out of [0, C).
__global__ void k_validate(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col, int64_t n,
                           const int32_t* __restrict__ y, int C, int* __restrict__ bad) {
    int f = 0;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    if (tid == 0 && row_ptr[0] != 0) f |= 1;
    for (int64_t v = tid; v < n; v += nth) {
        const int64_t rb = row_ptr[v], re = row_ptr[v + 1];
        if (re < rb) { f |= 1; continue; }
        if (y[v] < 0 || y[v] >= C) f |= 8;
    }
    const int64_t nnz = row_ptr[n];
    for (int64_t v = tid; v < n; v += nth) {   // rows: each entry vs its predecessor in the row
        const int64_t rb = row_ptr[v], re = row_ptr[v + 1];
        for (int64_t p = rb; p < re && p < nnz; ++p) {
            const int c = col[p];
            if (c < 0 || c >= n) f |= 2;
            if (p > rb && c <= col[p - 1]) f |= 4;
        }
    }
    if (f) atomicOr(bad, f);
}

// NEXT-2 cache fill: a warp per cached row, 16-byte chunks (the row read like the aggregation reads it).
__global__ void k_cache_fill(FeatRows src, const int32_t* __restrict__ ids, int64_t n, int ld, float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w0; i < n; i += nw) {
        const int64_t r = ids[i], sh = r / src.rps;   // the owner's copy (never the cache itself)
        const float4* p = reinterpret_cast<const float4*>(src.shards[sh] + (r - sh * src.rps) * ld);
        float4* q = reinterpret_cast<float4*>(out + i * ld);
        for (int c = lane; c < (ld >> 2); c += 32) q[c] = p[c];
    }
}

}  // namespace

void launch_cache_fill(FeatRows src, const int32_t* ids, int64_t n, int ld, float* out, cudaStream_t s) {
    if (n <= 0) return;
    k_cache_fill<<<148 * 8, 256, 0, s>>>(src, ids, n, ld, out);
}

int validate_graph(const int64_t* row_ptr, const int32_t* col, int64_t n, const int32_t* y, int C) {
    int* d = nullptr;
    if (cudaMalloc(&d, sizeof(int)) != cudaSuccess) return -1;
    int h = 0;
    bool ok = cudaMemset(d, 0, sizeof(int)) == cudaSuccess;
    if (ok) {
        k_validate<<<148 * 16, 256>>>(row_ptr, col, n, y, C, d);
        ok = cudaGetLastError() == cudaSuccess;
    }
    ok = ok && cudaMemcpy(&h, d, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess;
    cudaFree(d);
    return ok ? h : -1;
}

void apply_carveout(const void* kernel) {
    static const int pct = [] { const char* e = std::getenv("GS_CARVEOUT"); return e ? std::atoi(e) : -1; }();
    if (pct < 0) return;
    static std::mutex mu;
    static std::set<const void*> done;
    std::lock_guard<std::mutex> lk(mu);
    if (done.insert(kernel).second) cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

bool check_symmetric(const int64_t* row_ptr, const int32_t* col, int64_t n, bool* symmetric) {
    int* d = nullptr;
    if (cudaMalloc(&d, sizeof(int)) != cudaSuccess) return false;
    int h = 0;
    bool ok = cudaMemset(d, 0, sizeof(int)) == cudaSuccess;
    if (ok && n > 0) {
        k_check_symmetric<<<148 * 8, 256>>>(row_ptr, col, n, d);
        ok = cudaGetLastError() == cudaSuccess;
    }
    ok = ok && cudaMemcpy(&h, d, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess;
    cudaFree(d);
    *symmetric = h == 0;
    return ok;
}

void launch_perm_keys(const int32_t* train, int64_t n, uint64_t seed, int64_t epoch, uint64_t* keys, cudaStream_t s) {
    if (n <= 0) return;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    k_perm_keys<<<blocks, 256, 0, s>>>(train, n, seed, (uint32_t)epoch, keys);
}


}  // namespace gs
