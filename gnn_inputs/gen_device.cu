// Device-side INPUT GENERATOR (gnn_inputs, not the method): builds the papers100M-shaped
// synthetic graph (BASELINE.json configs[4]: 111M nodes, 1.6B CSR entries, 128-d features) in
// GPU memory in seconds, with the recipe of gnn_inputs/synth.py:
//   degrees   d_v = clamp(floor(dmin * u_v^(-1/(alpha-1))), 1, floor(sqrt(nnz))), alpha = 2.1,
//             dmin bisected so that sum 2*ceil(d_v/2) ~= nnz
//   endpoints Chung-Lu, symmetric: node v draws ceil(d_v/2) partners u with P(u) ∝ d_u; both
//             directions stored; self-loops and duplicates dropped; rows ascending
//   features  x[v,j] = (h >> 41) * 2^-22 - 1, h = splitmix64(seed, S_FEATURE, v*F + j)
//   labels    y_v = ((h >> 32) * C) >> 32,      h = splitmix64(seed, S_LABEL, v)
// The splitmix64 counter hash is bit-identical to synth.hash_u64, so features and labels equal
// synth.feature_rows / synth.make_labels exactly (the oracle recomputes feature rows by that
// formula).  The CSR is defined by this generator (device pow/searchsorted); the oracle gets the
// same CSR (copied to the host).  Holds none of the method's arithmetic (no sampling, relabel,
// aggregation, loss); shares no code with paper_2403_17092_b200/ or oracle/.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull, kM1 = 0xBF58476D1CE4E5B9ull, kM2 = 0x94D049BB133111EBull;
constexpr uint64_t kDegree = 1, kEndpoint = 2, kFeature = 3, kLabel = 4;

__host__ __device__ inline uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= kM1;
    x ^= x >> 27;
    x *= kM2;
    return x ^ (x >> 31);
}
__host__ __device__ inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
    return mix64(seed * 0x100000001B3ull + stream * 0x1F3D5B79ull);
}
__device__ inline uint64_t hash_at(uint64_t key, uint64_t idx) { return mix64(key + (idx + 1) * kGamma); }
__device__ inline double uniform01(uint64_t key, uint64_t idx) {   // (0, 1], 53 bits
    return ((double)(hash_at(key, idx) >> 11) + 1.0) * 0x1p-53;
}

__global__ void k_base(int64_t n, uint64_t key, double expo, double* base) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        base[v] = pow(uniform01(key, v), expo);
}
__device__ inline int64_t deg_of(double dmin, double b, int64_t cap) {
    double d = floor(dmin * b);
    d = d < 1.0 ? 1.0 : (d > (double)cap ? (double)cap : d);
    return (int64_t)d;
}
__global__ void k_total(int64_t n, const double* base, double dmin, int64_t cap, unsigned long long* tot) {
    unsigned long long s = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = deg_of(dmin, base[v], cap);
        s += (unsigned long long)(2 * ((d + 1) / 2));
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(tot, s);
}
__global__ void k_degrees(int64_t n, const double* base, double dmin, int64_t cap, double* degf, int64_t* draws) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = deg_of(dmin, base[v], cap);
        degf[v] = (double)d;
        draws[v] = (d + 1) / 2;
    }
}
// draw k (owner v: doff[v] <= k < doff[v+1]) picks partner u = lower_bound(cum, r * tot): the
// first u with cum[u] >= r*tot; keys (v*n + u) and (u*n + v), self loops -> ~0 (dropped).
__global__ void k_keys(int64_t n, int64_t ndraws, const int64_t* doff, const double* cum, double tot, uint64_t key,
                       uint64_t* keys) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ndraws; k += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n;   // owner: last v with doff[v] <= k
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (doff[mid] <= k) lo = mid; else hi = mid;
        }
        const int64_t v = lo;
        const double x = uniform01(key, (uint64_t)k) * tot;
        int64_t a = 0, b = n;     // first u with cum[u] >= x
        while (a < b) {
            const int64_t mid = (a + b) >> 1;
            if (cum[mid] < x) a = mid + 1; else b = mid;
        }
        const int64_t u = a < n - 1 ? a : n - 1;
        if (u == v) {
            keys[2 * k] = ~0ull;
            keys[2 * k + 1] = ~0ull;
        } else {
            keys[2 * k] = (uint64_t)v * (uint64_t)n + (uint64_t)u;
            keys[2 * k + 1] = (uint64_t)u * (uint64_t)n + (uint64_t)v;
        }
    }
}
// row_ptr[v] = first index i of the sorted unique keys with key[i] >= v*n
__global__ void k_rowptr(int64_t n, int64_t m, const uint64_t* keys, int64_t* row_ptr) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= n; v += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t x = (uint64_t)v * (uint64_t)n;
        int64_t a = 0, b = m;
        while (a < b) {
            const int64_t mid = (a + b) >> 1;
            if (keys[mid] < x) a = mid + 1; else b = mid;
        }
        row_ptr[v] = a;
    }
}
__global__ void k_col(int64_t m, int64_t n, const uint64_t* keys, int32_t* col) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        col[i] = (int32_t)(keys[i] % (uint64_t)n);
}
__global__ void k_features(int64_t r0, int64_t rows, int F, int stride, uint64_t key, float* X) {
    const int64_t total = rows * stride;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / stride;
        const int j = (int)(t - r * stride);
        float x = 0.f;
        if (j < F) {
            const uint64_t h = hash_at(key, (uint64_t)(r0 + r) * (uint64_t)F + (uint64_t)j);
            x = (float)((double)(h >> 41) * 0x1p-22 - 1.0);
        }
        X[t] = x;
    }
}
__global__ void k_labels(int64_t n, int C, uint64_t key, int32_t* y) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        y[v] = (int32_t)(((hash_at(key, (uint64_t)v) >> 32) * (uint64_t)C) >> 32);
}

constexpr int kGrid = 148 * 16, kBlock = 256;

int64_t isqrt64(int64_t x) {
    int64_t r = (int64_t)sqrt((double)x);
    while (r * r > x) --r;
    while ((r + 1) * (r + 1) <= x) ++r;
    return r;
}

double bisect_dmin(int64_t n, const double* base, int64_t nnz, int64_t cap, unsigned long long* tot_dev) {
    double lo = 1e-3, hi = (double)cap;
    for (int it = 0; it < 60; ++it) {
        const double mid = 0.5 * (lo + hi);
        cudaMemset(tot_dev, 0, sizeof(unsigned long long));
        k_total<<<kGrid, kBlock>>>(n, base, mid, cap, tot_dev);
        unsigned long long t = 0;
        cudaMemcpy(&t, tot_dev, sizeof(t), cudaMemcpyDeviceToHost);
        if ((double)t < (double)nnz) lo = mid; else hi = mid;
    }
    return hi;
}

}  // namespace

extern "C" {

// Builds the CSR of (n, nnz, seed) on the current device.  On success *row_ptr_out (int64[n+1])
// and *col_out (int32[*nnz_out]) are cudaMalloc'ed buffers the caller frees with gen_free.
// Returns 0, or a negative CUDA error.
int gen_graph(int64_t n, int64_t nnz, uint64_t seed, int64_t** row_ptr_out, int32_t** col_out, int64_t* nnz_out) {
    cudaError_t e = cudaSuccess;
    const int64_t cap = std::max<int64_t>(1, isqrt64(std::max<int64_t>(nnz, 1)));
    double *base = nullptr, *degf = nullptr;
    int64_t *draws = nullptr, *doff = nullptr, *row_ptr = nullptr;
    unsigned long long* tot_dev = nullptr;
    uint64_t *keys = nullptr, *keys2 = nullptr;
    int64_t* nsel = nullptr;
    int32_t* col = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    int64_t ndraws = 0, m = 0;
    double dmin = 0, tot = 0;
#define G(x) do { e = (x); if (e != cudaSuccess) goto out; } while (0)
    G(cudaMalloc(&base, sizeof(double) * n));
    G(cudaMalloc(&tot_dev, sizeof(unsigned long long)));
    k_base<<<kGrid, kBlock>>>(n, stream_key(seed, kDegree), -1.0 / (2.1 - 1.0), base);
    G(cudaGetLastError());
    dmin = bisect_dmin(n, base, nnz, cap, tot_dev);
    G(cudaMalloc(&degf, sizeof(double) * n));
    G(cudaMalloc(&draws, sizeof(int64_t) * (n + 1)));
    G(cudaMalloc(&doff, sizeof(int64_t) * (n + 1)));
    k_degrees<<<kGrid, kBlock>>>(n, base, dmin, cap, degf, draws);
    G(cudaMemset(draws + n, 0, sizeof(int64_t)));
    G(cudaFree(base));
    base = nullptr;
    // doff = exclusive scan of draws (n+1 entries: doff[n] = total draws); cum = inclusive scan of degf
    G(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, draws, doff, n + 1));
    G(cudaMalloc(&tmp, tmp_bytes));
    G(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, draws, doff, n + 1));
    G(cudaFree(tmp));
    tmp = nullptr;
    G(cudaMemcpy(&ndraws, doff + n, sizeof(int64_t), cudaMemcpyDeviceToHost));
    G(cudaFree(draws));
    draws = nullptr;
    {
        double* cum = nullptr;
        G(cudaMalloc(&cum, sizeof(double) * n));
        tmp_bytes = 0;
        G(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, degf, cum, n));
        G(cudaMalloc(&tmp, tmp_bytes));
        G(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, degf, cum, n));
        G(cudaFree(tmp));
        tmp = nullptr;
        G(cudaMemcpy(&tot, cum + n - 1, sizeof(double), cudaMemcpyDeviceToHost));
        G(cudaMalloc(&keys, sizeof(uint64_t) * 2 * ndraws));
        k_keys<<<kGrid, kBlock>>>(n, ndraws, doff, cum, tot, stream_key(seed, kEndpoint), keys);
        G(cudaGetLastError());
        G(cudaFree(cum));
    }
    G(cudaFree(degf));
    degf = nullptr;
    G(cudaFree(doff));
    doff = nullptr;
    {   // sort + unique (self-loop keys ~0 sort last and are dropped)
        const int64_t nk = 2 * ndraws;
        G(cudaMalloc(&keys2, sizeof(uint64_t) * nk));
        tmp_bytes = 0;
        G(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys, keys2, nk));
        G(cudaMalloc(&tmp, tmp_bytes));
        G(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, keys, keys2, nk));
        G(cudaFree(tmp));
        tmp = nullptr;
        G(cudaMalloc(&nsel, sizeof(int64_t)));
        tmp_bytes = 0;
        G(cub::DeviceSelect::Unique(nullptr, tmp_bytes, keys2, keys, nsel, nk));
        G(cudaMalloc(&tmp, tmp_bytes));
        G(cub::DeviceSelect::Unique(tmp, tmp_bytes, keys2, keys, nsel, nk));
        G(cudaFree(tmp));
        tmp = nullptr;
        G(cudaFree(keys2));
        keys2 = nullptr;
        G(cudaMemcpy(&m, nsel, sizeof(int64_t), cudaMemcpyDeviceToHost));
        uint64_t last = 0;
        if (m > 0) G(cudaMemcpy(&last, keys + m - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost));
        if (m > 0 && last == ~0ull) --m;
    }
    G(cudaMalloc(&row_ptr, sizeof(int64_t) * (n + 1)));
    G(cudaMalloc(&col, sizeof(int32_t) * std::max<int64_t>(m, 1)));
    k_rowptr<<<kGrid, kBlock>>>(n, m, keys, row_ptr);
    k_col<<<kGrid, kBlock>>>(m, n, keys, col);
    G(cudaGetLastError());
    G(cudaDeviceSynchronize());
    *row_ptr_out = row_ptr;
    *col_out = col;
    *nnz_out = m;
    row_ptr = nullptr;
    col = nullptr;
out:
    for (void* p : {(void*)base, (void*)degf, (void*)draws, (void*)doff, (void*)tot_dev, (void*)keys, (void*)keys2,
                    (void*)nsel, tmp, (void*)row_ptr, (void*)col})
        if (p) cudaFree(p);
#undef G
    return e == cudaSuccess ? 0 : -(int)e;
}

// Rows [r0, r0+rows) of the feature table (row stride `stride`, padding columns 0) into X (device).
int gen_features(int64_t r0, int64_t rows, int F, int stride, uint64_t seed, float* X) {
    k_features<<<kGrid, kBlock>>>(r0, rows, F, stride, stream_key(seed, kFeature), X);
    const cudaError_t e = cudaDeviceSynchronize();
    return e == cudaSuccess ? 0 : -(int)e;
}

int gen_labels(int64_t n, int C, uint64_t seed, int32_t* y) {
    k_labels<<<kGrid, kBlock>>>(n, C, stream_key(seed, kLabel), y);
    const cudaError_t e = cudaDeviceSynchronize();
    return e == cudaSuccess ? 0 : -(int)e;
}

void gen_free(void* p) { cudaFree(p); }

}  // extern "C"

extern "C" {
void* gen_alloc(int64_t bytes) {
    void* p = nullptr;
    return cudaMalloc(&p, (size_t)bytes) == cudaSuccess ? p : nullptr;
}
int gen_d2h(void* dst_host, const void* src_dev, int64_t bytes) {
    return cudaMemcpy(dst_host, src_dev, (size_t)bytes, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : -1;
}
int gen_set_device(int dev) { return cudaSetDevice(dev) == cudaSuccess ? 0 : -1; }
}
