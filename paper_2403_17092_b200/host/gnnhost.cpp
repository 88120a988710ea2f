// Host-core trainer rank (include/gnnhost.h; §3).
// The per-mini-batch step on the host's cores in fp32 with OpenMP: sampling (R3/R4/R6),
// GraphSAGE-mean / GCN layers (Eqs. 1-2; R11/R12), softmax
// cross-entropy (Eq. 3; R15) and its exact backward.  Independent of the CUDA
// path and of the oracle (no shared code).  Parallel loops write disjoint outputs, and every
// reduction runs in a fixed order, so results do not depend on the thread count.
#include "gnnhost.h"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;
int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

// ---------------------------------------------------------------- counter RNG (R3)
// Philox4x32-10: multipliers 0xD2511F53 / 0xCD9E8D57, Weyl increments 0x9E3779B9 / 0xBB67AE85.
struct Philox {
    uint32_t k0, k1;
    explicit Philox(uint64_t seed) : k0((uint32_t)seed), k1((uint32_t)(seed >> 32)) {}
    void block(uint32_t c[4]) const {
        uint32_t a = k0, b = k1;
        for (int round = 0; round < 10; ++round) {
            const uint64_t m0 = (uint64_t)0xD2511F53u * c[0], m1 = (uint64_t)0xCD9E8D57u * c[2];
            const uint32_t x0 = (uint32_t)(m1 >> 32) ^ c[1] ^ a, x2 = (uint32_t)(m0 >> 32) ^ c[3] ^ b;
            c[1] = (uint32_t)m1;
            c[3] = (uint32_t)m0;
            c[0] = x0;
            c[2] = x2;
            a += 0x9E3779B9u;
            b += 0xBB67AE85u;
        }
    }
    // word (draw mod 4) of the block at (a, b, tag | epoch | hop, draw / 4)
    uint32_t word(uint32_t tag, uint32_t a, uint32_t b, int64_t epoch, uint32_t hop, uint32_t draw) const {
        uint32_t c[4] = {a, b, (tag << 28) | ((uint32_t)(epoch & 0xFFFFF) << 8) | (hop & 0xFFu), draw >> 2};
        block(c);
        return c[draw & 3];
    }
};

// ---------------------------------------------------------------- batch structure
struct Block {               // one hop: dst rows (the first n_dst of src), CSR over local ids
    int32_t n_dst = 0, n_src = 0;
    std::vector<int32_t> rowptr, col, src;   // src: global ids of the local nodes
};

struct Layer {
    int in = 0, out = 0, rows = 0;   // rows of W: 2*in (SAGE [W_self; W_neigh]) or in (GCN)
    int64_t off = 0;
};

}  // namespace

struct gnnh_model {
    int64_t N = 0;
    const int64_t* row_ptr = nullptr;
    const int32_t* col = nullptr;
    const float* X = nullptr;
    int F = 0, ldx = 0, C = 0;
    const int32_t* y = nullptr;
    int model = GNNH_SAGE_MEAN, L = 0;
    std::vector<int> fanouts;   // input-layer-first
    float lr = 0.f;
    Philox rng{0};
    std::vector<Layer> layers;
    std::vector<float> W;       // flat parameters
    std::vector<Block> hops;    // of the last batch (seeds outward)
};

namespace {

// Floyd's k-of-d (R4): for i = 0..k-1, j = d-k+i, t = floor(r_i (j+1) / 2^32); keep t unless it
// was kept already, then keep j.  Positions come back ascending.
void floyd(const Philox& rng, int64_t epoch, uint32_t g, uint32_t hop, uint32_t v, int64_t d, int k,
           std::vector<int64_t>& pos) {
    pos.clear();
    for (int i = 0; i < k; ++i) {
        const int64_t j = d - k + i;
        const uint32_t r = rng.word(0u, v, g, epoch, hop, (uint32_t)i);
        const int64_t t = (int64_t)(((uint64_t)r * (uint64_t)(j + 1)) >> 32);
        pos.push_back(std::find(pos.begin(), pos.end(), t) == pos.end() ? t : j);
    }
    std::sort(pos.begin(), pos.end());
}

// Hop h of the batch: dst -> sampled neighbours (ascending CSR position) -> relabel: src = dst ++
// the new nodes in ascending global id (R6); the next hop's dst is this src.
void sample_hop(const gnnh_model& m, Block& b, const std::vector<int32_t>& dst, int k, int64_t epoch, uint32_t g,
                uint32_t hop) {
    const int64_t nd = (int64_t)dst.size();
    b.n_dst = (int32_t)nd;
    std::vector<int32_t> cnt(nd);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nd; ++i) {
        const int64_t d = m.row_ptr[dst[i] + 1] - m.row_ptr[dst[i]];
        cnt[i] = (int32_t)std::min<int64_t>(d, k);
    }
    b.rowptr.assign(nd + 1, 0);
    for (int64_t i = 0; i < nd; ++i) b.rowptr[i + 1] = b.rowptr[i] + cnt[i];
    std::vector<int32_t> nbr(b.rowptr[nd]);
#pragma omp parallel
    {
        std::vector<int64_t> pos;
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < nd; ++i) {
            const int32_t v = dst[i];
            const int64_t start = m.row_ptr[v], d = m.row_ptr[v + 1] - start;
            int32_t* o = nbr.data() + b.rowptr[i];
            if (d <= k) {
                for (int64_t q = 0; q < d; ++q) o[q] = m.col[start + q];
            } else {
                floyd(m.rng, epoch, g, hop, (uint32_t)v, d, k, pos);
                for (int q = 0; q < k; ++q) o[q] = m.col[start + pos[q]];
            }
        }
    }
    // relabel: dst keep their positions; the other neighbours get n_dst + rank in ascending id
    std::vector<int32_t> fresh(nbr);
    std::sort(fresh.begin(), fresh.end());
    fresh.erase(std::unique(fresh.begin(), fresh.end()), fresh.end());
    std::vector<int32_t> dsorted(dst);
    std::sort(dsorted.begin(), dsorted.end());
    std::vector<int32_t> news;
    news.reserve(fresh.size());
    std::set_difference(fresh.begin(), fresh.end(), dsorted.begin(), dsorted.end(), std::back_inserter(news));
    b.src = dst;
    b.src.insert(b.src.end(), news.begin(), news.end());
    b.n_src = (int32_t)b.src.size();
    // local id of a neighbour: a dst (binary search over (id, position) pairs) or a new node
    std::vector<std::pair<int32_t, int32_t>> dpos(nd);
    for (int64_t i = 0; i < nd; ++i) dpos[i] = {dst[i], (int32_t)i};
    std::sort(dpos.begin(), dpos.end());
    b.col.resize(nbr.size());
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < (int64_t)nbr.size(); ++e) {
        const int32_t u = nbr[e];
        auto it = std::lower_bound(dpos.begin(), dpos.end(), std::make_pair(u, INT32_MIN));
        if (it != dpos.end() && it->first == u) {
            b.col[e] = it->second;
        } else {
            b.col[e] = (int32_t)(nd + (std::lower_bound(news.begin(), news.end(), u) - news.begin()));
        }
    }
}

// Â (R11/R12) as per-edge weights and GCN self weights of a block.
void block_weights(int model, const Block& b, std::vector<float>& w_edge, std::vector<float>& w_self) {
    const int64_t ne = b.rowptr[b.n_dst];
    w_edge.assign(ne, 0.f);
    w_self.assign(b.n_dst, 0.f);
    if (model == GNNH_SAGE_MEAN) {
        for (int32_t v = 0; v < b.n_dst; ++v) {
            const int32_t deg = b.rowptr[v + 1] - b.rowptr[v];
            const float w = deg ? 1.0f / (float)deg : 0.f;
            for (int32_t e = b.rowptr[v]; e < b.rowptr[v + 1]; ++e) w_edge[e] = w;
        }
        return;
    }
    // d_in(v) = deg(v) + 1, d_out(u) = outdeg(u) + [u < n_dst]
    std::vector<int32_t> outdeg(b.n_src, 0);
    for (int64_t e = 0; e < ne; ++e) ++outdeg[b.col[e]];
    for (int32_t v = 0; v < b.n_dst; ++v) {
        const double din = (double)(b.rowptr[v + 1] - b.rowptr[v]) + 1.0;
        for (int32_t e = b.rowptr[v]; e < b.rowptr[v + 1]; ++e) {
            const int32_t u = b.col[e];
            const double dout = (double)outdeg[u] + (u < b.n_dst ? 1.0 : 0.0);
            w_edge[e] = (float)(1.0 / std::sqrt(din * dout));
        }
        w_self[v] = (float)(1.0 / std::sqrt(din * ((double)outdeg[v] + 1.0)));
    }
}

// C[M x N] = A[M x K] B[K x N] (row-major, fp32 accumulation in k order), rows in parallel
void gemm_nn(const float* A, const float* B, float* Cm, int64_t M, int K, int N) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < M; ++i) {
        float* c = Cm + i * N;
        std::fill(c, c + N, 0.f);
        const float* a = A + i * K;
        for (int k = 0; k < K; ++k) {
            const float av = a[k];
            const float* brow = B + (int64_t)k * N;
            for (int n = 0; n < N; ++n) c[n] += av * brow[n];
        }
    }
}
// C[M x K] = D[M x N] W^T, W [K x N]
void gemm_nt(const float* D, const float* Wm, float* Cm, int64_t M, int N, int K) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < M; ++i) {
        const float* d = D + i * N;
        for (int k = 0; k < K; ++k) {
            const float* w = Wm + (int64_t)k * N;
            float s = 0.f;
            for (int n = 0; n < N; ++n) s += d[n] * w[n];
            Cm[i * K + k] = s;
        }
    }
}
// G[K x N] = A^T D, A [M x K], D [M x N]: fixed row chunks, partials summed in chunk order
void gemm_tn(const float* A, const float* D, float* G, int64_t M, int K, int N) {
    const int64_t chunk = 512;
    const int64_t nchunks = (M + chunk - 1) / chunk;
    std::vector<float> part((size_t)std::max<int64_t>(nchunks, 1) * K * N, 0.f);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = 0; c < nchunks; ++c) {
        float* p = part.data() + c * (int64_t)K * N;
        for (int64_t i = c * chunk; i < std::min(M, (c + 1) * chunk); ++i) {
            const float* a = A + i * K;
            const float* d = D + i * N;
            for (int k = 0; k < K; ++k) {
                const float av = a[k];
                if (av == 0.f) continue;
                float* pr = p + (int64_t)k * N;
                for (int n = 0; n < N; ++n) pr[n] += av * d[n];
            }
        }
    }
    const int64_t KN = (int64_t)K * N;
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < KN; ++x) {
        float s = 0.f;
        for (int64_t c = 0; c < nchunks; ++c) s += part[c * KN + x];
        G[x] = s;
    }
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

const char* gnnh_last_error(void) { return g_err.c_str(); }

int gnnh_create(int64_t num_nodes, const int64_t* row_ptr, const int32_t* col, const float* features,
                int32_t feat_dim, int32_t feat_stride, const int32_t* labels, int32_t num_classes, int32_t model,
                int32_t num_layers, int32_t hidden, const int32_t* fanouts, float lr, uint64_t seed,
                gnnh_model** out) {
    if (!row_ptr || !col || !features || !labels || !fanouts || !out) return fail(GNNH_ERR_PARAM, "NULL argument");
    if (num_nodes <= 0 || num_nodes >= INT32_MAX) return fail(GNNH_ERR_RANGE, "num_nodes out of range");
    if (feat_dim <= 0 || feat_stride < feat_dim || num_classes <= 0 || hidden <= 0)
        return fail(GNNH_ERR_CONFIG, "bad feat_dim / feat_stride / num_classes / hidden");
    if (model != GNNH_SAGE_MEAN && model != GNNH_GCN) return fail(GNNH_ERR_CONFIG, "unknown model");
    if (num_layers < 1 || num_layers > 8) return fail(GNNH_ERR_CONFIG, "num_layers must be 1..8");
    for (int l = 0; l < num_layers; ++l)
        if (fanouts[l] < 1) return fail(GNNH_ERR_CONFIG, "fanouts must be >= 1");
    if (!(lr >= 0.f)) return fail(GNNH_ERR_PARAM, "lr must be >= 0");
    gnnh_model* m = new (std::nothrow) gnnh_model();
    if (!m) return fail(GNNH_ERR_OOM, "host allocation");
    m->N = num_nodes; m->row_ptr = row_ptr; m->col = col; m->X = features; m->F = feat_dim;
    m->ldx = feat_stride; m->y = labels; m->C = num_classes; m->model = model; m->L = num_layers;
    m->fanouts.assign(fanouts, fanouts + num_layers); m->lr = lr; m->rng = Philox(seed);
    int64_t off = 0;
    for (int l = 0; l < num_layers; ++l) {
        Layer ly;
        ly.in = l == 0 ? feat_dim : hidden;
        ly.out = l == num_layers - 1 ? num_classes : hidden;
        ly.rows = (model == GNNH_SAGE_MEAN ? 2 : 1) * ly.in;
        ly.off = off;
        off += (int64_t)ly.rows * ly.out;
        m->layers.push_back(ly);
    }
    m->W.assign(off, 0.f);
    *out = m;
    return GNNH_OK;
}

int gnnh_destroy(gnnh_model* m) {
    delete m;
    return GNNH_OK;
}

int64_t gnnh_param_count(const gnnh_model* m) { return m ? (int64_t)m->W.size() : 0; }

int gnnh_set_params(gnnh_model* m, const float* params, int64_t n) {
    if (!m || !params) return fail(GNNH_ERR_PARAM, "NULL argument");
    if (n != (int64_t)m->W.size()) return fail(GNNH_ERR_SHAPE, "n != param_count");
    std::memcpy(m->W.data(), params, sizeof(float) * n);
    return GNNH_OK;
}

int gnnh_get_params(const gnnh_model* m, float* params_out, int64_t n) {
    if (!m || !params_out) return fail(GNNH_ERR_PARAM, "NULL argument");
    if (n != (int64_t)m->W.size()) return fail(GNNH_ERR_SHAPE, "n != param_count");
    std::memcpy(params_out, m->W.data(), sizeof(float) * n);
    return GNNH_OK;
}

int gnnh_epoch_permutation(const gnnh_model* m, const int32_t* train_ids, int64_t n, int64_t epoch,
                           int32_t* perm_out) {
    if (!m || (n && (!train_ids || !perm_out))) return fail(GNNH_ERR_PARAM, "NULL argument");
    std::vector<std::pair<uint64_t, int32_t>> kv(n);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const uint32_t v = (uint32_t)train_ids[i];
        uint32_t c[4] = {v, 0u, (1u << 28) | ((uint32_t)(epoch & 0xFFFFF) << 8), 0u};
        m->rng.block(c);   // draws 0 and 1: words 0 and 1 of block 0
        kv[i] = {((uint64_t)c[0] << 32) | c[1], train_ids[i]};
    }
    std::sort(kv.begin(), kv.end());
    for (int64_t i = 0; i < n; ++i) perm_out[i] = kv[i].second;
    return GNNH_OK;
}

int gnnh_grads(gnnh_model* m, const int32_t* seeds, int32_t n_seeds, int32_t b_total, int64_t epoch, int64_t g,
               float* grads_out, float* loss_out) {
    if (!m || !grads_out || (n_seeds > 0 && !seeds)) return fail(GNNH_ERR_PARAM, "NULL argument");
    if (n_seeds < 0 || b_total < n_seeds) return fail(GNNH_ERR_PARAM, "need 0 <= n_seeds <= b_total");
    std::fill(grads_out, grads_out + m->W.size(), 0.f);
    if (loss_out) *loss_out = 0.f;
    if (n_seeds == 0) return GNNH_OK;
    {
        std::vector<int32_t> s(seeds, seeds + n_seeds);
        std::sort(s.begin(), s.end());
        for (int32_t i = 0; i < n_seeds; ++i) {
            if (s[i] < 0 || s[i] >= m->N) return fail(GNNH_ERR_RANGE, "seed id out of [0, N)");
            if (i && s[i] == s[i - 1]) return fail(GNNH_ERR_PARAM, "repeated seed id");
        }
    }
    const int L = m->L;
    // ---- sampling: hop h uses fanouts[L-1-h] (hop 0 = the seeds' neighbours)
    m->hops.assign(L, Block());
    std::vector<int32_t> dst(seeds, seeds + n_seeds);
    for (int h = 0; h < L; ++h) {
        sample_hop(*m, m->hops[h], dst, m->fanouts[L - 1 - h], epoch, (uint32_t)g, (uint32_t)h);
        dst = m->hops[h].src;
    }
    // ---- forward: layer l (0-based, input-first) aggregates over hop L-1-l
    std::vector<std::vector<float>> A(L), Pre(L), H(L + 1), wE(L), wS(L);
    {
        const Block& b0 = m->hops[L - 1];
        H[0].resize((size_t)b0.n_src * m->F);
#pragma omp parallel for schedule(static)
        for (int64_t r = 0; r < b0.n_src; ++r)
            std::memcpy(H[0].data() + r * m->F, m->X + (int64_t)b0.src[r] * m->ldx, sizeof(float) * m->F);
    }
    for (int l = 0; l < L; ++l) {
        const Block& b = m->hops[L - 1 - l];
        const Layer& ly = m->layers[l];
        const int in = ly.in;
        block_weights(m->model, b, wE[l], wS[l]);
        const bool sage = m->model == GNNH_SAGE_MEAN;
        A[l].assign((size_t)b.n_dst * ly.rows, 0.f);
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t v = 0; v < b.n_dst; ++v) {
            float* a = A[l].data() + v * ly.rows;
            float* agg = sage ? a + in : a;
            const float* hv = H[l].data() + v * in;
            if (sage) std::memcpy(a, hv, sizeof(float) * in);
            else for (int c = 0; c < in; ++c) agg[c] = wS[l][v] * hv[c];
            for (int32_t e = b.rowptr[v]; e < b.rowptr[v + 1]; ++e) {
                const float* hu = H[l].data() + (int64_t)b.col[e] * in;
                const float w = wE[l][e];
                for (int c = 0; c < in; ++c) agg[c] += w * hu[c];
            }
        }
        Pre[l].resize((size_t)b.n_dst * ly.out);
        gemm_nn(A[l].data(), m->W.data() + ly.off, Pre[l].data(), b.n_dst, ly.rows, ly.out);
        H[l + 1] = Pre[l];
        if (l < L - 1)
            for (float& x : H[l + 1]) x = x > 0.f ? x : 0.f;
    }
    // ---- loss: Σ_i (logsumexp(z_i) - z_{i,y_i}) / b_total; dZ = (softmax - onehot) / b_total
    const int C = m->C;
    std::vector<float> dP((size_t)m->hops[0].n_dst * C, 0.f);
    std::vector<double> rowloss(n_seeds);
    const float inv_bt = 1.0f / (float)b_total;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_seeds; ++i) {
        const float* z = Pre[L - 1].data() + i * C;
        const int yi = m->y[seeds[i]];
        float mx = z[0];
        for (int c = 1; c < C; ++c) mx = std::max(mx, z[c]);
        double s = 0.0;
        for (int c = 0; c < C; ++c) s += std::exp((double)z[c] - mx);
        rowloss[i] = (double)mx + std::log(s) - (double)z[yi];
        for (int c = 0; c < C; ++c)
            dP[i * C + c] = ((float)(std::exp((double)z[c] - mx) / s) - (c == yi ? 1.f : 0.f)) * inv_bt;
    }
    if (loss_out) {
        double tot = 0.0;
        for (int32_t i = 0; i < n_seeds; ++i) tot += rowloss[i];
        *loss_out = (float)(tot / b_total);
    }
    // ---- backward
    for (int l = L - 1; l >= 0; --l) {
        const Block& b = m->hops[L - 1 - l];
        const Layer& ly = m->layers[l];
        gemm_tn(A[l].data(), dP.data(), grads_out + ly.off, b.n_dst, ly.rows, ly.out);   // dW = A^T dPre
        if (l == 0) break;
        std::vector<float> dA((size_t)b.n_dst * ly.rows);
        gemm_nt(dP.data(), m->W.data() + ly.off, dA.data(), b.n_dst, ly.out, ly.rows);   // dA = dPre W^T
        // dH_{l-1} = self part + Â^T (neighbour part), gathered per source over the transposed block
        const int in = ly.in;
        const bool sage = m->model == GNNH_SAGE_MEAN;
        std::vector<int32_t> tptr(b.n_src + 1, 0), tdst(b.rowptr[b.n_dst]), tedge(b.rowptr[b.n_dst]);
        for (int32_t e = 0; e < b.rowptr[b.n_dst]; ++e) ++tptr[b.col[e] + 1];
        for (int32_t u = 0; u < b.n_src; ++u) tptr[u + 1] += tptr[u];
        {
            std::vector<int32_t> cur(tptr.begin(), tptr.end() - 1);
            for (int32_t v = 0; v < b.n_dst; ++v)   // ascending (dst, edge): a fixed order per source
                for (int32_t e = b.rowptr[v]; e < b.rowptr[v + 1]; ++e) {
                    const int32_t q = cur[b.col[e]]++;
                    tdst[q] = v;
                    tedge[q] = e;
                }
        }
        std::vector<float> dPn((size_t)b.n_src * in);
        const std::vector<float>& Hp = H[l];   // ReLU output of layer l-1 (its mask: H > 0)
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t u = 0; u < b.n_src; ++u) {
            float* o = dPn.data() + u * in;
            std::fill(o, o + in, 0.f);
            if (u < b.n_dst) {
                const float* ds = dA.data() + u * ly.rows;
                if (sage) for (int c = 0; c < in; ++c) o[c] = ds[c];
                else for (int c = 0; c < in; ++c) o[c] = wS[l][u] * ds[c];
            }
            for (int32_t q = tptr[u]; q < tptr[u + 1]; ++q) {
                const float* dm = dA.data() + (int64_t)tdst[q] * ly.rows + (sage ? in : 0);
                const float w = wE[l][tedge[q]];
                for (int c = 0; c < in; ++c) o[c] += w * dm[c];
            }
            const float* hp = Hp.data() + u * in;
            for (int c = 0; c < in; ++c) o[c] = hp[c] > 0.f ? o[c] : 0.f;
        }
        dP.swap(dPn);
    }
    return GNNH_OK;
}

int gnnh_apply(gnnh_model* m, const float* grads, int64_t n) {
    if (!m || !grads) return fail(GNNH_ERR_PARAM, "NULL argument");
    if (n != (int64_t)m->W.size()) return fail(GNNH_ERR_SHAPE, "n != param_count");
    const float neg = -m->lr;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) m->W[i] = std::fmaf(neg, grads[i], m->W[i]);
    return GNNH_OK;
}

int gnnh_last_src_ids(const gnnh_model* m, int32_t hop, int32_t* out, int64_t cap, int64_t* n_out) {
    if (!m || !n_out || (cap > 0 && !out)) return fail(GNNH_ERR_PARAM, "NULL argument");
    if (hop < 0 || hop >= (int32_t)m->hops.size()) return fail(GNNH_ERR_RANGE, "hop out of range");
    const Block& b = m->hops[hop];
    *n_out = b.n_src;
    std::memcpy(out, b.src.data(), sizeof(int32_t) * std::min<int64_t>(cap, b.n_src));
    return GNNH_OK;
}

}  // extern "C"
