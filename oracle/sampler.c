/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded C implementation of the integer half of the
 * per-mini-batch step (DESIGN.md oracle steps O0-O3).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load this library.  It shares no code, header, table or constant generator with
 * the CUDA path in paper_2403_17092_b200/csrc; neither includes the other.
 *
 *   O0 philox4x32-10 counter RNG          (§2.2 "randomly selects";
 *                                          DESIGN.md readings R3/R4: counter-based,
 *                                          Random123 Philox4x32-10)
 *   O1 epoch permutation + batching       (§2.2 "a batch of vertices";
 *                                          SPEC.md partition_seeds lines 107-115)
 *   O2 neighbour sampling + relabel       (§2.2; §5.1.2;
 *                                          SPEC.md neighbor_sample lines 117-125)
 *   O3 ShaDow induced subgraph            (§2.2; §5.3;
 *                                          SPEC.md shadow_sample lines 127-135)
 *
 * Every loop follows the step list in DESIGN.md "Oracle" in the stated order.
 * Error convention: return 0 on success, negative on a capacity/argument error.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------- O0: Philox4x32 (R rounds; R = 10 for the method) ---------------- */
void oracle_philox4x32(const uint32_t ctr[4], const uint32_t key[2], int rounds, uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < rounds; ++r) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }   /* key bump before rounds 2..R */
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* The method's draw: word (draw & 3) of Philox at
 *   ctr = (a, b, tag<<28 | (epoch & 0xFFFFF)<<8 | (hop & 0xFF), draw >> 2),
 *   key = (seed & 0xffffffff, seed >> 32)                         (R3)   */
static uint32_t draw_word(uint64_t seed, uint32_t tag, uint32_t a, uint32_t b,
                          int64_t epoch, int32_t hop, uint32_t draw)
{
    uint32_t key[2] = { (uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32) };
    uint32_t ctr[4] = { a, b,
                        (tag << 28) | ((uint32_t)(epoch & 0xFFFFF) << 8) | ((uint32_t)hop & 0xFFu),
                        draw >> 2 };
    uint32_t out[4];
    oracle_philox4x32(ctr, key, 10, out);
    return out[draw & 3];
}

/* ---------------- O1: epoch permutation ---------------- */
typedef struct { uint64_t key; int32_t id; } keyed_t;

static int cmp_keyed(const void* a, const void* b)
{
    const keyed_t* x = (const keyed_t*)a; const keyed_t* y = (const keyed_t*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    if (x->id != y->id) return x->id < y->id ? -1 : 1;
    return 0;
}

/* perm = train ids sorted by (key64(v), v), key64 = (w0<<32)|w1 of Philox tag 1 at (v, 0, epoch). */
int oracle_epoch_perm(const int32_t* train, int64_t n, uint64_t seed, int64_t epoch, int32_t* perm)
{
    if (n < 0) return -1;
    keyed_t* t = (keyed_t*)malloc(sizeof(keyed_t) * (size_t)(n > 0 ? n : 1));
    if (!t) return -2;
    for (int64_t i = 0; i < n; ++i) {
        uint32_t v = (uint32_t)train[i];
        uint64_t w0 = draw_word(seed, 1u, v, 0u, epoch, 0, 0u);
        uint64_t w1 = draw_word(seed, 1u, v, 0u, epoch, 0, 1u);
        t[i].key = (w0 << 32) | w1;
        t[i].id = train[i];
    }
    qsort(t, (size_t)n, sizeof(keyed_t), cmp_keyed);
    for (int64_t i = 0; i < n; ++i) perm[i] = t[i].id;
    free(t);
    return 0;
}

/* ---------------- O2: one row, Floyd's k-of-d selection ---------------- */
static int cmp_i64(const void* a, const void* b)
{
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* Positions (ascending) of the neighbours node v keeps at hop `hop` of batch g.
 * d <= k: all positions 0..d-1 (no draws).  Else Floyd: for i = 0..k-1, j = d-k+i,
 * t = floor(r_i * (j+1) / 2^32); add (t already chosen ? j : t).  Returns count. */
int oracle_sample_row(uint64_t seed, int64_t epoch, int64_t g, int32_t hop,
                      int32_t v, int64_t d, int32_t k, int64_t* pos)
{
    if (d <= (int64_t)k) {
        for (int64_t i = 0; i < d; ++i) pos[i] = i;
        return (int)d;
    }
    for (int32_t i = 0; i < k; ++i) {
        int64_t j = d - k + i;
        uint32_t r = draw_word(seed, 0u, (uint32_t)v, (uint32_t)g, epoch, hop, (uint32_t)i);
        int64_t t = (int64_t)(((uint64_t)r * (uint64_t)(j + 1)) >> 32);
        int seen = 0;
        for (int32_t q = 0; q < i; ++q) if (pos[q] == t) { seen = 1; break; }
        pos[i] = seen ? j : t;
    }
    qsort(pos, (size_t)k, sizeof(int64_t), cmp_i64);
    return k;
}

/* ---------------- O2: relabel helpers ---------------- */
static int cmp_i32(const void* a, const void* b)
{
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

typedef struct { int32_t id; int32_t idx; } idpair_t;

static int cmp_idpair(const void* a, const void* b)
{
    const idpair_t* x = (const idpair_t*)a; const idpair_t* y = (const idpair_t*)b;
    return (x->id > y->id) - (x->id < y->id);
}

static int64_t find_pair(const idpair_t* arr, int64_t n, int32_t id)
{
    int64_t lo = 0, hi = n - 1;
    while (lo <= hi) {
        int64_t mid = (lo + hi) / 2;
        if (arr[mid].id == id) return arr[mid].idx;
        if (arr[mid].id < id) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

static int64_t find_i32(const int32_t* arr, int64_t n, int32_t id)
{
    int64_t lo = 0, hi = n - 1;
    while (lo <= hi) {
        int64_t mid = (lo + hi) / 2;
        if (arr[mid] == id) return mid;
        if (arr[mid] < id) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

/* ---------------- O2: multi-hop neighbour sampling of one batch ----------------
 * dst_0 = seeds; hop h = 0..L-1 samples k = fanouts[L-1-h] per dst node;
 * blk_rowptr = exclusive scan of row counts; blk_nbr = concatenation;
 * src_h = dst_h ++ sorted(set(blk_nbr) - set(dst_h)); blk_col[e] = index of blk_nbr[e]
 * in src_h; dst_{h+1} = src_h.
 * Outputs per hop h (caller-allocated, capacities cap_src[h], cap_edges[h]):
 *   src_ids[h][n_src[h]], blk_rowptr[h][n_dst[h]+1], blk_col[h][n_edges[h]], blk_nbr[h][...]. */
int oracle_neighbor_sample(const int64_t* row_ptr, const int32_t* col, int64_t N,
                           const int32_t* seeds, int64_t n_seeds,
                           int32_t L, const int32_t* fanouts,
                           uint64_t seed, int64_t epoch, int64_t g,
                           const int64_t* cap_src, const int64_t* cap_edges,
                           int64_t* n_dst, int64_t* n_src, int64_t* n_edges,
                           int32_t* const* src_ids, int32_t* const* blk_rowptr,
                           int32_t* const* blk_col, int32_t* const* blk_nbr)
{
    const int32_t* dst = seeds;
    int64_t nd = n_seeds;
    for (int32_t h = 0; h < L; ++h) {
        int32_t k = fanouts[L - 1 - h];
        n_dst[h] = nd;
        /* step 2: per dst node, sampled neighbours in ascending CSR position */
        int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(k > 0 ? k : 1));
        int64_t e = 0;
        blk_rowptr[h][0] = 0;
        for (int64_t i = 0; i < nd; ++i) {
            int32_t v = dst[i];
            if (v < 0 || v >= N) { free(pos); return -3; }
            int64_t d = row_ptr[v + 1] - row_ptr[v];
            int cnt = oracle_sample_row(seed, epoch, g, h, v, d, k, pos);
            if (e + cnt > cap_edges[h]) { free(pos); return -4; }
            for (int q = 0; q < cnt; ++q) blk_nbr[h][e++] = col[row_ptr[v] + pos[q]];
            blk_rowptr[h][i + 1] = (int32_t)e;
        }
        free(pos);
        n_edges[h] = e;
        /* step 4: relabel */
        idpair_t* dsorted = (idpair_t*)malloc(sizeof(idpair_t) * (size_t)(nd > 0 ? nd : 1));
        for (int64_t i = 0; i < nd; ++i) { dsorted[i].id = dst[i]; dsorted[i].idx = (int32_t)i; }
        qsort(dsorted, (size_t)nd, sizeof(idpair_t), cmp_idpair);
        int32_t* uniq = (int32_t*)malloc(sizeof(int32_t) * (size_t)(e > 0 ? e : 1));
        memcpy(uniq, blk_nbr[h], sizeof(int32_t) * (size_t)e);
        qsort(uniq, (size_t)e, sizeof(int32_t), cmp_i32);
        int64_t nu = 0;
        for (int64_t i = 0; i < e; ++i)
            if (nu == 0 || uniq[nu - 1] != uniq[i]) uniq[nu++] = uniq[i];
        int64_t nnew = 0;
        for (int64_t i = 0; i < nu; ++i)          /* set difference, stays ascending */
            if (find_pair(dsorted, nd, uniq[i]) < 0) uniq[nnew++] = uniq[i];
        if (nd + nnew > cap_src[h]) { free(dsorted); free(uniq); return -5; }
        for (int64_t i = 0; i < nd; ++i) src_ids[h][i] = dst[i];
        for (int64_t i = 0; i < nnew; ++i) src_ids[h][nd + i] = uniq[i];
        n_src[h] = nd + nnew;
        for (int64_t i = 0; i < e; ++i) {
            int32_t u = blk_nbr[h][i];
            int64_t li = find_pair(dsorted, nd, u);
            if (li < 0) li = nd + find_i32(uniq, nnew, u);
            blk_col[h][i] = (int32_t)li;
        }
        free(dsorted); free(uniq);
        dst = src_ids[h];
        nd = n_src[h];
    }
    return 0;
}

/* ---------------- O3: induced subgraph over node set S ----------------
 * for i = 0..|S|-1, v = S[i], for each u in row v (CSR order) with u in S: edge local(u) -> i. */
int oracle_induce(const int64_t* row_ptr, const int32_t* col, int64_t N,
                  const int32_t* S, int64_t nS, int64_t cap_edges,
                  int32_t* ind_rowptr, int32_t* ind_col, int64_t* n_edges)
{
    idpair_t* ss = (idpair_t*)malloc(sizeof(idpair_t) * (size_t)(nS > 0 ? nS : 1));
    for (int64_t i = 0; i < nS; ++i) { ss[i].id = S[i]; ss[i].idx = (int32_t)i; }
    qsort(ss, (size_t)nS, sizeof(idpair_t), cmp_idpair);
    int64_t e = 0;
    ind_rowptr[0] = 0;
    for (int64_t i = 0; i < nS; ++i) {
        int32_t v = S[i];
        if (v < 0 || v >= N) { free(ss); return -3; }
        for (int64_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p) {
            int64_t li = find_pair(ss, nS, col[p]);
            if (li >= 0) {
                if (e >= cap_edges) { free(ss); return -4; }
                ind_col[e++] = (int32_t)li;
            }
        }
        ind_rowptr[i + 1] = (int32_t)e;
    }
    *n_edges = e;
    free(ss);
    return 0;
}
