/* gnnhost — the host-core trainer rank of the Unified CPU-GPU protocol (SURVEY.md §8(f) NEXT-4,
 * PAPER.md §3: "The CPU Process is responsible for executing GNN operations, such
 * as sampling and model propagation ... each CPU and GPU Process generates a local gradient; the
 * local gradients are then gathered to perform a synchronous stochastic gradient descent").
 *
 * A C++/OpenMP implementation of the same per-mini-batch step as libgnnstep.so (neighbour
 * sampling with the Philox counter RNG of DESIGN.md R3/R4, relabel R6, GraphSAGE-mean or GCN
 * aggregation R11/R12, dense update, softmax cross-entropy R15, the exact backward) on the
 * host's cores, in fp32.  It computes a rank's gradient; the caller all-reduces it with the GPU
 * ranks (torch.distributed gloo; libgnnstep's GNN_EXCH_HOST mode) and applies the update here
 * with gnnh_apply (W <- W - lr G as one fused multiply-add per weight, the GPU update's
 * arithmetic, so the replicas stay bit-identical).  It is a trainer of its own, not a fallback:
 * libgnnstep.so never calls it.  Neighbour sampler only (ShaDow blocks are out of its scope).
 *
 * Conventions (as gnnstep.h): every call returns 0 (GNNH_OK) or a negative code, with a message
 * in gnnh_last_error(); inputs are host pointers; the graph arrays are BORROWED (they must stay
 * valid and unchanged until gnnh_destroy); outputs go into caller buffers of the stated size.
 */
#ifndef GNNHOST_H
#define GNNHOST_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { GNNH_OK = 0, GNNH_ERR_RANGE = -1, GNNH_ERR_PARAM = -2, GNNH_ERR_SHAPE = -3, GNNH_ERR_CONFIG = -4,
       GNNH_ERR_OOM = -7 };
enum { GNNH_SAGE_MEAN = 0, GNNH_GCN = 1 };

typedef struct gnnh_model gnnh_model;
const char* gnnh_last_error(void);

/* Graph (CSR row_ptr int64[N+1], col int32[nnz], rows sorted ascending and duplicate-free;
 * features fp32 [N x feat_stride], the first feat_dim columns used; labels int32[N] in [0, C))
 * and model: model GNNH_SAGE_MEAN / GNNH_GCN, num_layers L (= number of fanouts), hidden width,
 * fanouts int32[L] input-layer-first (§5.1.2), lr, sampler seed.  Parameters
 * start at zero: set them with gnnh_set_params (the GPU ranks' initial parameters). */
int gnnh_create(int64_t num_nodes, const int64_t* row_ptr, const int32_t* col, const float* features,
                int32_t feat_dim, int32_t feat_stride, const int32_t* labels, int32_t num_classes,
                int32_t model, int32_t num_layers, int32_t hidden, const int32_t* fanouts, float lr,
                uint64_t seed, gnnh_model** out);
int gnnh_destroy(gnnh_model* m);
int64_t gnnh_param_count(const gnnh_model* m);   /* the flat layout of gnnstep.h's params */
int gnnh_set_params(gnnh_model* m, const float* params, int64_t n);
int gnnh_get_params(const gnnh_model* m, float* params_out, int64_t n);

/* The epoch's seed order (R7): ids sorted by (Philox key64(id, epoch), id). */
int gnnh_epoch_permutation(const gnnh_model* m, const int32_t* train_ids, int64_t n, int64_t epoch,
                           int32_t* perm_out);

/* One mini-batch on the host cores: sample the L hops from `seeds` (int32[n_seeds], distinct
 * node ids; the Philox counter uses batch id g and `epoch`), forward, loss, backward.
 * grads_out: fp32[param_count], the gradient of Σ_i ℓ_i / b_total over this rank's seeds
 * (b_total = the seeds of the whole synchronous step, over every rank); loss_out (nullable):
 * Σ_i ℓ_i / b_total.  n_seeds = 0 writes a zero gradient (an inactive rank).
 * RANGE for a seed outside [0, N); PARAM for b_total < n_seeds or a repeated seed. */
int gnnh_grads(gnnh_model* m, const int32_t* seeds, int32_t n_seeds, int32_t b_total, int64_t epoch, int64_t g,
               float* grads_out, float* loss_out);

/* W <- W - lr * G (fmaf(-lr, G, W) per weight). */
int gnnh_apply(gnnh_model* m, const float* grads, int64_t n);

/* Parity hook: the source ids of hop h (seeds outward) of the last gnnh_grads call, int32;
 * *n_out = n_src of that hop; BUFFER-free: copies min(cap, n_src). */
int gnnh_last_src_ids(const gnnh_model* m, int32_t hop, int32_t* out, int64_t cap, int64_t* n_out);

#ifdef __cplusplus
}
#endif
#endif
