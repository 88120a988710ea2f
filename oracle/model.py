"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Dense half of the step in float64 numpy (DESIGN.md oracle steps O4-O9), written as
the plain definitions, in the paper's notation:

  O4 gather        X_in = H^0[src ids of the layer-1 block]            (§2.2 l.160)
                   (H^0 an array, or a function of the row ids: the formula-recompute mode)
  O5 forward       GCN   H^(l) = σ(Â H^(l-1) W^(l))                     (Eq. 1, l.131-137)
                   SAGE  H^(l) = σ(H^(l-1) W_1 + Â H^(l-1) W_2)         (Eq. 2, l.139-142)
                   σ = ReLU for l < L, identity at l = L                (R14)
  O6 loss          mean softmax cross-entropy over the batch           (Eq. 3, l.161-165; R15)
  O7 backward      exact reverse-mode of O5/O6
  O8 allreduce     G = Σ_p G_p with each G_p already divided by b_total (§2.2 l.173-175; R9)
  O9 SGD           W <- W - lr G                                        (§2.2 l.157-158; R16)

Â (R11/R12):
  SAGE-mean: Â[v,u] = (#edges u->v) / deg_blk(v); row of a degree-0 node is 0.
  GCN:       Â[v,u] = Σ_{edges u->v} 1/sqrt(d_in(v) d_out(u)) + [u = v < n_dst]/sqrt(d_in(v) d_out(v)),
             d_in(v) = deg_blk(v) + 1, d_out(u) = outdeg_blk(u) + [u < n_dst].
Sparse products use scipy.sparse (a library matmul, as a step), everything in fp64.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


# ---------------------------------------------------------------- params layout
def layer_shapes(dims, model):
    """(rows, cols) of each layer's weight block in the flat parameter vector."""
    return [((2 if model == "sage" else 1) * dims[l], dims[l + 1]) for l in range(len(dims) - 1)]


def unflatten(flat, dims, model):
    Ws, off = [], 0
    for r, c in layer_shapes(dims, model):
        Ws.append(np.asarray(flat[off:off + r * c], dtype=np.float64).reshape(r, c))
        off += r * c
    assert off == len(flat)
    return Ws


def flatten(Ws):
    return np.concatenate([W.reshape(-1) for W in Ws])


# ---------------------------------------------------------------- Â
def normalized_adjacency(block, model):
    nd, ns = block["n_dst"], block["n_src"]
    rp = np.asarray(block["blk_rowptr"], dtype=np.int64)
    col = np.asarray(block["blk_col"], dtype=np.int64)
    deg = np.diff(rp)
    rows = np.repeat(np.arange(nd), deg)
    if model == "sage":
        w = 1.0 / deg[rows].astype(np.float64) if rows.size else np.zeros(0)
        return sp.csr_matrix((w, (rows, col)), shape=(nd, ns))
    d_in = deg.astype(np.float64) + 1.0
    outdeg = np.bincount(col, minlength=ns).astype(np.float64)
    d_out = outdeg + (np.arange(ns) < nd)
    w = 1.0 / np.sqrt(d_in[rows] * d_out[col])
    self_r = np.arange(nd)
    self_w = 1.0 / np.sqrt(d_in[self_r] * d_out[self_r])
    return sp.csr_matrix((np.concatenate([w, self_w]),
                          (np.concatenate([rows, self_r]), np.concatenate([col, self_r]))),
                         shape=(nd, ns))


# ---------------------------------------------------------------- O5
def forward(Ws, model, blocks, X_in):
    """blocks: per layer l = 1..L (input-first).  Returns cache with A_l (GEMM operand),
    Pre_l, H_l and the Â used per layer."""
    H = np.asarray(X_in, dtype=np.float64)
    L = len(blocks)
    cache = dict(A=[], Pre=[], H=[H], Ahat=[])
    for l in range(L):
        blk = blocks[l]
        assert H.shape[0] == blk["n_src"], (H.shape, blk["n_src"])
        Ahat = normalized_adjacency(blk, model)
        agg = Ahat @ H
        if model == "sage":
            A = np.concatenate([H[:blk["n_dst"]], agg], axis=1)
        else:
            A = agg
        Pre = A @ Ws[l]
        H = np.maximum(Pre, 0.0) if l < L - 1 else Pre
        cache["A"].append(A)
        cache["Pre"].append(Pre)
        cache["H"].append(H)
        cache["Ahat"].append(Ahat)
    return cache


# ---------------------------------------------------------------- O6
def cross_entropy(Z, y, b_total):
    """ℓ_i = logsumexp(z_i) - z_{i,y_i}; rank loss = Σℓ_i / b_total; dZ = (softmax - onehot)/b_total."""
    Z = np.asarray(Z, dtype=np.float64)
    m = Z.max(axis=1, keepdims=True) if Z.shape[0] else np.zeros((0, 1))
    lse = m[:, 0] + np.log(np.exp(Z - m).sum(axis=1)) if Z.shape[0] else np.zeros(0)
    ell = lse - Z[np.arange(Z.shape[0]), y]
    P = np.exp(Z - lse[:, None]) if Z.shape[0] else Z
    dZ = P.copy()
    dZ[np.arange(Z.shape[0]), y] -= 1.0
    return ell.sum() / b_total, dZ / b_total


# ---------------------------------------------------------------- O7
def relu_mask(Pre, override=None):
    """[Pre > 0] (ReLU'(0) = 0).  `override` = (rows, cols, values) replaces the decision at
    kink-ambiguous units (|Pre| within the fp32 error of the GEMM, R27): there
    either decision is a correct result, the caller validates which one it supplies."""
    mask = Pre > 0.0
    if override is not None:
        r, c, v = override
        mask[r, c] = v
    return mask


def backward(Ws, model, blocks, cache, dZ, mask_override=None):
    L = len(blocks)
    grads = [None] * L
    dPre = np.zeros_like(cache["Pre"][L - 1])
    dPre[:dZ.shape[0]] = dZ
    for l in range(L - 1, -1, -1):
        A = cache["A"][l]
        grads[l] = A.T @ dPre
        if l == 0:
            break
        dA = dPre @ Ws[l].T
        blk = blocks[l]
        Ahat = cache["Ahat"][l]
        if model == "sage":
            fin = Ws[l].shape[0] // 2
            dSelf, dM = dA[:, :fin], dA[:, fin:]
            dH = Ahat.T @ dM
            dH[:blk["n_dst"]] += dSelf
        else:
            dH = Ahat.T @ dA
        ovr = mask_override.get(l - 1) if mask_override else None
        dPre = dH * relu_mask(cache["Pre"][l - 1], ovr)
    return grads


# ---------------------------------------------------------------- batch assembly
def layer_blocks(sample, sampler, num_layers):
    """Neighbour: layer l uses hop L-l.  ShaDow: every layer uses the induced block."""
    if sampler == "neighbor":
        hops = sample
        L = len(hops)
        blocks = [hops[L - 1 - l] for l in range(L)]
        return blocks, blocks[0]["src_ids"]
    hops, block = sample
    return [block] * num_layers, block["src_ids"]


def minibatch_grad(Ws, model, blocks, input_ids, X, labels, b, b_total, mask_override=None):
    """One rank's O4-O7: returns (rank loss, list of dW, cache)."""
    ids = np.asarray(input_ids, dtype=np.int64)
    # formula-recompute mode (configs[4]: the 57 GB table is never materialised on the host): X is
    # a function returning the feature rows of the given ids (gnn_inputs.feature_rows)
    X_in = np.asarray(X(ids), dtype=np.float64) if callable(X) else np.asarray(X, dtype=np.float64)[ids]
    cache = forward(Ws, model, blocks, X_in)
    Z = cache["H"][-1][:b]
    loss, dZ = cross_entropy(Z, labels, b_total)
    grads = backward(Ws, model, blocks, cache, dZ, mask_override)
    return loss, grads, cache


def sgd(Ws, G, lr):
    """O9."""
    return [W - lr * g for W, g in zip(Ws, G)]


def adam(Ws, G, state, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """NEXT-4: Adam, the optimizer of the paper's training listings
    (`torch.optim.Adam(...)`; standard defaults,
    no weight decay, no amsgrad).  Kingma & Ba, Algorithm 1, as torch.optim.Adam states it:
        t <- t + 1;  m <- b1 m + (1 - b1) g;  v <- b2 v + (1 - b2) g^2
        W <- W - lr * (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)
    `state` = dict(t, m, v) (m, v lists like Ws, zero at t = 0); updated in place."""
    if not state:
        state.update(t=0, m=[np.zeros_like(W) for W in Ws], v=[np.zeros_like(W) for W in Ws])
    state["t"] += 1
    t = state["t"]
    bc1, bc2 = 1.0 - beta1 ** t, 1.0 - beta2 ** t
    out = []
    for i, (W, g) in enumerate(zip(Ws, G)):
        state["m"][i] = beta1 * state["m"][i] + (1.0 - beta1) * g
        state["v"][i] = beta2 * state["v"][i] + (1.0 - beta2) * g * g
        out.append(W - lr * (state["m"][i] / bc1) / (np.sqrt(state["v"][i] / bc2) + eps))
    return out


def allreduce(rank_grads):
    """O8: Σ_p G_p in rank order."""
    out = [np.zeros_like(g) for g in rank_grads[0]]
    for G in rank_grads:
        for i, g in enumerate(G):
            out[i] = out[i] + g
    return out
