"""ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of the per-mini-batch GNN
training step of arXiv 2403.17092 (§2.1 Eqs. 1-2, §2.2 Eq. 3, Neighbor /
ShaDow sampling, synchronous SGD), written from the paper and DESIGN.md's readings:

  oracle/sampler.c   O0 Philox, O1 epoch permutation, O2 neighbour sampling + relabel,
                     O3 ShaDow induce            (integer, exact)
  oracle/model.py    O4 gather .. O9 SGD          (float64 numpy / scipy.sparse)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import, call, link or execute anything under oracle/.  It shares no code with
the CUDA path (paper_2403_17092_b200/), and neither imports the other; the only
common dependency is the seeded input generator gnn_inputs/, which holds none of the
method's arithmetic.

Pins (tests/test_oracle_*.py, -m "not gpu"): Random123 Philox KAT vectors; a
hand-derived Floyd example; brute-force k-subset enumeration and χ² uniformity;
relabel/ShaDow definitional invariants and brute-force membership filter; dense Â
closed forms (mean, Kipf-Welling); loss invariants and torch CPU cross-entropy;
central finite differences for every weight; virtual-rank equivalence; SGD
arithmetic.  End-to-end values at products/Reddit scale are "parity unpinned"
beyond those piecewise pins (the paper prints no numeric example).
"""
from __future__ import annotations

import numpy as np

from . import sampling, model

__all__ = ["sampling", "model", "sample_batch", "train_step", "n_batches"]


def n_batches(n_train: int, batch_size: int) -> int:
    return (n_train + batch_size - 1) // batch_size


def sample_batch(w, graph, epoch: int, g: int, perm=None):
    """O1 + O2 (+ O3) for global batch g of `epoch`.  Returns (sample, seeds)."""
    if perm is None:
        perm = sampling.epoch_perm(graph["train"], w.sampler_seed, epoch)
    seeds = sampling.batch_seeds(perm, w.batch_size, g)
    if w.sampler == "neighbor":
        s = sampling.neighbor_sample(graph["row_ptr"], graph["col"], seeds, list(w.fanouts),
                                     w.sampler_seed, epoch, g)
    else:
        s = sampling.shadow_sample(graph["row_ptr"], graph["col"], seeds, list(w.fanouts),
                                   w.num_layers, w.sampler_seed, epoch, g)
    return s, seeds


def train_step(w, graph, params_flat, epoch: int, step: int, world: int, perm=None, X=None,
               lr=None, mask_override=None, keep_cache=False):
    """One synchronous-SGD step with `world` virtual ranks (O1-O9).
    Rank p trains global batch g = step*world + p (inactive if g >= n_batches).
    Returns dict(loss=global loss, rank_losses, rank_grads, grad (allreduced, flat),
    params (after SGD, flat), logits per rank)."""
    if perm is None:
        perm = sampling.epoch_perm(graph["train"], w.sampler_seed, epoch)
    X = graph["X"] if X is None else X
    lr = w.lr if lr is None else lr
    nb = n_batches(len(graph["train"]), w.batch_size)
    Ws = model.unflatten(params_flat, w.dims, w.model)
    gs = [step * world + p for p in range(world)]
    sizes = [len(sampling.batch_seeds(perm, w.batch_size, g)) if g < nb else 0 for g in gs]
    b_total = sum(sizes)
    rank_losses, rank_grads, logits, caches = [], [], [], []
    for p, g in enumerate(gs):
        if g >= nb:
            rank_losses.append(0.0)
            rank_grads.append([np.zeros_like(W) for W in Ws])
            logits.append(None)
            caches.append(None)
            continue
        s, seeds = sample_batch(w, graph, epoch, g, perm)
        blocks, input_ids = model.layer_blocks(s, w.sampler, w.num_layers)
        labels = graph["y"][seeds]
        ovr = mask_override[p] if mask_override else None
        loss, grads, cache = model.minibatch_grad(Ws, w.model, blocks, input_ids, X, labels,
                                                  len(seeds), b_total, ovr)
        caches.append(dict(cache, Ws=Ws) if keep_cache else None)
        rank_losses.append(loss)
        rank_grads.append(grads)
        logits.append(cache["H"][-1][:len(seeds)])
    G = model.allreduce(rank_grads)
    newW = model.sgd(Ws, G, lr)
    return dict(loss=float(sum(rank_losses)), rank_losses=rank_losses,
                rank_grads=[model.flatten(g) for g in rank_grads], grad=model.flatten(G),
                params=model.flatten(newW), logits=logits, b_total=b_total, caches=caches)
