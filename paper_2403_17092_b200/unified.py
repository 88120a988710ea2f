"""The Unified CPU-GPU protocol's synchronous step (§3, §4;
SURVEY.md §8(f) NEXT-4): every trainer process — GPU ranks (libgnnstep, GNN_EXCH_HOST) and host
ranks (libgnnhost) — computes the gradient of its own sub-batch, the gradients are summed by a
torch.distributed all-reduce over the host (gloo), and every rank applies the same update.

Sub-batch assignment (the paper's workload ratio, §4 "Static Load Balancing", lines 276-281): the
step's global mini-batch perm[s*T, (s+1)*T), T = Σ_r sizes[r], is cut into consecutive slices of
sizes[r] seeds, rank r's slice keyed by batch id g = s*world + r for the sampler's counter RNG.
With every size equal to the batch size this is the engine's own rule (g = s*world + r,
seeds = perm[g*B, (g+1)*B)).  Plumbing only: the arithmetic runs in the two libraries.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def ratio_sizes(batch_size: int, speeds) -> list[int]:
    """Sub-batch sizes by the workload ratio: the fastest rank takes a
    full batch (its capacity), every other rank batch_size * speed_r / speed_max seeds, at least
    one for a rank of nonzero speed.  speeds: mini-batches/s of each rank at the full batch."""
    sp = np.asarray(speeds, dtype=np.float64)
    top = sp.max()
    sizes = [batch_size if x == top else (max(1, int(batch_size * x / top)) if x > 0 else 0) for x in sp]
    return [int(v) for v in sizes]


def step_slice(perm: np.ndarray, sizes, step: int, rank: int):
    """(g, seeds, b_total) of `rank` at synchronous step `step`."""
    world = len(sizes)
    T = int(sum(sizes))
    base = step * T
    lo = base + int(sum(sizes[:rank]))
    seeds = perm[min(lo, len(perm)):min(lo + sizes[rank], len(perm))]
    b_total = max(0, min(len(perm), base + T) - min(len(perm), base))
    return step * world + rank, np.ascontiguousarray(seeds, dtype=np.int32), int(b_total)


def unified_step(trainer, perm, batch_size: int, epoch: int, step: int, rank: int, world: int, sizes=None):
    """One synchronous step of this rank: its gradient, the all-reduce (sum; gradients are
    already divided by the step's b_total), the update.  trainer: a HostModel or a GpuRank.
    Returns this rank's loss share (Σ_i ℓ_i / b_total over its seeds)."""
    sizes = sizes if sizes is not None else [batch_size] * world
    g, seeds, b_total = step_slice(perm, sizes, step, rank)
    grad, loss = trainer.grads(seeds, max(b_total, 1), epoch, g)
    t = torch.from_numpy(np.ascontiguousarray(grad, dtype=np.float32))
    dist.all_reduce(t)
    trainer.apply(t.numpy())
    return loss


class GpuRank:
    """A libgnnstep model as a Unified-protocol rank: its step stops at the reduced gradient
    (GNN_EXCH_HOST); apply() uploads the all-reduced gradient and runs the update kernel."""

    def __init__(self, model, rank: int, world: int):
        self.m = model
        model.set_rank(rank, world)
        model.set_exchange("host")

    def grads(self, seeds, b_total, epoch, g):
        loss = self.m.train_batch_host(seeds, b_total, epoch, g)
        return self.m.grads(), loss

    def apply(self, grad):
        self.m.apply_update(grad)
