"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

NEXT-3: the paper's Dynamic Load Balancer (§4)
re-aimed at homogeneous trainers.

  workload(sample)  "the total number of aggregations that need to be performed using the
                    computational graph of the mini-batches" (line 285): the edges of the
                    block each layer aggregates over, summed over the layers.
  plan(work, P)     "sorts the mini-batches by their estimated workload" (line 287) and assigns
                    them: consecutive groups of P (heaviest first, ties by batch index) form one
                    synchronous step, so the ranks of a step carry similar work; steps ordered by
                    their smallest batch index, the ragged (lightest) group last.
  makespan          Σ over steps of the slowest rank's work (sync SGD waits for it).
"""
from __future__ import annotations

import numpy as np

from . import model


def workload(sample, sampler: str, num_layers: int) -> int:
    blocks, _ = model.layer_blocks(sample, sampler, num_layers)
    return int(sum(b["n_edges"] for b in blocks))


def plan(work, world: int) -> list:
    n = len(work)
    idx = sorted(range(n), key=lambda i: (-int(work[i]), i))
    groups = [idx[s * world:(s + 1) * world] for s in range((n + world - 1) // world)]
    full = [gr for gr in groups if len(gr) == world]
    ragged = [gr for gr in groups if len(gr) < world]
    full.sort(key=min)
    order = []
    for gr in full + ragged:
        order.extend(gr)
    return order


def makespan(order, work, world: int) -> int:
    return int(sum(max(int(work[b]) for b in order[s:s + world]) for s in range(0, len(order), world)))
