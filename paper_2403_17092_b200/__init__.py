"""B200-native (sm_100a) per-mini-batch GNN training step of arXiv 2403.17092.

The product is the C-ABI library libgnnstep.so (include/gnnstep.h, sources in csrc/);
this package is its thin Python binding.  No CPU fallback exists.
"""
from .gnnstep import (Graph, Model, GnnError, comm_get_unique_id, lib, KERNEL_IDS, plan_step,  # noqa: F401
                      steps_per_epoch, ShardedGraph, shard_rows, plan_balanced,
                      cache_plan_by_degree, DeviceGraph)

__all__ = ["Graph", "Model", "GnnError", "comm_get_unique_id", "lib", "KERNEL_IDS"]
