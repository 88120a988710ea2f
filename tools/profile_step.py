"""Run a few training steps of a workload for Nsight Compute (kernels of the profiled steps
are inside an NVTX range "steps").  Not a benchmark: timings under ncu are not bench values.

  ncu --nvtx --nvtx-include "steps/" ... python tools/profile_step.py --config products
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from gnn_inputs import WORKLOADS, build_inputs  # noqa: E402
from paper_2403_17092_b200 import Graph, Model  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="products")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--graph", action="store_true")
    ap.add_argument("--precision", default="fp32")
    a = ap.parse_args()
    w = WORKLOADS[a.config]
    inp = build_inputs(w)
    g = Graph(inp["row_ptr"], inp["col"], inp["X"], inp["y"], w.num_classes, feat_dim=w.feat_dim)
    m = Model(g, model=w.model, sampler=w.sampler, num_layers=w.num_layers, hidden=w.hidden,
              batch_size=w.batch_size, fanouts=w.fanouts, precision=a.precision, use_graph=a.graph,
              lr=w.lr, seed=w.sampler_seed, init_seed=w.init_seed)
    m.set_train_nodes(inp["train"])
    m.set_params(inp["params"])
    for s in range(a.warmup):
        m.train_minibatch(0, s)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("steps")
    for s in range(a.warmup, a.warmup + a.steps):
        m.train_minibatch(0, s, sync=False)
    m.synchronize()
    torch.cuda.nvtx.range_pop()
    print("sizes", m.last_sizes())


if __name__ == "__main__":
    main()
