"""A few tiny steps of every kernel family under compute-sanitizer (memcheck / racecheck /
synccheck): SAGE + neighbour (sampling kernel, layer-1 bulk-copy gather, tcgen05 GEMMs, fused CE,
backward, SGD), GCN + neighbour, GCN + ShaDow (balanced aggregation), the NCCL exchange branch.

  compute-sanitizer --tool racecheck python tools/sanitize.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from gnn_inputs import WORKLOADS, build_inputs  # noqa: E402
from paper_2403_17092_b200 import Graph, Model  # noqa: E402


def run(name, steps=2, exchange="auto", use_graph=False):
    w = WORKLOADS[name]
    inp = build_inputs(w)
    g = Graph(inp["row_ptr"], inp["col"], inp["X"], inp["y"], w.num_classes, feat_dim=w.feat_dim)
    m = Model(g, model=w.model, sampler=w.sampler, num_layers=w.num_layers, hidden=w.hidden,
              batch_size=w.batch_size, fanouts=w.fanouts, use_graph=use_graph, lr=w.lr,
              seed=w.sampler_seed, init_seed=w.init_seed)
    m.set_train_nodes(inp["train"])
    m.set_params(inp["params"])
    if exchange != "auto":
        m.set_exchange(exchange)
    for s in range(steps):
        loss = m.train_minibatch(0, s)
    m.sample(0, 3)
    print(name, exchange, "loss", loss, flush=True)
    m.close()
    g.close()


if __name__ == "__main__":
    run("tiny")
    run("tiny", exchange="nccl")
    run("tiny_gcn")
    run("tiny_shadow_l5")
