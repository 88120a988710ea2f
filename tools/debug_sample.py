"""Sample a few batches of a workload through the C-ABI (for compute-sanitizer runs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gnn_inputs import WORKLOADS, build_inputs
from paper_2403_17092_b200 import Graph, Model
w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "tiny"]
inp = build_inputs(w)
g = Graph(inp["row_ptr"], inp["col"], inp["X"], inp["y"], w.num_classes, feat_dim=w.feat_dim)
m = Model(g, model=w.model, sampler=w.sampler, num_layers=w.num_layers, hidden=w.hidden, batch_size=w.batch_size,
          fanouts=w.fanouts, lr=w.lr, seed=w.sampler_seed, init_seed=w.init_seed, use_graph=False)
m.set_train_nodes(inp["train"]); m.set_params(inp["params"])
for b in range(3):
    m.sample(0, b)
    print("sampled", b, flush=True)
for s in range(3):
    print("loss", m.train_minibatch(0, s), flush=True)
