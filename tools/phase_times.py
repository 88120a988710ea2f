"""Per-phase times of the persistent sampling kernel (globaltimer at each grid barrier)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from gnn_inputs import WORKLOADS, build_inputs
from paper_2403_17092_b200 import Graph, Model
w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "products"]
inp = build_inputs(w)
g = Graph(inp["row_ptr"], inp["col"], inp["X"], inp["y"], w.num_classes, feat_dim=w.feat_dim)
m = Model(g, model=w.model, sampler=w.sampler, num_layers=w.num_layers, hidden=w.hidden, batch_size=w.batch_size,
          fanouts=w.fanouts, lr=w.lr, seed=w.sampler_seed, init_seed=w.init_seed)
m.set_train_nodes(inp["train"]); m.set_params(inp["params"])
acc = []
for s in range(12):
    m.train_minibatch(0, s)
    if s >= 2:
        acc.append(m.sampling_phases_us())
a = np.mean(acc, axis=0)
print("phase us:", np.round(a, 1).tolist(), "total", round(float(a.sum()), 1))
print("sizes", m.last_sizes())
