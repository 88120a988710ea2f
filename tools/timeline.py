"""Step timeline of the overlapped training loop (GS_TIMELINE=1): when each batch's sampling
kernel runs relative to the training graph it overlaps.  Diagnostics only.

  GS_TIMELINE=1 python tools/timeline.py [config] [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

os.environ["GS_TIMELINE"] = "1"
from gnn_inputs import WORKLOADS, build_inputs  # noqa: E402
from paper_2403_17092_b200 import Graph, Model, lib  # noqa: E402
from paper_2403_17092_b200.gnnstep import _check, _ptr  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "products"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
w = WORKLOADS[name]
inp = build_inputs(w)
g = Graph(inp["row_ptr"], inp["col"], inp["X"], inp["y"], w.num_classes, feat_dim=w.feat_dim)
m = Model(g, model=w.model, sampler=w.sampler, num_layers=w.num_layers, hidden=w.hidden, batch_size=w.batch_size,
          fanouts=w.fanouts, lr=w.lr, seed=w.sampler_seed, init_seed=w.init_seed)
m.set_train_nodes(inp["train"])
m.set_params(inp["params"])
buf = np.zeros(4 * 4096 + 1, np.float32)
for s in range(20):
    m.train_minibatch(0, s, sync=False)
m.synchronize()
_check(lib().gnn_debug_get(m.h, 10, _ptr(buf), buf.shape[0]))
for s in range(20, 20 + steps):
    m.train_minibatch(0, s, sync=False)
m.synchronize()
_check(lib().gnn_debug_get(m.h, 10, _ptr(buf), buf.shape[0]))
k = int(buf[0])
t = buf[1:1 + 4 * k].reshape(k, 4)
print("step  samp_start samp_end  train_start train_end | samp_dur train_dur gap(train_start - prev train_end)")
for i in range(k):
    gap = t[i, 2] - t[i - 1, 3] if i else 0.0
    print(f"{i:4d} {t[i,0]:10.1f} {t[i,1]:9.1f} {t[i,2]:10.1f} {t[i,3]:9.1f} | {t[i,1]-t[i,0]:8.1f} {t[i,3]-t[i,2]:8.1f} {gap:8.1f}")
d = np.diff(t[:, 2])
print(f"mean step (train start to start) {d.mean():.1f} us; mean sampling {np.mean(t[:,1]-t[:,0]):.1f} us; "
      f"mean training span {np.mean(t[:,3]-t[:,2]):.1f} us")
