import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from oracle import sampling as OS
from tests.gpu_common import inputs_for, make_gpu, rel
w, inp, graph = inputs_for("tiny")
g, m = make_gpu(w, inp, use_graph=True)
params = inp["params"].astype(np.float64)
perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
for step in range(w.n_batches):
    loss = m.train_minibatch(0, step)
    out = oracle.train_step(w, graph, params, 0, step, 1, perm=perm)
    b = len(OS.batch_seeds(perm, w.batch_size, step))
    gg = m.grads(); og = out["grad"]
    # per layer
    n1 = 2*32*32
    if rel(gg, og) > 1e-5 or step > 150: print(step, f"loss {abs(loss-out['loss'])/abs(out['loss']):.2e} logits {rel(m.logits(b, w.num_classes), out['logits'][0]):.2e} grad {rel(gg, og):.2e} L1 {rel(gg[:n1], og[:n1]):.2e} L2 {rel(gg[n1:], og[n1:]):.2e} p {rel(m.get_params(), out['params']):.2e}")
    params = out["params"]
