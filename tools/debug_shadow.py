"""Run a few ShaDow steps (compute-sanitizer target for the receptive-field compaction path)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.gpu_common import inputs_for, make_gpu  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "tiny_sage_shadow"
w, inp, graph = inputs_for(name)
g, m = make_gpu(w, inp, use_graph=False)
for s in range(2):
    print(name, s, m.train_minibatch(0, s), flush=True)
