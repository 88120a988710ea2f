"""Transposed rows longer than the sampling kernel's shared-memory sort buffer (8192 entries,
sample_step.cu: the rank-counting fallback) on a star graph: node 0 joined to 20000 leaves, a
batch of 9000 leaves, so hop 0's transposed row of the centre holds 9000 destinations.  Sampling
bit-exact against the oracle and one training step (whose backward aggregation walks that sorted
row) within 1e-4 of the oracle, for GraphSAGE and GCN."""
import dataclasses

import numpy as np
import pytest

import oracle
from oracle import sampling as OS
from gnn_inputs import WORKLOADS
from gnn_inputs.synth import make_features, make_labels, make_params
from tests.gpu_common import assert_blocks_equal, check_train_step, make_gpu

pytestmark = pytest.mark.gpu

LEAVES = 20_000


def star_inputs(w):
    n = LEAVES + 1
    row_ptr = np.zeros(n + 1, np.int64)
    row_ptr[1] = LEAVES
    row_ptr[2:] = LEAVES + np.arange(1, n, dtype=np.int64)
    col = np.concatenate([np.arange(1, n, dtype=np.int32), np.zeros(LEAVES, np.int32)])
    X = make_features(n, w.feat_dim, w.graph_seed, w.feat_stride)
    y = make_labels(n, w.num_classes, w.graph_seed)
    train = np.arange(1, n, dtype=np.int32)
    return dict(row_ptr=row_ptr, col=col, X=X, y=y, train=train, params=make_params(w.dims, w.model, w.init_seed))


@pytest.mark.parametrize("model", ["sage", "gcn"])
def test_hub_row_longer_than_sort_buffer(model):
    w = dataclasses.replace(WORKLOADS["tiny"], name="star", num_nodes=LEAVES + 1, nnz=2 * LEAVES, model=model,
                            fanouts=(3, 2), batch_size=9000, n_train=LEAVES)
    inp = star_inputs(w)
    graph = dict(row_ptr=inp["row_ptr"], col=inp["col"], X=inp["X"][:, :w.feat_dim], y=inp["y"], train=inp["train"])
    g, m = make_gpu(w, inp)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    want, _ = oracle.sample_batch(w, graph, 0, 0, perm)
    got = m.sample(0, 0)
    assert_blocks_equal(got, want)
    assert np.bincount(want[0]["blk_col"]).max() > 8192   # the centre's transposed row
    loss = m.train_minibatch(0, 0)
    check_train_step(m, w, graph, inp["params"].astype(np.float64), 0, 0, perm, loss)
