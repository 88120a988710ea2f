"""Transposed rows longer than the sampling kernel's shared-memory sort buffer (8192 entries,
sample_step.cu: the rank-counting fallback).  A two-level star: 1024 leaves (the batch), each
joined to 10 middle nodes of its own, every middle node joined to one centre.  Hop 0 takes each
leaf's 10 middles, hop 1 each middle's leaf and the centre, so hop 1's transposed row of the centre
holds 10240 destinations.  Sampling bit-exact against the oracle and one training step (whose
backward aggregation walks that row) within 1e-4 of the oracle, for GraphSAGE and GCN (L = 3)."""
import dataclasses

import numpy as np
import pytest

import oracle
from oracle import sampling as OS
from gnn_inputs import WORKLOADS
from gnn_inputs.synth import make_features, make_labels, make_params
from tests.gpu_common import assert_blocks_equal, check_train_step, make_gpu

pytestmark = pytest.mark.gpu

LEAVES, ARMS = 1024, 10
MID = LEAVES * ARMS
CENTRE = LEAVES + MID
N = CENTRE + 1


def star_graph():
    rows = [[LEAVES + ARMS * i + j for j in range(ARMS)] for i in range(LEAVES)]
    rows += [[t // ARMS, CENTRE] for t in range(MID)]
    rows += [list(range(LEAVES, CENTRE))]
    row_ptr = np.zeros(N + 1, np.int64)
    row_ptr[1:] = np.cumsum([len(r) for r in rows])
    col = np.concatenate([np.asarray(r, np.int32) for r in rows])
    return row_ptr, col


def star_workload(model):
    return dataclasses.replace(WORKLOADS["tiny"], name="star2", num_nodes=N, nnz=2 * (MID + MID), model=model,
                               fanouts=(2, 2, ARMS), num_layers=3, batch_size=LEAVES, n_train=LEAVES)


def star_inputs(w):
    row_ptr, col = star_graph()
    X = make_features(N, w.feat_dim, w.graph_seed, w.feat_stride)
    y = make_labels(N, w.num_classes, w.graph_seed)
    train = np.arange(LEAVES, dtype=np.int32)
    return dict(row_ptr=row_ptr, col=col, X=X, y=y, train=train, params=make_params(w.dims, w.model, w.init_seed))


@pytest.mark.parametrize("model", ["sage", "gcn"])
def test_hub_row_longer_than_sort_buffer(model):
    w = star_workload(model)
    inp = star_inputs(w)
    graph = dict(row_ptr=inp["row_ptr"], col=inp["col"], X=inp["X"][:, :w.feat_dim], y=inp["y"], train=inp["train"])
    g, m = make_gpu(w, inp)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    want, _ = oracle.sample_batch(w, graph, 0, 0, perm)
    assert np.bincount(want[1]["blk_col"]).max() > 8192   # the centre's transposed row at hop 1
    assert_blocks_equal(m.sample(0, 0), want)
    loss = m.train_minibatch(0, 0)
    check_train_step(m, w, graph, inp["params"].astype(np.float64), 0, 0, perm, loss)
