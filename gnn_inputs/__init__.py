"""Seeded synthetic input generators (no method arithmetic).  Serves both the oracle
(tests, cpu_baseline) and the CUDA path (tests, bench)."""
from .configs import WORKLOADS, Workload
from .synth import (make_graph, make_features, feature_rows, make_labels, make_params,
                    param_count, hash_u64)

_graph_cache = {}


def build_inputs(w: Workload, with_features: bool = True):
    """Graph + features + labels + train ids + initial params for a workload."""
    key = (w.num_nodes, w.nnz, w.graph_seed, w.feat_dim, w.num_classes, with_features)
    if key not in _graph_cache:
        row_ptr, col = make_graph(w.num_nodes, w.nnz, w.graph_seed)
        X = make_features(w.num_nodes, w.feat_dim, w.graph_seed, w.feat_stride) if with_features else None
        y = make_labels(w.num_nodes, w.num_classes, w.graph_seed)
        _graph_cache.clear()
        _graph_cache[key] = (row_ptr, col, X, y)
    row_ptr, col, X, y = _graph_cache[key]
    import numpy as np
    train = np.arange(w.n_train, dtype=np.int32)
    params = make_params(w.dims, w.model, w.init_seed)
    return dict(row_ptr=row_ptr, col=col, X=X, y=y, train=train, params=params)
