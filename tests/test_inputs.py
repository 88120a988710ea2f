"""Input generator: CSR invariants (SPEC.md graph lines 25-27, 34), determinism, symmetry."""
import numpy as np

from gnn_inputs import make_graph, make_features, feature_rows, make_labels, make_params, param_count
from gnn_inputs import WORKLOADS


def test_csr_invariants_and_determinism():
    rp, col = make_graph(3000, 30000, 5)
    assert rp[0] == 0 and rp[-1] == col.shape[0]
    assert np.all(np.diff(rp) >= 0)
    assert col.min() >= 0 and col.max() < 3000
    for v in range(3000):
        row = col[rp[v]:rp[v + 1]]
        assert np.all(np.diff(row) > 0)          # sorted, duplicate-free
        assert not np.any(row == v)              # no self loops
    rp2, col2 = make_graph(3000, 30000, 5)
    assert np.array_equal(rp, rp2) and np.array_equal(col, col2)
    # symmetric: u in N(v) <=> v in N(u)
    rows = np.repeat(np.arange(3000), np.diff(rp))
    fwd = set(zip(rows.tolist(), col.tolist()))
    assert all((c, r) in fwd for r, c in fwd)
    # skewed degrees (power law), close to the target nnz
    deg = np.diff(rp)
    assert deg.max() > 5 * deg.mean()
    assert 0.9 * 30000 < rp[-1] <= 1.05 * 30000


def test_features_labels_params():
    X = make_features(100, 5, 3, stride=8)
    assert X.shape == (100, 8) and np.all(X[:, 5:] == 0)
    assert X[:, :5].min() >= -1 and X[:, :5].max() < 1
    # exact multiples of 2^-22 (exactly representable, recomputable by formula)
    q = (X[:, :5].astype(np.float64) + 1.0) * 2 ** 22
    assert np.all(q == np.round(q))
    assert np.array_equal(feature_rows(np.array([7, 3]), 5, 3, 8), X[[7, 3]])
    y = make_labels(1000, 8, 3)
    assert y.min() >= 0 and y.max() < 8 and len(np.unique(y)) == 8
    w = WORKLOADS["products"]
    assert param_count(w.dims, "sage") == 206_336
    assert param_count(w.dims, "gcn") == 103_168
    assert param_count(WORKLOADS["reddit"].dims, "sage") == 329_216
    p = make_params([4, 3, 2], "sage", 1)
    assert p.shape == (2 * 4 * 3 + 2 * 3 * 2,)
    assert np.abs(p[:24]).max() <= np.sqrt(6 / 7)
