"""Seeded synthetic inputs shaped like the paper's workloads (§5.1.2 Table 2,
lines 373-386; BASELINE.json configs).  Shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no sampling, no relabel, no
aggregation, no loss).  It only manufactures inputs: a CSR graph, node features,
labels, train ids and initial weights.  Randomness is a splitmix64 counter hash
(not the Philox stream the method itself draws from, §2.2 / DESIGN.md R3),
so the generator and the method share no RNG code either.

Recipe:
  * degrees  d_v = clamp(floor(dmin * u_v^(-1/(alpha-1))), 1, floor(sqrt(nnz)))
    alpha = 2.1, u_v in (0,1]; dmin bisected so sum 2*ceil(d_v/2) ~= target nnz
    (the paper's "highly skewed workload distribution", §4.2).
  * endpoints: Chung-Lu, symmetric.  Node v draws ceil(d_v/2) partners u with
    P(u) ∝ d_u; both directions stored; self-loops and duplicates dropped; rows
    sorted ascending (SPEC.md graph invariants, lines 25-27, 34).
  * features x[v,j] = (h >> 41) * 2^-22 - 1  in [-1, 1), exact in fp32.
  * labels  y_v = (h >> 32) * C >> 32.
  * train ids = [0, n_train); node ids are exchangeable by construction.
"""
from __future__ import annotations

import math
import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# stream ids
S_DEGREE, S_ENDPOINT, S_FEATURE, S_LABEL, S_PARAM = 1, 2, 3, 4, 5


def _mix64(x: np.ndarray) -> np.ndarray:
    x = x ^ (x >> np.uint64(30))
    x = x * _M1
    x = x ^ (x >> np.uint64(27))
    x = x * _M2
    return x ^ (x >> np.uint64(31))


def hash_u64(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """splitmix64 output number idx+1 of the sequence keyed by (seed, stream)."""
    with np.errstate(over="ignore"):
        key = _mix64(np.array([(seed * 0x100000001B3 + stream * 0x1F3D5B79) & (2**64 - 1)],
                              dtype=np.uint64))[0]
        idx = np.asarray(idx, dtype=np.uint64)
        return _mix64(key + (idx + np.uint64(1)) * _GAMMA)


def _uniform01(seed, stream, idx):
    """uniform in (0, 1], 53 bits."""
    h = hash_u64(seed, stream, idx)
    return ((h >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)


def _degrees(n: int, nnz: int, seed: int, alpha: float = 2.1) -> np.ndarray:
    u = _uniform01(seed, S_DEGREE, np.arange(n, dtype=np.uint64))
    base = u ** (-1.0 / (alpha - 1.0))
    cap = max(1, int(math.isqrt(max(nnz, 1))))

    def total(dmin):
        d = np.clip(np.floor(dmin * base), 1, cap)
        return float((2 * np.ceil(d / 2)).sum())

    lo, hi = 1e-3, float(cap)
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        if total(mid) < nnz:
            lo = mid
        else:
            hi = mid
    return np.clip(np.floor(hi * base), 1, cap).astype(np.int64)


def _chung_lu(n: int, deg: np.ndarray, seed: int, chunk: int = 1 << 25):
    m = ((deg + 1) // 2).astype(np.int64)
    owners = np.repeat(np.arange(n, dtype=np.int64), m)
    cum = np.cumsum(deg.astype(np.float64))
    tot = cum[-1]
    partners = np.empty(owners.shape[0], dtype=np.int64)
    import torch  # CPU only: a multi-threaded searchsorted (numpy's is ~10x slower here)
    tcum = torch.from_numpy(cum)
    for s in range(0, owners.shape[0], chunk):
        e = min(s + chunk, owners.shape[0])
        r = _uniform01(seed, S_ENDPOINT, np.arange(s, e, dtype=np.uint64))
        p = torch.searchsorted(tcum, torch.from_numpy(r * tot), right=False).numpy()
        partners[s:e] = np.minimum(p, n - 1)
    keep = owners != partners
    a, b = owners[keep], partners[keep]
    keys = np.concatenate([a * n + b, b * n + a])
    del a, b, owners, partners
    keys.sort()
    if keys.shape[0]:
        first = np.empty(keys.shape[0], dtype=bool)
        first[0] = True
        np.not_equal(keys[1:], keys[:-1], out=first[1:])
        keys = keys[first]
    rows = keys // n
    cols = (keys - rows * n).astype(np.int32)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    return row_ptr, cols


def make_graph(n: int, nnz: int, seed: int):
    """Symmetric power-law CSR (row_ptr int64[n+1], col int32[nnz'])."""
    deg = _degrees(n, nnz, seed)
    row_ptr, col = _chung_lu(n, deg, seed)
    got = int(row_ptr[-1])
    if got < 0.97 * nnz:  # one correction pass for duplicate loss on dense graphs
        deg = _degrees(n, int(nnz * nnz / max(got, 1)), seed)
        row_ptr, col = _chung_lu(n, deg, seed)
    return row_ptr, col


def feature_rows(rows: np.ndarray, F: int, seed: int, stride: int | None = None) -> np.ndarray:
    """Rows of the feature matrix by formula (so any row is recomputable)."""
    stride = F if stride is None else stride
    rows = np.asarray(rows, dtype=np.int64)
    out = np.zeros((rows.shape[0], stride), dtype=np.float32)
    idx = (rows[:, None].astype(np.uint64) * np.uint64(F) + np.arange(F, dtype=np.uint64)[None, :])
    h = hash_u64(seed, S_FEATURE, idx)
    out[:, :F] = ((h >> np.uint64(41)).astype(np.float64) * (2.0 ** -22) - 1.0).astype(np.float32)
    return out


def make_features(n: int, F: int, seed: int, stride: int | None = None, chunk: int = 1 << 18) -> np.ndarray:
    stride = F if stride is None else stride
    X = np.empty((n, stride), dtype=np.float32)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        X[s:e] = feature_rows(np.arange(s, e), F, seed, stride)
    return X


def make_labels(n: int, C: int, seed: int) -> np.ndarray:
    h = hash_u64(seed, S_LABEL, np.arange(n, dtype=np.uint64))
    return (((h >> np.uint64(32)) * np.uint64(C)) >> np.uint64(32)).astype(np.int32)


def make_params(dims, model: str, seed: int) -> np.ndarray:
    """Glorot-uniform weights, flat fp32 in the library's layout:
    per layer l (input-first): SAGE -> [W_self; W_neigh] as (2*in) x out row-major;
    GCN -> W as in x out row-major."""
    parts = []
    off = 0
    for l in range(len(dims) - 1):
        fi, fo = dims[l], dims[l + 1]
        rows = 2 * fi if model == "sage" else fi
        cnt = rows * fo
        a = math.sqrt(6.0 / (fi + fo))
        h = hash_u64(seed, S_PARAM, np.arange(off, off + cnt, dtype=np.uint64))
        u = (h >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)  # [0,1)
        parts.append(((2.0 * u - 1.0) * a).astype(np.float32))
        off += cnt
    return np.concatenate(parts)


def param_count(dims, model: str) -> int:
    return sum((2 if model == "sage" else 1) * dims[l] * dims[l + 1] for l in range(len(dims) - 1))
