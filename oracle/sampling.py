"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

ctypes front end of oracle/sampler.c (steps O0-O3).  Builds liboracle.so with gcc on
first use.  Argument marshalling only; every step of O0-O3 is in the C file.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sampler.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        _lib.oracle_philox4x32.argtypes = [P, P, C.c_int, P]
        _lib.oracle_epoch_perm.argtypes = [P, C.c_int64, C.c_uint64, C.c_int64, P]
        _lib.oracle_sample_row.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int32,
                                           C.c_int32, C.c_int64, C.c_int32, P]
        _lib.oracle_neighbor_sample.argtypes = [P, P, C.c_int64, P, C.c_int64, C.c_int32, P,
                                                C.c_uint64, C.c_int64, C.c_int64, P, P,
                                                P, P, P, P, P, P, P]
        _lib.oracle_induce.argtypes = [P, P, C.c_int64, P, C.c_int64, C.c_int64, P, P, P]
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def philox4x32(ctr, key, rounds: int = 10):
    c = np.asarray(ctr, dtype=np.uint32).copy()
    k = np.asarray(key, dtype=np.uint32).copy()
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32(_p(c), _p(k), rounds, _p(out))
    return out


def epoch_perm(train: np.ndarray, seed: int, epoch: int) -> np.ndarray:
    t = np.ascontiguousarray(train, dtype=np.int32)
    out = np.empty_like(t)
    rc = lib().oracle_epoch_perm(_p(t), t.shape[0], seed, epoch, _p(out))
    assert rc == 0
    return out


def batch_seeds(perm: np.ndarray, batch_size: int, g: int) -> np.ndarray:
    """Batch g = perm[g*B : min((g+1)*B, n)] (O1)."""
    return perm[g * batch_size: min((g + 1) * batch_size, perm.shape[0])]


def sample_row(seed, epoch, g, hop, v, d, k) -> np.ndarray:
    pos = np.zeros(max(k, d if d <= k else k, 1), dtype=np.int64)
    cnt = lib().oracle_sample_row(seed, epoch, g, hop, v, d, k, _p(pos))
    return pos[:cnt].copy()


def neighbor_sample(row_ptr, col, seeds, fanouts, seed, epoch, g):
    """O2.  Returns a list over hops h = 0..L-1 (seeds outward) of dicts with
    n_dst, n_src, n_edges, src_ids, blk_rowptr, blk_col, blk_nbr."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    seeds = np.ascontiguousarray(seeds, dtype=np.int32)
    N = row_ptr.shape[0] - 1
    L = len(fanouts)
    fan = np.asarray(fanouts, dtype=np.int32)
    cap_src, cap_edges = [], []
    nd = seeds.shape[0]
    for h in range(L):
        k = int(fan[L - 1 - h])
        ce = nd * k
        cs = min(nd + ce, N) if N > 0 else nd
        cap_edges.append(ce)
        cap_src.append(max(cs, nd))
        nd = cap_src[-1]
    cap_src_a = np.asarray(cap_src, dtype=np.int64)
    cap_edges_a = np.asarray(cap_edges, dtype=np.int64)
    bufs_src = [np.zeros(max(c, 1), dtype=np.int32) for c in cap_src]
    dst_caps = [seeds.shape[0]] + cap_src[:-1]
    bufs_rp = [np.zeros(c + 1, dtype=np.int32) for c in dst_caps]
    bufs_col = [np.zeros(max(c, 1), dtype=np.int32) for c in cap_edges]
    bufs_nbr = [np.zeros(max(c, 1), dtype=np.int32) for c in cap_edges]
    n_dst = np.zeros(L, dtype=np.int64)
    n_src = np.zeros(L, dtype=np.int64)
    n_edges = np.zeros(L, dtype=np.int64)

    def ptrs(bufs):
        arr = (C.c_void_p * L)(*[b.ctypes.data for b in bufs])
        return arr

    rc = lib().oracle_neighbor_sample(_p(row_ptr), _p(col), N, _p(seeds), seeds.shape[0], L, _p(fan),
                                      seed, epoch, g, _p(cap_src_a), _p(cap_edges_a),
                                      _p(n_dst), _p(n_src), _p(n_edges),
                                      ptrs(bufs_src), ptrs(bufs_rp), ptrs(bufs_col), ptrs(bufs_nbr))
    assert rc == 0, rc
    hops = []
    for h in range(L):
        hops.append(dict(n_dst=int(n_dst[h]), n_src=int(n_src[h]), n_edges=int(n_edges[h]),
                         src_ids=bufs_src[h][:n_src[h]].copy(),
                         blk_rowptr=bufs_rp[h][:n_dst[h] + 1].copy(),
                         blk_col=bufs_col[h][:n_edges[h]].copy(),
                         blk_nbr=bufs_nbr[h][:n_edges[h]].copy()))
    return hops


def induce(row_ptr, col, S):
    """O3 step 2: induced CSR over node set S (local ids)."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    S = np.ascontiguousarray(S, dtype=np.int32)
    cap = int((row_ptr[S.astype(np.int64) + 1] - row_ptr[S.astype(np.int64)]).sum()) if S.shape[0] else 0
    rp = np.zeros(S.shape[0] + 1, dtype=np.int32)
    ic = np.zeros(max(cap, 1), dtype=np.int32)
    ne = np.zeros(1, dtype=np.int64)
    rc = lib().oracle_induce(_p(row_ptr), _p(col), row_ptr.shape[0] - 1, _p(S), S.shape[0], cap,
                             _p(rp), _p(ic), _p(ne))
    assert rc == 0, rc
    return rp, ic[:ne[0]].copy()


def shadow_sample(row_ptr, col, seeds, fanouts, num_layers, seed, epoch, g):
    """O3: L' = len(fanouts) hops of O2, S = final src list, induced square block used by
    all num_layers layers.  Returns (hops_of_O2, block) with block a dict like a hop."""
    hops = neighbor_sample(row_ptr, col, seeds, fanouts, seed, epoch, g)
    S = hops[-1]["src_ids"]
    rp, ic = induce(row_ptr, col, S)
    nbr = S[ic] if ic.shape[0] else np.zeros(0, dtype=np.int32)
    block = dict(n_dst=int(S.shape[0]), n_src=int(S.shape[0]), n_edges=int(ic.shape[0]),
                 src_ids=S.copy(), blk_rowptr=rp, blk_col=ic, blk_nbr=nbr.astype(np.int32))
    return hops, block
