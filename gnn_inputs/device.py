"""Device-side input generator (gnn_inputs/gen_device.cu -> libgnngen.so): the papers100M-shaped
workload (BASELINE.json configs[4]) built directly in GPU memory, where the host could not hold it
(57 GB of features).  Input manufacturing only, like synth.py; holds none of the method's
arithmetic.  Features and labels are bit-identical to synth.feature_rows / synth.make_labels, so
the oracle recomputes any feature row by formula; the CSR is copied to the host for the oracle."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "gen_device.cu")
LIB = os.path.join(HERE, "libgnngen.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".{os.getpid()}.tmp"
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler",
                        "-fPIC", "-shared", "-o", tmp, SRC], check=True, capture_output=True)
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P, I32, I64, U64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
        for name, args, res in [("gen_graph", [I64, I64, U64, P, P, P], I32),
                                ("gen_features", [I64, I64, I32, I32, U64, P], I32),
                                ("gen_labels", [I64, I32, U64, P], I32), ("gen_free", [P], None),
                                ("gen_alloc", [I64], P), ("gen_d2h", [P, P, I64], I32),
                                ("gen_set_device", [I32], I32)]:
            f = getattr(_lib, name)
            f.argtypes, f.restype = args, res
    return _lib


class DeviceBuffer:
    """A cudaMalloc'ed buffer (its own allocation: CUDA IPC can export it)."""

    def __init__(self, nbytes: int, dtype):
        self.ptr = lib().gen_alloc(max(int(nbytes), 16))
        if not self.ptr:
            raise MemoryError(f"cudaMalloc of {nbytes} bytes failed")
        self.nbytes, self.dtype = int(nbytes), np.dtype(dtype)

    def to_host(self, count=None) -> np.ndarray:
        n = self.nbytes // self.dtype.itemsize if count is None else int(count)
        out = np.empty(n, dtype=self.dtype)
        if n and lib().gen_d2h(out.ctypes.data, self.ptr, n * self.dtype.itemsize) != 0:
            raise RuntimeError("device -> host copy failed")
        return out

    def free(self):
        if self.ptr:
            lib().gen_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def make_graph_device(n: int, nnz: int, seed: int, device: int = 0):
    """Symmetric power-law Chung-Lu CSR built on the device (the synth.make_graph recipe, with its
    one correction pass when duplicates drop the count below 97 % of the target)."""
    L = lib()
    L.gen_set_device(device)

    def once(target):
        rp, col, m = C.c_void_p(), C.c_void_p(), C.c_int64()
        rc = L.gen_graph(n, target, seed, C.byref(rp), C.byref(col), C.byref(m))
        if rc != 0:
            raise RuntimeError(f"gen_graph failed ({rc})")
        a = DeviceBuffer.__new__(DeviceBuffer)
        a.ptr, a.nbytes, a.dtype = rp.value, 8 * (n + 1), np.dtype(np.int64)
        b = DeviceBuffer.__new__(DeviceBuffer)
        b.ptr, b.nbytes, b.dtype = col.value, 4 * max(m.value, 1), np.dtype(np.int32)
        return a, b, m.value

    rp, col, got = once(nnz)
    if got < 0.97 * nnz:
        rp.free(); col.free()
        rp, col, got = once(int(nnz * nnz / max(got, 1)))
    return rp, col, got


def make_features_device(n: int, F: int, seed: int, stride: int, r0: int = 0, r1: int | None = None,
                         device: int = 0) -> DeviceBuffer:
    """Rows [r0, r1) of the feature table (synth.feature_rows bit for bit) in a new allocation."""
    r1 = n if r1 is None else r1
    L = lib()
    L.gen_set_device(device)
    X = DeviceBuffer(4 * (r1 - r0) * stride, np.float32)
    if L.gen_features(r0, r1 - r0, F, stride, seed, X.ptr) != 0:
        raise RuntimeError("gen_features failed")
    return X


def make_labels_device(n: int, C_: int, seed: int, device: int = 0) -> DeviceBuffer:
    L = lib()
    L.gen_set_device(device)
    y = DeviceBuffer(4 * n, np.int32)
    if L.gen_labels(n, C_, seed, y.ptr) != 0:
        raise RuntimeError("gen_labels failed")
    return y


def build_inputs_device(w, nshards: int = 1, shard: int = 0, host_csr: bool = False, device: int = 0):
    """configs[4]-scale inputs on the device: CSR, this shard's feature rows, labels (device
    buffers), train ids and initial params (host).  host_csr: also the CSR on the host (oracle)."""
    from .synth import make_params
    rp, col, nnz = make_graph_device(w.num_nodes, w.nnz, w.graph_seed, device)
    rps = (w.num_nodes + nshards - 1) // nshards
    r0 = min(w.num_nodes, shard * rps)
    r1 = min(w.num_nodes, r0 + rps)
    X = make_features_device(w.num_nodes, w.feat_dim, w.graph_seed, w.feat_stride, r0, r1, device)
    y = make_labels_device(w.num_nodes, w.num_classes, w.graph_seed, device)
    out = dict(row_ptr_dev=rp, col_dev=col, nnz=nnz, X_dev=X, y_dev=y, rows=(r0, r1),
               train=np.arange(w.n_train, dtype=np.int32), params=make_params(w.dims, w.model, w.init_seed))
    if host_csr:
        out["row_ptr"] = rp.to_host()
        out["col"] = col.to_host(nnz)
    return out
