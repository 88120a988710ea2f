"""ctypes binding of libgnnhost.so (include/gnnhost.h): the host-core trainer rank of the
Unified CPU-GPU protocol (§3).  Argument
marshalling only: the step runs in the C++ library."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build as _build

_LIB = None
GNNH_SAGE_MEAN, GNNH_GCN = 0, 1


class HostError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"gnnhost error {code}: {msg}")
        self.code = code


def lib():
    global _LIB
    if _LIB is None:
        path = _build.build_host()
        L = C.CDLL(path)
        L.gnnh_last_error.restype = C.c_char_p
        L.gnnh_param_count.restype = C.c_int64
        L.gnnh_create.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                  C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_float, C.c_uint64,
                                  C.POINTER(C.c_void_p)]
        L.gnnh_destroy.argtypes = [C.c_void_p]
        L.gnnh_param_count.argtypes = [C.c_void_p]
        L.gnnh_set_params.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.gnnh_get_params.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.gnnh_epoch_permutation.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p]
        L.gnnh_grads.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int64, C.c_void_p,
                                 C.c_void_p]
        L.gnnh_apply.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.gnnh_last_src_ids.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
        _LIB = L
    return _LIB


def _check(rc):
    if rc != 0:
        raise HostError(rc, lib().gnnh_last_error().decode())


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class HostModel:
    """One host-core trainer: gradients of its mini-batches, applied after the all-reduce."""

    def __init__(self, row_ptr, col, X, y, num_classes, feat_dim, model="sage", num_layers=2, hidden=32,
                 fanouts=(10, 5), lr=0.01, seed=1):
        # the library borrows the graph arrays: keep contiguous copies alive with the model
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.col = np.ascontiguousarray(col, dtype=np.int32)
        self.X = np.ascontiguousarray(X, dtype=np.float32)
        self.y = np.ascontiguousarray(y, dtype=np.int32)
        self.fanouts = np.ascontiguousarray(fanouts, dtype=np.int32)
        h = C.c_void_p()
        _check(lib().gnnh_create(self.row_ptr.shape[0] - 1, _p(self.row_ptr), _p(self.col), _p(self.X), feat_dim,
                                 self.X.shape[1], _p(self.y), num_classes,
                                 GNNH_SAGE_MEAN if model == "sage" else GNNH_GCN, num_layers, hidden,
                                 _p(self.fanouts), lr, seed, C.byref(h)))
        self.h = h
        self.param_count = lib().gnnh_param_count(h)

    def close(self):
        if self.h:
            lib().gnnh_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_params(self, p):
        p = np.ascontiguousarray(p, dtype=np.float32)
        _check(lib().gnnh_set_params(self.h, _p(p), p.shape[0]))

    def get_params(self):
        out = np.zeros(self.param_count, np.float32)
        _check(lib().gnnh_get_params(self.h, _p(out), out.shape[0]))
        return out

    def epoch_permutation(self, train_ids, epoch):
        t = np.ascontiguousarray(train_ids, dtype=np.int32)
        out = np.zeros_like(t)
        _check(lib().gnnh_epoch_permutation(self.h, _p(t), t.shape[0], epoch, _p(out)))
        return out

    def grads(self, seeds, b_total, epoch, g):
        """(grad fp32[param_count], loss) of this rank's mini-batch (gnnh_grads)."""
        s = np.ascontiguousarray(seeds, dtype=np.int32)
        out = np.zeros(self.param_count, np.float32)
        loss = C.c_float()
        _check(lib().gnnh_grads(self.h, _p(s), s.shape[0], b_total, epoch, g, _p(out), C.byref(loss)))
        return out, loss.value

    def apply(self, grads):
        g = np.ascontiguousarray(grads, dtype=np.float32)
        _check(lib().gnnh_apply(self.h, _p(g), g.shape[0]))

    def last_src_ids(self, hop):
        n = C.c_int64()
        _check(lib().gnnh_last_src_ids(self.h, hop, None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1), np.int32)
        _check(lib().gnnh_last_src_ids(self.h, hop, _p(out), out.shape[0], C.byref(n)))
        return out[:n.value]
