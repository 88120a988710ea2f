"""Thin ctypes binding of libgnnstep.so (include/gnnstep.h).  Argument marshalling only:
every step of the hot path runs in the library's sm_100a kernels.  There is no CPU
fallback: if the library cannot be loaded, import fails loudly."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build as _build

GNN_SAGE_MEAN, GNN_GCN = 0, 1
GNN_NEIGHBOR, GNN_SHADOW = 0, 1
GNN_FP32, GNN_BF16_GEMM = 0, 1
GNN_SRC_IDS, GNN_BLK_ROWPTR, GNN_BLK_COL, GNN_BLK_NBR = 0, 1, 2, 3
GNN_DBG_LOGITS, GNN_DBG_GRADS, GNN_DBG_LOSS, GNN_DBG_ACT = 0, 1, 2, 16
GNN_SGD, GNN_ADAM = 0, 1
GNN_EXCH_AUTO, GNN_EXCH_NCCL, GNN_EXCH_PEER, GNN_EXCH_HOST = 0, 1, 2, 3
ABI_VERSION = 2   # include/gnnstep.h GNN_ABI_VERSION
KERNEL_IDS = dict(sample=0, relabel=1, agg_l1=2, agg=3, gemm_fwd=4, gemm_dgrad=5, gemm_wgrad=6,
                  spmm_bwd=7, ce=8, sgd=9, transpose=10, induce=11, allreduce=12, scan=13, other=14)

_STATUS = {0: "OK", -1: "RANGE", -2: "PARAM", -3: "SHAPE", -4: "CONFIG", -5: "STATE", -6: "BUFFER",
           -7: "OOM", -8: "CUDA", -9: "NCCL"}


class GnnError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"gnnstep {_STATUS.get(code, code)}: {msg}")
        self.code = code


class _Config(C.Structure):
    _fields_ = [("model", C.c_int32), ("sampler", C.c_int32), ("num_layers", C.c_int32),
                ("hidden", C.c_int32), ("batch_size", C.c_int32), ("num_fanouts", C.c_int32),
                ("fanouts", C.c_int32 * 8), ("precision", C.c_int32), ("use_graph", C.c_int32),
                ("lr", C.c_float), ("seed", C.c_uint64), ("init_seed", C.c_uint64),
                ("optimizer", C.c_int32), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float)]


class _Sizes(C.Structure):
    _fields_ = [("num_hops", C.c_int32), ("n_dst", C.c_int64 * 9), ("n_src", C.c_int64 * 9),
                ("n_edges", C.c_int64 * 9)]


class _EpochStats(C.Structure):
    _fields_ = [("seconds", C.c_double), ("steps", C.c_int64), ("minibatches", C.c_int64),
                ("mean_loss", C.c_double)]


_lib = None


def lib():
    """Load the in-tree library (building it with nvcc if it is missing or stale)."""
    global _lib
    if _lib is None:
        # GS_LIB: an A/B experiment variant built by build.py --out (never the default)
        path = os.environ.get("GS_LIB") or _build.build()
        _lib = C.CDLL(path)
        P, I32, I64 = C.c_void_p, C.c_int32, C.c_int64
        sig = {
            "gnn_last_error": ([], C.c_char_p), "gnn_abi_version": ([], I32),
            "gnn_graph_create": ([I64, P, P, I32, I32, P, P, I32, I32, P], I32),
            "gnn_graph_destroy": ([P], I32),
            "gnn_model_create": ([P, P, P], I32), "gnn_model_destroy": ([P], I32),
            "gnn_set_stream": ([P, P], I32), "gnn_set_train_nodes": ([P, P, I64], I32),
            "gnn_param_count": ([P], I64), "gnn_num_batches": ([P], I64),
            "gnn_get_params": ([P, P, I64], I32), "gnn_set_params": ([P, P, I64], I32),
            "gnn_comm_get_unique_id": ([P], I32), "gnn_comm_init": ([P, I32, I32, P], I32),
            "gnn_epoch_permutation": ([P, I64, P, I64], I32),
            "gnn_sample": ([P, I64, I64, P], I32), "gnn_sample_fetch": ([P, I32, I32, P, I64], I32),
            "gnn_train_minibatch": ([P, I64, I64, P], I32),
            "gnn_train_batch_host": ([P, P, I32, I32, I64, I64, P, I32, I32, I64, P], I32),
            "gnn_set_overlap": ([P, I32], I32),
            "gnn_train_epoch": ([P, I64, P], I32), "gnn_synchronize": ([P], I32),
            "gnn_debug_get": ([P, I32, P, I64], I32), "gnn_last_sizes": ([P, P], I32),
            "gnn_profile_enable": ([P, I32], I32), "gnn_profile_read": ([P, I32, P, P], I32),
            "gnn_profile_reset": ([P], I32), "gnn_launches_per_step": ([P], I64),
            "gnn_graph_symmetric": ([P], I32),
            "gnn_estimate_workload": ([P, I64, P, I64], I32), "gnn_plan_balanced": ([P, I64, I32, P], I32),
            "gnn_set_schedule": ([P, P, I64], I32), "gnn_set_exchange": ([P, I32], I32),
            "gnn_cache_stats": ([P, I32, P], I32), "gnn_exchange_export": ([P, I32, I32, P], I32),
            "gnn_exchange_import": ([P, P], I32),
            "gnn_apply_update": ([P, P, I64], I32), "gnn_set_rank": ([P, I32, I32], I32),
        }
        for name, (args, res) in sig.items():
            f = getattr(_lib, name)
            f.argtypes = args
            f.restype = res
        if _lib.gnn_abi_version() != ABI_VERSION:
            v, _lib = _lib.gnn_abi_version(), None
            raise RuntimeError(f"libgnnstep ABI {v} != binding ABI {ABI_VERSION} (rebuild)")
    return _lib


def _check(rc):
    if rc != 0:
        raise GnnError(rc, lib().gnn_last_error().decode())


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def comm_get_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().gnn_comm_get_unique_id(buf))
    return bytes(buf)


class Graph:
    """gnn_graph_create: CSR + features + labels, copied to HBM of `device`."""

    def __init__(self, row_ptr, col, X, y, num_classes, feat_dim=None, device=0):
        self._keep = None
        row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        col = np.ascontiguousarray(col, dtype=np.int32)
        X = np.ascontiguousarray(X, dtype=np.float32)
        y = np.ascontiguousarray(y, dtype=np.int32)
        n = row_ptr.shape[0] - 1
        stride = X.shape[1]
        self.num_nodes, self.num_classes = n, num_classes
        self.feat_dim = stride if feat_dim is None else feat_dim
        self.device = device
        h = C.c_void_p()
        _check(lib().gnn_graph_create(n, _ptr(row_ptr), _ptr(col), self.feat_dim, stride, _ptr(X), _ptr(y),
                                      num_classes, device, C.byref(h)))
        self.h = h

    @property
    def symmetric(self) -> bool:
        return lib().gnn_graph_symmetric(self.h) == 1

    def close(self):
        if self.h:
            lib().gnn_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Model:
    """gnn_model_create + the training / sampling calls of include/gnnstep.h."""

    def __init__(self, graph: Graph, model="sage", sampler="neighbor", num_layers=2, hidden=32,
                 batch_size=64, fanouts=(10, 5), precision="fp32", use_graph=True, lr=0.01, seed=1,
                 init_seed=2, optimizer="sgd", betas=(0.9, 0.999), eps=1e-8):
        cfg = _Config()
        cfg.model = GNN_SAGE_MEAN if model == "sage" else GNN_GCN
        cfg.sampler = GNN_NEIGHBOR if sampler == "neighbor" else GNN_SHADOW
        cfg.num_layers, cfg.hidden, cfg.batch_size = num_layers, hidden, batch_size
        cfg.num_fanouts = len(fanouts)
        for i, f in enumerate(fanouts):
            cfg.fanouts[i] = f
        cfg.precision = GNN_FP32 if precision == "fp32" else GNN_BF16_GEMM
        cfg.use_graph = 1 if use_graph else 0
        cfg.lr, cfg.seed, cfg.init_seed = lr, seed, init_seed
        if optimizer not in ("sgd", "adam"):
            raise ValueError("optimizer must be 'sgd' or 'adam'")
        cfg.optimizer = GNN_SGD if optimizer == "sgd" else GNN_ADAM
        cfg.beta1, cfg.beta2, cfg.eps = betas[0], betas[1], eps
        self.graph = graph
        self.model, self.sampler, self.num_layers = model, sampler, num_layers
        self.fanouts = tuple(fanouts)
        h = C.c_void_p()
        _check(lib().gnn_model_create(graph.h, C.byref(cfg), C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            lib().gnn_model_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- setup
    def set_stream(self, stream):
        """stream: torch.cuda.Stream, an int handle, or None (library's own)."""
        handle = getattr(stream, "cuda_stream", stream)
        _check(lib().gnn_set_stream(self.h, C.c_void_p(handle) if handle else None))

    def set_train_nodes(self, ids):
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        _check(lib().gnn_set_train_nodes(self.h, _ptr(ids), ids.shape[0]))
        self._n_train = ids.shape[0]

    @property
    def param_count(self) -> int:
        return lib().gnn_param_count(self.h)

    @property
    def num_batches(self) -> int:
        return lib().gnn_num_batches(self.h)

    def get_params(self) -> np.ndarray:
        out = np.empty(self.param_count, dtype=np.float32)
        _check(lib().gnn_get_params(self.h, _ptr(out), out.shape[0]))
        return out

    def set_params(self, p):
        p = np.ascontiguousarray(p, dtype=np.float32)
        _check(lib().gnn_set_params(self.h, _ptr(p), p.shape[0]))

    def set_exchange(self, mode: str):
        """gnn_set_exchange: "auto" (world 1: reduce fused into the update), "nccl" (per-layer
        reduce -> ncclAllReduce buckets -> update, on any world; world 1 uses a one-rank
        communicator) or "peer" (one-shot all-reduce over CUDA-IPC peer memory, after
        exchange_export / exchange_import)."""
        _check(lib().gnn_set_exchange(self.h, {"auto": GNN_EXCH_AUTO, "nccl": GNN_EXCH_NCCL,
                                               "peer": GNN_EXCH_PEER, "host": GNN_EXCH_HOST}[mode]))

    def set_rank(self, rank: int, world: int):
        """gnn_set_rank: rank/world of the batch -> rank rule without an NCCL communicator."""
        _check(lib().gnn_set_rank(self.h, rank, world))

    def apply_update(self, grads=None):
        """gnn_apply_update (GNN_EXCH_HOST): the update with the all-reduced gradient (fp32 host
        array of param_count; None: the device gradient as it stands)."""
        if grads is None:
            _check(lib().gnn_apply_update(self.h, None, 0))
            return
        g = np.ascontiguousarray(grads, dtype=np.float32)
        _check(lib().gnn_apply_update(self.h, _ptr(g), g.shape[0]))

    def exchange_export(self, rank: int, world: int) -> bytes:
        """gnn_exchange_export: allocate this rank's inbox; returns its 64-byte CUDA IPC handle."""
        buf = (C.c_uint8 * 64)()
        _check(lib().gnn_exchange_export(self.h, rank, world, buf))
        return bytes(buf)

    def exchange_import(self, handles):
        """gnn_exchange_import: map every rank's inbox (handles in rank order)."""
        blob = b"".join(handles)
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        _check(lib().gnn_exchange_import(self.h, buf))

    def comm_init(self, rank: int, world: int, uid: bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib().gnn_comm_init(self.h, rank, world, buf))

    def epoch_permutation(self, epoch: int) -> np.ndarray:
        """gnn_epoch_permutation: the epoch's seed order (batch g = perm[g*B:(g+1)*B])."""
        n = int(self._n_train)
        out = np.zeros(max(n, 1), dtype=np.int32)
        _check(lib().gnn_epoch_permutation(self.h, epoch, _ptr(out), out.shape[0]))
        return out[:n]

    # ---------------------------------------------------------------- sampling (parity hook)
    def sample(self, epoch: int, g: int):
        """gnn_sample + gnn_sample_fetch.  Returns hop dicts (seeds outward) in the oracle's
        format; for ShaDow also the induced block: (hops, block)."""
        sz = _Sizes()
        _check(lib().gnn_sample(self.h, epoch, g, C.byref(sz)))

        def fetch(hop, what, n):
            out = np.zeros(max(n, 1), dtype=np.int32)
            _check(lib().gnn_sample_fetch(self.h, hop, what, _ptr(out), out.shape[0]))
            return out[:n]

        def block(h):
            nd, ns, ne = sz.n_dst[h], sz.n_src[h], sz.n_edges[h]
            return dict(n_dst=nd, n_src=ns, n_edges=ne, src_ids=fetch(h, GNN_SRC_IDS, ns),
                        blk_rowptr=fetch(h, GNN_BLK_ROWPTR, nd + 1), blk_col=fetch(h, GNN_BLK_COL, ne),
                        blk_nbr=fetch(h, GNN_BLK_NBR, ne))

        hops = [block(h) for h in range(sz.num_hops)]
        if self.sampler == "shadow":
            return hops, block(sz.num_hops)
        return hops

    # ---------------------------------------------------------------- training
    def train_minibatch(self, epoch: int, step: int, sync: bool = True):
        if not sync:
            _check(lib().gnn_train_minibatch(self.h, epoch, step, None))
            return None
        loss = C.c_float()
        _check(lib().gnn_train_minibatch(self.h, epoch, step, C.byref(loss)))
        return loss.value

    def train_batch_host(self, seeds: np.ndarray, b_total: int, epoch: int, g: int, next_seeds=None,
                         next_b_total: int = 0, next_g: int = -1) -> float:
        """End-to-end call: host seeds -> device, one step, loss -> host (synchronous).  With
        next_g >= 0 the next call's batch (next_seeds, next_b_total, next_g) is sampled while
        this one trains."""
        seeds = np.ascontiguousarray(seeds, dtype=np.int32)
        nxt = np.ascontiguousarray(next_seeds if next_seeds is not None else np.zeros(0), dtype=np.int32)
        loss = C.c_float()
        _check(lib().gnn_train_batch_host(self.h, _ptr(seeds), seeds.shape[0], b_total, epoch, g,
                                          _ptr(nxt), nxt.shape[0], next_b_total, next_g, C.byref(loss)))
        return loss.value

    def train_batch_host_ptr(self, seeds_ptr: int, n: int, b_total: int, epoch: int, g: int,
                             loss_ptr: int, next_ptr: int = 0, next_n: int = 0, next_b_total: int = 0,
                             next_g: int = -1):
        """Same as train_batch_host with raw host pointers; no numpy copies."""
        _check(lib().gnn_train_batch_host(self.h, C.c_void_p(seeds_ptr), n, b_total, epoch, g,
                                          C.c_void_p(next_ptr) if next_ptr else None, next_n, next_b_total,
                                          next_g, C.c_void_p(loss_ptr)))

    def set_overlap(self, enable: bool):
        """gnn_set_overlap: sample step s+1 while step s trains (default on)."""
        _check(lib().gnn_set_overlap(self.h, 1 if enable else 0))

    def train_epoch(self, epoch: int):
        st = _EpochStats()
        _check(lib().gnn_train_epoch(self.h, epoch, C.byref(st)))
        return dict(seconds=st.seconds, steps=st.steps, minibatches=st.minibatches, mean_loss=st.mean_loss)

    def synchronize(self):
        _check(lib().gnn_synchronize(self.h))

    # ---------------------------------------------------------------- introspection
    def sample_sizes(self, epoch: int, g: int):
        """gnn_sample's per-hop sizes of global batch g (full relabel of every hop)."""
        sz = _Sizes()
        _check(lib().gnn_sample(self.h, epoch, g, C.byref(sz)))
        n = sz.num_hops + 1
        return dict(n_dst=list(sz.n_dst[:n]), n_src=list(sz.n_src[:n]), n_edges=list(sz.n_edges[:n]))

    def last_sizes(self):
        sz = _Sizes()
        _check(lib().gnn_last_sizes(self.h, C.byref(sz)))
        n = sz.num_hops + 1
        return dict(n_dst=list(sz.n_dst[:n]), n_src=list(sz.n_src[:n]), n_edges=list(sz.n_edges[:n]))

    def logits(self, b: int, C_: int) -> np.ndarray:
        out = np.zeros(max(b * C_, 1), dtype=np.float32)
        _check(lib().gnn_debug_get(self.h, GNN_DBG_LOGITS, _ptr(out), out.shape[0]))
        return out[:b * C_].reshape(b, C_)

    def grads(self) -> np.ndarray:
        out = np.zeros(self.param_count, dtype=np.float32)
        _check(lib().gnn_debug_get(self.h, GNN_DBG_GRADS, _ptr(out), out.shape[0]))
        return out

    def activation(self, layer: int, rows: int, out: int) -> np.ndarray:
        buf = np.zeros(max(rows * out, 1), dtype=np.float32)
        _check(lib().gnn_debug_get(self.h, GNN_DBG_ACT + layer, _ptr(buf), buf.shape[0]))
        return buf[:rows * out].reshape(rows, out)

    def loss(self) -> float:
        out = np.zeros(1, dtype=np.float32)
        _check(lib().gnn_debug_get(self.h, GNN_DBG_LOSS, _ptr(out), 1))
        return float(out[0])

    def profile_enable(self, on: bool = True):
        _check(lib().gnn_profile_enable(self.h, 1 if on else 0))

    def profile_reset(self):
        _check(lib().gnn_profile_reset(self.h))

    def profile_read(self, kernel: str):
        ms, n = C.c_double(), C.c_int64()
        _check(lib().gnn_profile_read(self.h, KERNEL_IDS[kernel], C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def estimate_workload(self, epoch: int) -> np.ndarray:
        """gnn_estimate_workload: aggregations (Σ_l E(block_l)) of every batch of `epoch`."""
        out = np.zeros(self.num_batches, dtype=np.int64)
        _check(lib().gnn_estimate_workload(self.h, epoch, _ptr(out), out.shape[0]))
        return out

    def set_schedule(self, order):
        """gnn_set_schedule: step s, rank r trains batch order[s*world + r]; None restores the default."""
        if order is None:
            _check(lib().gnn_set_schedule(self.h, None, 0))
            return
        o = np.ascontiguousarray(order, dtype=np.int64)
        _check(lib().gnn_set_schedule(self.h, _ptr(o), o.shape[0]))

    @property
    def launches_per_step(self) -> int:
        return lib().gnn_launches_per_step(self.h)


def _phases(self, n=32):
    out = np.zeros(n, dtype=np.float32)
    _check(lib().gnn_debug_get(self.h, 8, _ptr(out), n))
    nz = np.nonzero(out)[0]
    return out[:int(nz[-1]) + 1] if len(nz) else out[:0]


Model.sampling_phases_us = _phases


def _reuse(self):
    """gnn_debug_get(GNN_DBG_REUSE): (steps whose batch was prefetched, steps that sampled first)."""
    out = np.zeros(2, dtype=np.float32)
    _check(lib().gnn_debug_get(self.h, 9, _ptr(out), 2))
    return int(out[0]), int(out[1])


Model.prefetch_reuse = _reuse


def plan_step(n_train: int, batch_size: int, world: int, rank: int, step: int):
    """gnn_plan_step: (g, n, offset, b_total) of `rank` at `step` (host only)."""
    L = lib()
    L.gnn_plan_step.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int64,
                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.gnn_plan_step.restype = C.c_int32
    g, off = C.c_int64(), C.c_int64()
    n, bt = C.c_int32(), C.c_int32()
    _check(L.gnn_plan_step(n_train, batch_size, world, rank, step, C.byref(g), C.byref(n), C.byref(off),
                           C.byref(bt)))
    return g.value, n.value, off.value, bt.value


def plan_balanced(work, world: int) -> np.ndarray:
    """gnn_plan_balanced (host only): the workload-balanced batch order (NEXT-3)."""
    w = np.ascontiguousarray(work, dtype=np.int64)
    out = np.zeros(w.shape[0], dtype=np.int64)
    _check(lib().gnn_plan_balanced(_ptr(w), w.shape[0], world, _ptr(out)))
    return out


def steps_per_epoch(n_train: int, batch_size: int, world: int) -> int:
    L = lib()
    L.gnn_steps_per_epoch.argtypes = [C.c_int64, C.c_int32, C.c_int32]
    L.gnn_steps_per_epoch.restype = C.c_int64
    return L.gnn_steps_per_epoch(n_train, batch_size, world)


class ShardedGraph(Graph):
    """gnn_graph_create_sharded: full CSR + labels, this process's block of feature rows."""

    def __init__(self, row_ptr, col, X_shard, y, num_classes, nshards, shard, feat_dim=None, device=0):
        row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        col = np.ascontiguousarray(col, dtype=np.int32)
        X_shard = np.ascontiguousarray(X_shard, dtype=np.float32)
        y = np.ascontiguousarray(y, dtype=np.int32)
        n = row_ptr.shape[0] - 1
        stride = X_shard.shape[1]
        self.num_nodes, self.num_classes, self.device = n, num_classes, device
        self.feat_dim = stride if feat_dim is None else feat_dim
        self.nshards, self.shard = nshards, shard
        L = lib()
        L.gnn_graph_create_sharded.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                               C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32,
                                               C.c_int32, C.c_void_p]
        L.gnn_graph_create_sharded.restype = C.c_int32
        h = C.c_void_p()
        _check(L.gnn_graph_create_sharded(n, _ptr(row_ptr), _ptr(col), self.feat_dim, stride, nshards, shard,
                                          _ptr(X_shard), _ptr(y), num_classes, device, C.byref(h)))
        self.h = h

    def export_handle(self) -> bytes:
        buf = (C.c_uint8 * 64)()
        L = lib()
        L.gnn_shard_export.argtypes = [C.c_void_p, C.c_void_p]
        L.gnn_shard_export.restype = C.c_int32
        _check(L.gnn_shard_export(self.h, buf))
        return bytes(buf)

    def cache_rows(self, ids):
        """gnn_cache_rows: replicate these remote rows locally (NEXT-2); empty/None drops the cache."""
        L = lib()
        L.gnn_cache_rows.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.gnn_cache_rows.restype = C.c_int32
        if ids is None or len(ids) == 0:
            _check(L.gnn_cache_rows(self.h, None, 0))
            return
        a = np.ascontiguousarray(ids, dtype=np.int32)
        _check(L.gnn_cache_rows(self.h, _ptr(a), a.shape[0]))

    def cache_stats(self, enable=-1):
        """gnn_cache_stats: row reads {local, peer, cache} since the last reset (synchronizes);
        enable 1 = reset + count, 0 = reset + stop, -1 = read only."""
        out = np.zeros(3, dtype=np.int64)
        _check(lib().gnn_cache_stats(self.h, enable, _ptr(out)))
        return dict(local=int(out[0]), peer=int(out[1]), cache=int(out[2]))

    def import_handles(self, handles):
        blob = b"".join(handles)
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        L = lib()
        L.gnn_shard_import.argtypes = [C.c_void_p, C.c_void_p]
        L.gnn_shard_import.restype = C.c_int32
        _check(L.gnn_shard_import(self.h, buf))


class DeviceGraph(ShardedGraph):
    """gnn_graph_create_device: the graph from device buffers, borrowed (no copy).  row_ptr,
    col, X (this shard's rows), y: objects with a `.ptr` device address (or ints); they are kept
    alive by this object and must not change while it lives."""

    def __init__(self, num_nodes, row_ptr, col, X, y, num_classes, feat_dim, feat_stride, nshards=1, shard=0,
                 device=0):
        self._keep = (row_ptr, col, X, y)
        self.num_nodes, self.num_classes, self.device = num_nodes, num_classes, device
        self.feat_dim, self.nshards, self.shard = feat_dim, nshards, shard
        addr = lambda o: C.c_void_p(getattr(o, "ptr", o))
        L = lib()
        L.gnn_graph_create_device.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                              C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
        L.gnn_graph_create_device.restype = C.c_int32
        h = C.c_void_p()
        _check(L.gnn_graph_create_device(num_nodes, addr(row_ptr), addr(col), feat_dim, feat_stride, nshards, shard,
                                         addr(X), addr(y), num_classes, device, C.byref(h)))
        self.h = h


def cache_plan_by_degree(row_ptr, nshards: int, shard: int, capacity: int) -> np.ndarray:
    """gnn_cache_plan_by_degree (host only): the hottest remote rows of `shard` (NEXT-2)."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    n = rp.shape[0] - 1
    out = np.zeros(max(min(capacity, n), 1), dtype=np.int32)
    cnt = C.c_int64()
    L = lib()
    L.gnn_cache_plan_by_degree.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int64, C.c_void_p,
                                           C.c_void_p]
    L.gnn_cache_plan_by_degree.restype = C.c_int32
    _check(L.gnn_cache_plan_by_degree(_ptr(rp), n, nshards, shard, min(capacity, n), _ptr(out), C.byref(cnt)))
    return out[:cnt.value].copy()


def shard_rows(num_nodes: int, nshards: int, shard: int):
    """[begin, end) rows of block `shard` (the library's uniform row blocks)."""
    rps = (num_nodes + nshards - 1) // nshards
    b = min(num_nodes, shard * rps)
    return b, min(num_nodes, b + rps)
