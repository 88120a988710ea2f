"""Helpers for the -m gpu parity tests: build the CUDA path and the oracle on the same
seeded inputs (gnn_inputs), compare element by element."""
import numpy as np

from gnn_inputs import WORKLOADS, build_inputs

TOL_FP32 = 1e-4     # BASELINE.json north_star: fp32 loss/logits/grads within 1e-4 relative
TOL_BF16 = 2e-2     # bf16-GEMM variant


# Kink ambiguity (reading R27): a ReLU decision may differ from the oracle's only where |Pre| is
# within the GEMM's rounding error of 0.  fp32 path (3-term bf16 split, R28): ~2^-16 per product,
# bound 1e-5 * (|A||W|).  bf16-GEMM variant: both operands rounded to bf16 (2^-9 each, 2^-8 per
# product) and the input H of layer l > 1 already carries the previous layer's bf16 error, so
# 2^-6 * (|A||W|) (R33).
KINK = {"fp32": 1e-5, "bf16": 2.0 ** -6}
# A flip is rare: at most this share of a layer's units (plus a few) may be kink-ambiguous.
MAX_FLIP_SHARE = {"fp32": 1e-5, "bf16": 2e-3}


def rel(a, b):
    """DESIGN.md R24: per-tensor ||gpu - oracle||_2 / ||oracle||_2."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def elem_rel(a, b):
    """SURVEY §8(c) C24's elementwise report: max |gpu - oracle| / (|oracle| + 1e-3 max|oracle|)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    if b.size == 0:
        return 0.0
    den = np.abs(b) + 1e-3 * max(np.abs(b).max(), 1e-300)
    return float(np.max(np.abs(a - b) / den))


def layer_slices(w):
    """Offsets of each layer's dW in the flat gradient (the library's layer order)."""
    out, off = [], 0
    for li in range(w.num_layers):
        n = (2 if w.model == "sage" else 1) * w.dims[li] * w.dims[li + 1]
        out.append(slice(off, off + n))
        off += n
    return out


_cache = {}


def inputs_for(name):
    if name not in _cache:
        w = WORKLOADS[name]
        inp = build_inputs(w)
        graph = dict(row_ptr=inp["row_ptr"], col=inp["col"], X=inp["X"][:, :w.feat_dim],
                     y=inp["y"], train=inp["train"])
        _cache.clear()
        _cache[name] = (w, inp, graph)
    return _cache[name]


def make_gpu(w, inp, use_graph=True, precision="fp32", batch_size=None, params=None, optimizer="sgd",
             exchange="auto"):
    from paper_2403_17092_b200 import Graph, Model
    g = Graph(inp["row_ptr"], inp["col"], inp["X"], inp["y"], w.num_classes, feat_dim=w.feat_dim)
    m = Model(g, model=w.model, sampler=w.sampler, num_layers=w.num_layers, hidden=w.hidden,
              batch_size=batch_size or w.batch_size, fanouts=w.fanouts, precision=precision,
              use_graph=use_graph, lr=w.lr, seed=w.sampler_seed, init_seed=w.init_seed, optimizer=optimizer)
    m.set_train_nodes(inp["train"])
    m.set_params(inp["params"] if params is None else params)
    if exchange != "auto":
        m.set_exchange(exchange)
    return g, m


def assert_blocks_equal(gpu_hops, ora_hops):
    assert len(gpu_hops) == len(ora_hops)
    for h, (a, b) in enumerate(zip(gpu_hops, ora_hops)):
        for k in ("n_dst", "n_src", "n_edges"):
            assert a[k] == b[k], (h, k, a[k], b[k])
        for k in ("src_ids", "blk_rowptr", "blk_col", "blk_nbr"):
            assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), (h, k)


def kink_override(m, cache, w, b, precision="fp32"):
    """Reading R27: the ReLU mask is a floating-point decision.  Where the GPU's decision
    (sign of its H^(l)) differs from the oracle's, the unit must be kink-ambiguous:
    |Pre| <= 1e-5 * (|A| |W|)_uj, i.e. inside the fp32 rounding error of the GEMM; there
    both decisions are correct results.  Returns the validated GPU decisions as an oracle
    mask override, and how many units differed."""
    ovr, n = {}, 0
    L = w.num_layers
    for li in range(L - 1):
        Pre = cache["Pre"][li]
        rows, out = Pre.shape
        H = m.activation(li, rows, out)
        gpu_pos = H > 0
        diff = gpu_pos != (Pre > 0)
        if w.sampler == "shadow" and li == L - 2:
            # DESIGN.md R19: layer L-1 is computed only on the rows the last layer reads (the
            # seeds and their in-neighbours in the induced block); the other rows are not outputs
            Ah = cache["Ahat"][L - 1].tocsr()
            keep = np.zeros(rows, dtype=bool)
            keep[:b] = True
            keep[Ah[:b].indices] = True
            diff &= keep[:, None]
        r, c = np.nonzero(diff)
        if r.size:
            S = (np.abs(cache["A"][li][r]) @ np.abs(cache["Ws"][li]))[np.arange(r.size), c]
            assert np.all(np.abs(Pre[r, c]) <= KINK[precision] * S), \
                ("ReLU decision differs at a unit that is not kink-ambiguous", li, np.abs(Pre[r, c]).max())
            assert r.size <= 4 + MAX_FLIP_SHARE[precision] * Pre.size, \
                ("too many kink-ambiguous ReLU decisions", li, r.size, Pre.size)
            ovr[li] = (r, c, gpu_pos[r, c])
            n += r.size
    return ovr, n


def check_train_step(m, w, graph, params, epoch, step, perm, loss, tol=None, precision="fp32"):
    """Compare one GPU step (already run) with the oracle step from `params` (the oracle's
    own trajectory).  Per tensor (C24): loss, logits, the whole gradient and EVERY layer's dW
    within `tol` (default: 1e-4 fp32, 2e-2 bf16-GEMM variant); the elementwise metric of C24 is
    reported in out["elem"].  Returns the oracle result (its params continue the trajectory)."""
    import oracle
    from oracle import sampling as OS
    tol = tol if tol is not None else (TOL_FP32 if precision == "fp32" else TOL_BF16)
    out = oracle.train_step(w, graph, params, epoch, step, 1, perm=perm, keep_cache=True)
    b = len(OS.batch_seeds(perm, w.batch_size, step))
    logits = m.logits(b, w.num_classes)
    err = dict(loss=abs(loss - out["loss"]) / abs(out["loss"]),
               logits=rel(logits, out["logits"][0]))
    ovr, nflip = kink_override(m, out["caches"][0], w, b, precision)
    gref = out["grad"]
    if nflip:
        gref = oracle.train_step(w, graph, params, epoch, step, 1, perm=perm, mask_override=[ovr])["grad"]
    grads = m.grads()
    err["grad"] = rel(grads, gref)
    elem = dict(logits=elem_rel(logits, out["logits"][0]), grad=elem_rel(grads, gref))
    for li, sl in enumerate(layer_slices(w)):
        err[f"dW{li + 1}"] = rel(grads[sl], gref[sl])
        elem[f"dW{li + 1}"] = elem_rel(grads[sl], gref[sl])
    for k, v in err.items():
        assert v <= tol, (step, k, v, nflip)
    out["errors"], out["elem"], out["kink_flips"] = err, elem, nflip
    out["caches"] = None
    return out
