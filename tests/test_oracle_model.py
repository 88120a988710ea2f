"""Pins for oracle O4-O9.  CPU only."""
import math

import numpy as np
import pytest
import torch

import oracle
from oracle import model as M
from oracle import sampling as S


def _block(n_dst, n_src, rows):
    """rows: list (len n_dst) of lists of local src ids."""
    rp = np.zeros(n_dst + 1, dtype=np.int32)
    col = []
    for i, r in enumerate(rows):
        col += r
        rp[i + 1] = len(col)
    return dict(n_dst=n_dst, n_src=n_src, n_edges=len(col), blk_rowptr=rp,
                blk_col=np.asarray(col, dtype=np.int32), src_ids=np.arange(n_src, dtype=np.int32))


def _dense_adj(blk):
    A = np.zeros((blk["n_dst"], blk["n_src"]))
    rp, col = blk["blk_rowptr"], blk["blk_col"]
    for v in range(blk["n_dst"]):
        for e in range(rp[v], rp[v + 1]):
            A[v, col[e]] += 1.0
    return A


# ---------------------------------------------------------------- Â closed forms
def test_sage_mean_deg3_is_one_third():
    blk = _block(1, 4, [[1, 2, 3]])
    Ah = M.normalized_adjacency(blk, "sage").toarray()
    assert np.allclose(Ah, [[0, 1 / 3, 1 / 3, 1 / 3]], rtol=0, atol=1e-15)


def test_gcn_single_node_self_weight_one():
    blk = _block(1, 1, [[]])
    assert M.normalized_adjacency(blk, "gcn").toarray()[0, 0] == 1.0


def test_sage_forward_matches_dense_mean():
    rng = np.random.default_rng(0)
    blk = _block(4, 9, [[4, 5, 6], [], [0, 7, 8, 2], [3]])
    H = rng.standard_normal((9, 3))
    A = _dense_adj(blk)
    deg = A.sum(1, keepdims=True)
    mean = np.divide(A, deg, out=np.zeros_like(A), where=deg > 0) @ H
    W = rng.standard_normal((6, 2))
    want = H[:4] @ W[:3] + mean @ W[3:]                                      # Eq. (2)
    got = M.forward([W], "sage", [blk], H)["H"][-1]
    assert np.allclose(got, want, rtol=1e-13, atol=1e-13)


def test_gcn_symmetric_square_block_is_kipf_welling():
    # square symmetric block (as ShaDow produces): Â = D~^-1/2 (A+I) D~^-1/2, D~ = rowsum(A+I)
    rng = np.random.default_rng(1)
    n = 7
    A = np.zeros((n, n))
    for u in range(n):
        for v in range(u + 1, n):
            if rng.random() < 0.4:
                A[u, v] = A[v, u] = 1
    blk = _block(n, n, [list(np.nonzero(A[v])[0]) for v in range(n)])
    At = A + np.eye(n)
    Dm = np.diag(1 / np.sqrt(At.sum(1)))
    want = Dm @ At @ Dm
    got = M.normalized_adjacency(blk, "gcn").toarray()
    assert np.allclose(got, want, rtol=1e-14, atol=1e-15)


def _read_gcn_golden():
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "gcn_bipartite_block.txt")
    cases, cur = {}, None
    for ln in open(path):
        f = ln.split()
        if not f or f[0].startswith("#"):
            continue
        if f[0] in ("block", "star"):
            cur = cases.setdefault(f[0], dict(n_dst=int(f[1]), n_src=int(f[2]), want={}))
        elif f[0] in ("rowptr", "col"):
            cur[f[0]] = [int(x) for x in f[1:]]
        else:
            cur["want"][(int(f[1]), int(f[2]))] = float(f[3])
    return cases


@pytest.mark.parametrize("case", ["block", "star"])
def test_gcn_bipartite_block_golden(case):
    """Â of reading R12 on a bipartite block (and SPEC's star), against weights derived by hand in
    tests/golden/gcn_bipartite_block.txt.  A "+1 on every source out-degree" or a "self weight
    1/(deg_in+1)" misreading fails here (both change a hand-derived entry)."""
    c = _read_gcn_golden()[case]
    rp, col = c["rowptr"], c["col"]
    blk = _block(c["n_dst"], c["n_src"], [col[rp[v]:rp[v + 1]] for v in range(c["n_dst"])])
    got = M.normalized_adjacency(blk, "gcn").toarray()
    want = np.zeros_like(got)
    for (v, u), x in c["want"].items():
        want[v, u] = x
    assert len(c["want"]) == got.size or case == "star"
    assert np.allclose(got, want, rtol=1e-15, atol=1e-16)
    if case == "star":   # the documented deviation from SPEC.md normalize_block (line 186)
        spec = np.array([[1 / 4, 1 / math.sqrt(8), 1 / math.sqrt(8), 1 / math.sqrt(8)]])
        assert not np.allclose(got, spec)


# ---------------------------------------------------------------- O6
def test_ce_invariants_and_torch():
    C = 8
    loss, dZ = M.cross_entropy(np.zeros((5, C)), np.array([0, 1, 2, 3, 4]), 5)
    assert abs(loss - math.log(C)) < 1e-15
    assert np.allclose(dZ.sum(1), 0, atol=1e-16)
    rng = np.random.default_rng(2)
    Z = rng.standard_normal((6, 5)) * 30
    y = rng.integers(0, 5, 6)
    loss, dZ = M.cross_entropy(Z, y, 6)
    tz = torch.tensor(Z, dtype=torch.float64, requires_grad=True)
    tl = torch.nn.functional.cross_entropy(tz, torch.tensor(y), reduction="mean")
    tl.backward()
    assert abs(loss - tl.item()) < 1e-12
    assert np.allclose(dZ, tz.grad.numpy(), rtol=1e-12, atol=1e-14)
    assert np.allclose(dZ.sum(1), 0, atol=1e-15)


def test_zero_weights_give_ln_c(tiny_inputs):
    w, g = tiny_inputs
    p0 = np.zeros_like(g["params"])
    out = oracle.train_step(w, g, p0, 0, 0, 1)
    assert abs(out["loss"] - math.log(w.num_classes)) < 1e-12


def test_sgd_arithmetic():
    W = M.sgd([np.array([[1.0]])], [np.array([[0.5]])], 0.1)
    assert W[0][0, 0] == pytest.approx(0.95, abs=1e-15)
    W = M.sgd([np.array([[1.0]])], [np.array([[0.5]])], 0.0)
    assert W[0][0, 0] == 1.0


# ---------------------------------------------------------------- O7 finite differences
def _small_problem(model, sampler, seed=0):
    rng = np.random.default_rng(seed)
    n = 30
    edges = set()
    for u in range(n):
        for v in range(n):
            if u != v and rng.random() < 0.15:
                edges.add((u, v)); edges.add((v, u))
    rp = np.zeros(n + 1, dtype=np.int64)
    col = []
    for v in range(n):
        r = sorted(u for (a, u) in edges if a == v)
        col += r
        rp[v + 1] = len(col)
    col = np.asarray(col, dtype=np.int32)
    F, Hd, C = 5, 4, 3
    X = rng.standard_normal((n, F))
    y = rng.integers(0, C, n).astype(np.int32)
    seeds = np.array([2, 11, 19, 25], dtype=np.int32)
    dims = [F, Hd, C]
    if sampler == "neighbor":
        samp = S.neighbor_sample(rp, col, seeds, [3, 2], 4, 0, 0)
    else:
        samp = S.shadow_sample(rp, col, seeds, [3, 2], 2, 4, 0, 0)
    blocks, ids = M.layer_blocks(samp, sampler, 2)
    nparam = sum(r * c for r, c in M.layer_shapes(dims, model))
    flat = rng.standard_normal(nparam) * 0.7
    return dims, blocks, ids, X, y[seeds], len(seeds), flat


@pytest.mark.parametrize("model,sampler", [("sage", "neighbor"), ("gcn", "neighbor"),
                                           ("gcn", "shadow"), ("sage", "shadow")])
def test_backward_matches_central_differences(model, sampler):
    dims, blocks, ids, X, y, b, flat = _small_problem(model, sampler)

    def loss_of(f):
        Ws = M.unflatten(f, dims, model)
        return M.minibatch_grad(Ws, model, blocks, ids, X, y, b, b)[0]

    Ws = M.unflatten(flat, dims, model)
    loss, grads, cache = M.minibatch_grad(Ws, model, blocks, ids, X, y, b, b)
    g = M.flatten(grads)
    h = 1e-6
    fd = np.zeros_like(flat)
    for i in range(flat.size):
        fp, fm = flat.copy(), flat.copy()
        fp[i] += h
        fm[i] -= h
        fd[i] = (loss_of(fp) - loss_of(fm)) / (2 * h)
    # per-tensor relative L2 (R24) and elementwise
    assert np.linalg.norm(fd - g) <= 1e-6 * np.linalg.norm(g)
    assert np.allclose(fd, g, rtol=1e-4, atol=1e-8)
    # pre-activations away from kinks so FD is valid (h << |pre|)
    assert np.abs(cache["Pre"][0]).min() > 1e-4


# ---------------------------------------------------------------- O8 virtual ranks
def test_duplicated_batch_leaves_gradient_unchanged():
    dims, blocks, ids, X, y, b, flat = _small_problem("sage", "neighbor", 3)
    Ws = M.unflatten(flat, dims, "sage")
    _, g1, _ = M.minibatch_grad(Ws, "sage", blocks, ids, X, y, b, b)
    _, g2, _ = M.minibatch_grad(Ws, "sage", blocks, ids, X, y, b, 2 * b)
    G = M.allreduce([g2, g2])
    for a, c in zip(g1, G):
        assert np.allclose(a, c, rtol=1e-14, atol=1e-16)


def test_virtual_ranks_equal_weighted_single_rank(tiny_inputs):
    w, g = tiny_inputs
    perm = S.epoch_perm(g["train"], w.sampler_seed, 0)
    two = oracle.train_step(w, g, g["params"], 0, 3, 2, perm=perm)            # batches 6, 7
    a = oracle.train_step(w, g, g["params"], 0, 6, 1, perm=perm)
    b = oracle.train_step(w, g, g["params"], 0, 7, 1, perm=perm)
    ba, bb = a["b_total"], b["b_total"]
    want = (ba * a["grad"] + bb * b["grad"]) / (ba + bb)                       # P:L173 larger batch
    assert np.allclose(two["grad"], want, rtol=1e-12, atol=1e-15)
    assert two["loss"] == pytest.approx((ba * a["loss"] + bb * b["loss"]) / (ba + bb), rel=1e-12)


def test_ragged_last_step_inactive_ranks(tiny_inputs):
    w, g = tiny_inputs
    nb = oracle.n_batches(w.n_train, w.batch_size)          # 157 = 156*64 + 16
    assert nb == 157
    out = oracle.train_step(w, g, g["params"], 0, 39, 4)    # g = 156..159: only 156 active
    assert out["b_total"] == 16
    assert all(np.all(r == 0) for r in out["rank_grads"][1:])


# ---------------------------------------------------------------- NEXT-4: Adam
def test_adam_matches_torch_optim_adam():
    """The oracle's Adam against the library routine the paper's listings call
    (torch.optim.Adam, float64 on CPU), five steps on random weights and gradients."""
    rng = np.random.default_rng(5)
    Ws = [rng.standard_normal((6, 4)), rng.standard_normal((8, 3))]
    grads = [[rng.standard_normal(W.shape) * 10.0 ** rng.integers(-3, 2) for W in Ws] for _ in range(5)]
    tp = [torch.tensor(W.copy(), dtype=torch.float64, requires_grad=True) for W in Ws]
    opt = torch.optim.Adam(tp, lr=0.01, betas=(0.9, 0.999), eps=1e-8)
    state, cur = {}, Ws
    for G in grads:
        cur = M.adam(cur, G, state, 0.01)
        for p, g in zip(tp, G):
            p.grad = torch.tensor(g, dtype=torch.float64)
        opt.step()
    for a, p in zip(cur, tp):
        assert np.allclose(a, p.detach().numpy(), rtol=1e-12, atol=1e-14)


def test_adam_first_step_closed_form():
    """t = 1: m/(1-b1) = g and v/(1-b2) = g^2, so each weight moves by lr*g/(|g|+eps)
    (= lr*sign(g) up to eps), and a zero gradient leaves the weight unchanged."""
    g = np.array([[3.0, -0.5, 0.0, 1e-3]])
    W = np.zeros_like(g)
    state = {}
    out = M.adam([W], [g], state, lr=0.1)[0]
    assert np.allclose(out, -0.1 * g / (np.abs(g) + 1e-8), rtol=1e-12, atol=0)
    assert out[0, 2] == 0.0 and state["t"] == 1


# ---------------------------------------------------------------- NEXT-3: workload-aware assignment
def _partitions(items, size):
    """All ways to split `items` into groups of `size` (the last group may be smaller)."""
    if len(items) <= size:
        yield [items]
        return
    import itertools
    first, rest = items[0], items[1:]
    for comb in itertools.combinations(rest, size - 1):
        group = [first, *comb]
        left = [x for x in rest if x not in comb]
        for p in _partitions(left, size):
            yield [group] + p


def test_balanced_plan_is_optimal_by_brute_force():
    """Sorted consecutive grouping minimises Σ_steps max work (exchange argument); pinned by
    enumerating every grouping of up to 8 batches into steps of P = 2 and 3 (when P divides n,
    so that every step has P batches)."""
    from oracle import balance
    rng = np.random.default_rng(3)
    for n, P in ((4, 2), (6, 2), (6, 3), (8, 2)):
        for _ in range(5):
            work = rng.integers(1, 100, size=n)
            best = min(sum(max(work[i] for i in g) for g in part) for part in _partitions(list(range(n)), P))
            order = balance.plan(work, P)
            assert sorted(order) == list(range(n))
            assert balance.makespan(order, work, P) == best


def test_balanced_plan_never_worse_than_round_robin():
    from oracle import balance
    rng = np.random.default_rng(4)
    for _ in range(50):
        n, P = int(rng.integers(1, 60)), int(rng.integers(1, 9))
        work = rng.pareto(1.5, size=n) * 100 + 1
        work = work.astype(np.int64)
        assert balance.makespan(balance.plan(work, P), work, P) <= balance.makespan(list(range(n)), work, P)


def test_workload_closed_form_when_every_degree_exceeds_fanout():
    """On a complete graph K_n every frontier node has degree n-1 >= k, so hop h samples exactly
    k_h edges per destination: workload = Σ_h n_dst(h) * k_h (SPEC-style closed form)."""
    from oracle import balance
    n = 40
    row_ptr = np.arange(0, n * (n - 1) + 1, n - 1, dtype=np.int64)
    col = np.array([u for v in range(n) for u in range(n) if u != v], dtype=np.int32)
    fan = [4, 3]                      # input-layer-first: seeds sample 3, then 4
    seeds = np.array([0, 5, 7], dtype=np.int32)
    hops = S.neighbor_sample(row_ptr, col, seeds, fan, 1, 0, 0)
    want = hops[0]["n_dst"] * 3 + hops[1]["n_dst"] * 4
    assert balance.workload(hops, "neighbor", 2) == want


def test_library_planner_matches_oracle_plan():
    """gnn_plan_balanced (host-only C++ in libgnnstep.so) == the oracle's plan."""
    from oracle import balance
    from paper_2403_17092_b200 import plan_balanced
    rng = np.random.default_rng(6)
    for _ in range(40):
        n, P = int(rng.integers(0, 300)), int(rng.integers(1, 9))
        work = rng.integers(0, 50, size=n).astype(np.int64)   # many ties
        assert list(plan_balanced(work, P)) == balance.plan(work, P), (n, P)


def test_formula_recompute_feature_mode(tiny_inputs):
    """The oracle's formula-recompute mode (X given as a function of the row ids, used for
    configs[4] whose 57 GB table is never on the host) gives exactly the array mode's step."""
    from gnn_inputs import feature_rows
    w, inp = tiny_inputs
    graph = dict(row_ptr=inp["row_ptr"], col=inp["col"], X=inp["X"][:, :w.feat_dim], y=inp["y"], train=inp["train"])
    a = oracle.train_step(w, graph, inp["params"], 0, 3, 1)
    graph_f = dict(graph, X=lambda ids: feature_rows(ids, w.feat_dim, w.graph_seed))
    b = oracle.train_step(w, graph_f, inp["params"], 0, 3, 1)
    assert a["loss"] == b["loss"] and np.array_equal(a["grad"], b["grad"])
