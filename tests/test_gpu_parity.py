"""CUDA path (through the C-ABI) vs the oracle, element by element, on the same seeded
inputs.  Integer work (sampling, relabel, induce) bit-exact; fp32 loss/logits/grads within
1e-4 relative (per-tensor L2, R24)."""
import numpy as np
import pytest

import oracle
from oracle import sampling as OS
from tests.gpu_common import (TOL_BF16, TOL_FP32, assert_blocks_equal, check_train_step, inputs_for, make_gpu,
                              rel)

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------- configs[0] tiny
def test_tiny_sampling_all_batches_bitexact():
    w, inp, graph = inputs_for("tiny")
    g, m = make_gpu(w, inp)
    for epoch, batches in ((0, range(157)), (1, (0, 156))):
        perm = OS.epoch_perm(graph["train"], w.sampler_seed, epoch)
        for b in batches:
            want, _ = oracle.sample_batch(w, graph, epoch, b, perm)
            assert_blocks_equal(m.sample(epoch, b), want)


@pytest.mark.parametrize("use_graph", [True, False])
def test_tiny_epoch_training_parity(use_graph):
    w, inp, graph = inputs_for("tiny")
    g, m = make_gpu(w, inp, use_graph=use_graph)
    params = inp["params"].astype(np.float64)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    worst, flips = 0.0, 0
    for step in range(w.n_batches):
        loss = m.train_minibatch(0, step)
        out = check_train_step(m, w, graph, params, 0, step, perm, loss)
        worst = max(worst, max(out["errors"].values()))
        flips += out["kink_flips"]
        params = out["params"]
    assert rel(m.get_params(), params) <= TOL_FP32
    print(f"worst per-step rel err {worst:.2e}, kink-ambiguous ReLU decisions {flips}")


def test_tiny_epoch_training_parity_l1_on_sampler(monkeypatch):
    """Layer 1's gather on the sampling stream (GS_L1_ON_SAMPLER=1): every step of a whole epoch
    within tolerance of the oracle, then gnn_train_epoch of the next epoch."""
    monkeypatch.setenv("GS_L1_ON_SAMPLER", "1")
    w, inp, graph = inputs_for("tiny")
    g, m = make_gpu(w, inp)
    params = inp["params"].astype(np.float64)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    for step in range(w.n_batches):
        loss = m.train_minibatch(0, step)
        out = check_train_step(m, w, graph, params, 0, step, perm, loss)
        params = out["params"]
    assert rel(m.get_params(), params) <= TOL_FP32
    st = m.train_epoch(1)
    assert st["steps"] == w.n_batches


def test_tiny_determinism_and_graph_equals_eager():
    w, inp, graph = inputs_for("tiny")
    runs = []
    for use_graph in (True, True, False):
        g, m = make_gpu(w, inp, use_graph=use_graph)
        losses = [m.train_minibatch(0, s) for s in range(5)]
        runs.append((np.array(losses), m.grads(), m.get_params()))
        m.close(); g.close()
    for r in runs[1:]:
        for a, b in zip(runs[0], r):
            assert np.array_equal(a, b)


def test_tiny_e2e_host_call_equals_device_call():
    w, inp, graph = inputs_for("tiny")
    g1, m1 = make_gpu(w, inp)
    g2, m2 = make_gpu(w, inp)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    for step in range(3):
        seeds = OS.batch_seeds(perm, w.batch_size, step)
        l1 = m1.train_minibatch(0, step)
        l2 = m2.train_batch_host(seeds, len(seeds), 0, step)
        assert l1 == l2
    assert np.array_equal(m1.get_params(), m2.get_params())


def test_tiny_overlap_is_invisible():
    """Sampling step s+1 on the sampling stream while step s trains (two batch sets) gives
    bit-identical results to sample-then-train, also when the caller interleaves parity
    samples, jumps steps, or changes epoch mid-way."""
    w, inp, graph = inputs_for("tiny")
    schedule = [(0, s) for s in range(6)] + [(0, 9), (0, 10), (1, 0), (1, 1), (0, 3)]
    runs = []
    for overlap in (False, True):
        g, m = make_gpu(w, inp)
        m.set_overlap(overlap)
        losses = []
        for i, (e, s) in enumerate(schedule):
            losses.append(m.train_minibatch(e, s))
            if i == 3:
                m.sample(0, 5)              # parity hook between steps clobbers a set
        runs.append((np.array(losses), m.grads(), m.get_params()))
        m.close(); g.close()
    for a, b in zip(*runs):
        assert np.array_equal(a, b)


def test_tiny_e2e_prefetch_equals_plain():
    w, inp, graph = inputs_for("tiny")
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    seeds = [OS.batch_seeds(perm, w.batch_size, s) for s in range(5)]
    g1, m1 = make_gpu(w, inp)
    g2, m2 = make_gpu(w, inp)
    for s in range(5):
        l1 = m1.train_batch_host(seeds[s], len(seeds[s]), 0, s)
        nxt = dict(next_seeds=seeds[s + 1], next_b_total=len(seeds[s + 1]), next_g=s + 1) if s < 4 else {}
        l2 = m2.train_batch_host(seeds[s], len(seeds[s]), 0, s, **nxt)
        assert l1 == l2
    assert np.array_equal(m1.get_params(), m2.get_params())


def test_tiny_virtual_ranks_inactive_rank_and_ragged_step():
    """A rank with no batch (g >= n_batches) contributes zero gradient; b_total counts only
    the active seeds (reading R8/R9).  Emulated on one GPU through the e2e call."""
    w, inp, graph = inputs_for("tiny")
    g, m = make_gpu(w, inp)
    loss = m.train_batch_host(np.zeros(0, np.int32), 16, 0, 157)
    assert loss == 0.0 and np.all(m.grads() == 0)
    assert np.array_equal(m.get_params(), inp["params"])
    # ragged last batch (16 seeds) at world 4: b_total = 16
    out = oracle.train_step(w, graph, inp["params"], 0, 39, 4)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    seeds = OS.batch_seeds(perm, w.batch_size, 156)
    loss = m.train_batch_host(seeds, 16, 0, 156)
    assert abs(loss - out["rank_losses"][0]) <= TOL_FP32 * abs(out["rank_losses"][0])
    assert rel(m.grads(), out["grad"]) <= TOL_FP32


def test_degenerate_batches():
    """Batch of one seed; isolated seeds (degree 0 -> no edges, mean = 0)."""
    w, inp, graph = inputs_for("tiny")
    rp = inp["row_ptr"].copy()
    # a graph where nodes 0..9 are isolated: drop their rows' entries and references to them
    import gnn_inputs
    n = w.num_nodes
    rows = np.repeat(np.arange(n), np.diff(rp))
    col = inp["col"]
    keep = (rows >= 10) & (col >= 10)
    rp2 = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows[keep], minlength=n), out=rp2[1:])
    inp2 = dict(inp, row_ptr=rp2, col=col[keep].astype(np.int32))
    graph2 = dict(graph, row_ptr=rp2, col=inp2["col"])
    g, m = make_gpu(w, inp2)
    for seeds in (np.array([3], np.int32), np.array([0, 1, 2, 500], np.int32), np.array([77], np.int32)):
        loss = m.train_batch_host(seeds, len(seeds), 0, 0)
        hops = OS.neighbor_sample(rp2, inp2["col"], seeds, list(w.fanouts), w.sampler_seed, 0, 0)
        from oracle import model as M
        blocks, ids = M.layer_blocks(hops, "neighbor", w.num_layers)
        Ws = M.unflatten(inp["params"], w.dims, "sage")
        l_or, grads, _ = M.minibatch_grad(Ws, "sage", blocks, ids, graph["X"], graph["y"][seeds],
                                          len(seeds), len(seeds))
        m.set_params(inp["params"])      # undo the SGD step for the next case
        assert abs(loss - l_or) <= TOL_FP32 * abs(l_or)
        assert rel(m.grads(), M.flatten(grads)) <= TOL_FP32


def test_epoch_permutation_bitexact():
    w, inp, graph = inputs_for("tiny")
    g, m = make_gpu(w, inp)
    for epoch in (0, 1, 7):
        assert np.array_equal(m.epoch_permutation(epoch), OS.epoch_perm(graph["train"], w.sampler_seed, epoch))


# ---------------------------------------------------------------- the rest of the model x sampler grid
# (Table 3: GCN and SAGE under both samplers, and
# the ShaDow depth setting L = 5 layers on L' = 2 hops)
@pytest.mark.parametrize("name,transpose", [("tiny_gcn", 0), ("tiny_sage_shadow", 0), ("tiny_shadow_l5", 0),
                                            ("tiny_sage_shadow", 1), ("tiny_shadow_l5", 1)])
def test_grid_sampling_and_training_parity(name, transpose, monkeypatch):
    """transpose=1: the ShaDow backward over an explicitly built, sorted transposed block (the
    path of non-symmetric graphs) instead of the symmetric block itself."""
    w, inp, graph = inputs_for(name)
    monkeypatch.setenv("GS_SHADOW_TRANSPOSE", str(transpose))
    g, m = make_gpu(w, inp)
    assert g.symmetric          # the generator's graphs are symmetric (Chung-Lu, both directions)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    for b in (0, 1, w.n_batches - 1):
        want, _ = oracle.sample_batch(w, graph, 0, b, perm)
        got = m.sample(0, b)
        if w.sampler == "shadow":
            assert_blocks_equal(got[0], want[0])
            assert_blocks_equal([got[1]], [want[1]])
        else:
            assert_blocks_equal(got, want)
    params = inp["params"].astype(np.float64)
    for step in list(range(12)) + [w.n_batches - 1]:
        if step == w.n_batches - 1:
            m.set_params(params)          # ragged last batch from the oracle's current params
        loss = m.train_minibatch(0, step)
        out = check_train_step(m, w, graph, params, 0, step, perm, loss)
        params = out["params"]
        assert rel(m.get_params(), params) <= TOL_FP32


def test_symmetry_check():
    """gnn_graph_symmetric: the device check against a host brute force on a symmetric graph and
    on the same graph with one reverse entry removed."""
    from paper_2403_17092_b200 import Graph
    w, inp, graph = inputs_for("tiny")
    rp, col = inp["row_ptr"], inp["col"]
    g = Graph(rp, col, inp["X"], inp["y"], w.num_classes, feat_dim=w.feat_dim)
    assert g.symmetric
    g.close()
    # drop the first entry of row v (v -> u): row u still lists v, so the graph is not symmetric
    v = int(np.nonzero(np.diff(rp) > 0)[0][0])
    keep = np.ones(col.shape[0], dtype=bool)
    keep[rp[v]] = False
    rp2 = rp.copy()
    rp2[v + 1:] -= 1
    g2 = Graph(rp2, col[keep], inp["X"], inp["y"], w.num_classes, feat_dim=w.feat_dim)
    assert not g2.symmetric


# ---------------------------------------------------------------- NEXT-4: Adam
@pytest.mark.parametrize("name", ["tiny", "tiny_gcn"])
def test_adam_training_parity(name):
    """Adam on the device (fused with the split-K reduce and the weight repack) against the
    oracle's Adam (oracle.model.adam, pinned to torch.optim.Adam) applied to the oracle's own
    gradients: 20 steps and the ragged last batch; loss/logits/grads per step and the
    parameters after every update within 1e-4."""
    from oracle import model as OM
    w, inp, graph = inputs_for(name)
    g, m = make_gpu(w, inp, optimizer="adam")
    params = inp["params"].astype(np.float64)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    state = {}
    for step in list(range(20)) + [w.n_batches - 1]:
        loss = m.train_minibatch(0, step)
        out = check_train_step(m, w, graph, params, 0, step, perm, loss)
        Ws = OM.unflatten(params, w.dims, w.model)
        G = OM.unflatten(out["grad"], w.dims, w.model)
        params = OM.flatten(OM.adam(Ws, G, state, w.lr))
        assert rel(m.get_params(), params) <= TOL_FP32, step


# ---------------------------------------------------------------- NEXT-3: workload-aware batch assignment
@pytest.mark.parametrize("name", ["tiny", "tiny_sage_shadow"])
def test_workload_estimate_equals_oracle(name):
    """gnn_estimate_workload (the sampler run over the whole epoch) == the oracle's
    aggregation count of every batch."""
    from oracle import balance
    w, inp, graph = inputs_for(name)
    g, m = make_gpu(w, inp)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    got = m.estimate_workload(0)
    batches = range(w.n_batches) if name == "tiny" else (0, 1, w.n_batches - 1)
    for b in batches:
        s, _ = oracle.sample_batch(w, graph, 0, b, perm)
        assert got[b] == balance.workload(s, w.sampler, w.num_layers), b


def test_scheduled_training_parity():
    """With the balanced schedule (world = 1: step s trains batch order[s]) every step equals
    the oracle step on that batch, including the ragged last batch wherever it lands."""
    from oracle import balance
    from paper_2403_17092_b200 import plan_balanced
    w, inp, graph = inputs_for("tiny")
    g, m = make_gpu(w, inp)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    work = m.estimate_workload(0)
    order = plan_balanced(work, 1)
    assert list(order) == balance.plan(work, 1)
    m.set_schedule(order)
    params = inp["params"].astype(np.float64)
    ragged = int(np.nonzero(order == w.n_batches - 1)[0][0])
    for step in list(range(6)) + [ragged]:
        m.set_params(params)
        loss = m.train_minibatch(0, step)
        out = check_train_step(m, w, graph, params, 0, int(order[step]), perm, loss)
        params = out["params"]
        assert rel(m.get_params(), params) <= TOL_FP32
    m.set_schedule(None)


# ---------------------------------------------------------------- round 2: the parity holes of VERDICT r1
def test_tiny_bf16_gemm_epoch_parity():
    """The bf16-GEMM variant (BASELINE.json north_star: "a bf16-GEMM variant within 2e-2"): every
    step of the tiny epoch, loss / logits / every layer's dW within 2e-2 of the fp64 oracle, and
    the parameters after the epoch."""
    w, inp, graph = inputs_for("tiny")
    g, m = make_gpu(w, inp, precision="bf16")
    params = inp["params"].astype(np.float64)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    worst, flips = {}, 0
    for step in range(w.n_batches):
        loss = m.train_minibatch(0, step)
        out = check_train_step(m, w, graph, params, 0, step, perm, loss, precision="bf16")
        for k, v in out["errors"].items():
            worst[k] = max(worst.get(k, 0.0), v)
        flips += out["kink_flips"]
        params = out["params"]
    assert rel(m.get_params(), params) <= TOL_BF16
    print("bf16 worst per-step errors", {k: f"{v:.2e}" for k, v in worst.items()}, "flips", flips)


@pytest.mark.parametrize("use_graph", [True, False])
def test_exchange_nccl_one_rank_equals_fused(use_graph):
    """The multi-rank step branch (split-K reduce kernel -> ncclAllReduce -> update kernel) run on
    one GPU through a one-rank communicator: bit-identical to the fused one-rank path (same
    fixed-order reduce; a one-rank all-reduce is a copy), and within 1e-4 of the oracle."""
    w, inp, graph = inputs_for("tiny")
    runs = []
    for exch in ("auto", "nccl"):
        g, m = make_gpu(w, inp, use_graph=use_graph, exchange=exch)
        losses = [m.train_minibatch(0, s) for s in range(6)]
        runs.append((np.array(losses), m.grads(), m.get_params()))
        if exch == "nccl":
            assert m.launches_per_step >= 2 or not use_graph
        m.close(); g.close()
    for a, b in zip(*runs):
        assert np.array_equal(a, b)
    g, m = make_gpu(w, inp, use_graph=use_graph, exchange="nccl")
    params = inp["params"].astype(np.float64)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    for step in range(3):
        loss = m.train_minibatch(0, step)
        params = check_train_step(m, w, graph, params, 0, step, perm, loss)["params"]
        assert rel(m.get_params(), params) <= TOL_FP32


def test_train_epoch_matches_oracle_epoch():
    """gnn_train_epoch (all steps of an epoch, sampling of step s+1 overlapped with step s) against
    the oracle's epoch: mean loss and the parameters after epoch 0 and after epoch 1."""
    w, inp, graph = inputs_for("tiny")
    g, m = make_gpu(w, inp)
    params = inp["params"].astype(np.float64)
    for epoch in (0, 1):
        st = m.train_epoch(epoch)
        perm = OS.epoch_perm(graph["train"], w.sampler_seed, epoch)
        losses = []
        for step in range(w.n_batches):
            out = oracle.train_step(w, graph, params, epoch, step, 1, perm=perm)
            losses.append(out["loss"])
            params = out["params"]
        assert st["steps"] == w.n_batches and st["minibatches"] == w.n_batches
        assert abs(st["mean_loss"] - np.mean(losses)) <= TOL_FP32 * abs(np.mean(losses)), (st, np.mean(losses))
        assert rel(m.get_params(), params) <= TOL_FP32, epoch
        assert st["seconds"] > 0


def test_host_seeds_validated():
    """host seeds out of [0, N) -> RANGE, repeated -> PARAM, before any device work;
    the model stays usable."""
    from paper_2403_17092_b200.gnnstep import GnnError
    w, inp, graph = inputs_for("tiny")
    g, m = make_gpu(w, inp)
    for bad, code in ((np.array([3, w.num_nodes], np.int32), -1), (np.array([-1], np.int32), -1),
                      (np.array([5, 7, 5], np.int32), -2)):
        with pytest.raises(GnnError) as ei:
            m.train_batch_host(bad, len(bad), 0, 0)
        assert ei.value.code == code
    # a bad PREFETCH batch is refused too
    with pytest.raises(GnnError):
        m.train_batch_host(np.array([1, 2], np.int32), 2, 0, 0, next_seeds=np.array([9, 9], np.int32),
                           next_b_total=2, next_g=1)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    m.set_params(inp["params"])
    seeds = OS.batch_seeds(perm, w.batch_size, 0)
    loss = m.train_batch_host(seeds, len(seeds), 0, 0)
    check_train_step(m, w, graph, inp["params"].astype(np.float64), 0, 0, perm, loss)


def test_prefetched_set_not_reused_for_other_seeds():
    """a batch prefetched from the epoch permutation (train_minibatch) must not serve a
    host-seeded call with the same (epoch, g, n, b_total) but other seeds, and a host prefetch is
    reused only for the same seeds."""
    w, inp, graph = inputs_for("tiny")
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    other = np.ascontiguousarray(perm[::-1][:w.batch_size])      # 64 other seeds
    g1, m1 = make_gpu(w, inp)
    m1.train_minibatch(0, 0)          # prefetches step 1 (g = 1) from the permutation
    m1.set_params(inp["params"])
    l1 = m1.train_batch_host(other, len(other), 0, 1, next_seeds=perm[128:192], next_b_total=64, next_g=2)
    m1.set_params(inp["params"])
    l1b = m1.train_batch_host(other, len(other), 0, 2)       # same key as the prefetch, other seeds
    g2, m2 = make_gpu(w, inp)
    l2 = m2.train_batch_host(other, len(other), 0, 1)
    m2.set_params(inp["params"])
    l2b = m2.train_batch_host(other, len(other), 0, 2)
    assert l1 == l2 and l1b == l2b


def test_set_train_nodes_drops_schedule():
    """a schedule lists one split's batches; a new split drops it (no stale batch ids)."""
    w, inp, graph = inputs_for("tiny")
    g, m = make_gpu(w, inp)
    order = np.arange(w.n_batches)[::-1].copy()
    m.set_schedule(order)
    m.set_train_nodes(inp["train"][:1000])          # 16 batches now
    perm = OS.epoch_perm(inp["train"][:1000], w.sampler_seed, 0)
    loss = m.train_minibatch(0, 15)                 # the ragged last batch under the default rule
    graph2 = dict(graph, train=inp["train"][:1000])
    check_train_step(m, w, graph2, inp["params"].astype(np.float64), 0, 15, perm, loss)


def test_hub_row_beyond_block_sort():
    """A transposed row longer than the sampling kernel's shared-memory sort (8192 entries) takes
    its rank-counting fallback: node 0 is a neighbour of every node, the seeds
    keep all of their ~31 neighbours and so does hop 1 (fanout 32 >= degree), so node 0's row of the
    hop-1 transposed block holds every hop-1 destination (~30k).  Sampling bit-exact, one step
    within 1e-4."""
    from gnn_inputs import Workload, make_params
    from gnn_inputs.synth import feature_rows, make_labels
    n = 40_000
    rng = np.random.default_rng(5)
    a = np.concatenate([np.arange(1, n), np.repeat(np.arange(1, n), 15)])
    b = np.concatenate([np.zeros(n - 1, np.int64), rng.integers(1, n, size=15 * (n - 1))])
    keep = a != b
    a, b = a[keep], b[keep]
    keys = np.unique(np.concatenate([a * n + b, b * n + a]))
    rows, cols = keys // n, (keys % n).astype(np.int32)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rp[1:])
    w = Workload("hub", n, int(rp[-1]), 32, 8, "sage", "neighbor", (2, 32, 32), 3, 32, 1024, n)
    X = feature_rows(np.arange(n), 32, 7)
    inp = dict(row_ptr=rp, col=cols, X=X, y=make_labels(n, 8, 7), train=np.arange(n, dtype=np.int32),
               params=make_params(w.dims, "sage", 3))
    graph = dict(row_ptr=rp, col=cols, X=X, y=inp["y"], train=inp["train"])
    g, m = make_gpu(w, inp)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    want, _ = oracle.sample_batch(w, graph, 0, 0, perm)
    got = m.sample(0, 0)
    assert_blocks_equal(got, want)
    assert int(np.sum(want[1]["blk_nbr"] == 0)) > 8192      # node 0's transposed row at hop 1
    loss = m.train_minibatch(0, 0)
    check_train_step(m, w, graph, inp["params"].astype(np.float64), 0, 0, perm, loss)


@pytest.mark.parametrize("name", ["tiny", "tiny_gcn"])
def test_tiny_epoch_last_layer_fused(name, monkeypatch):
    """GS_LAST_FUSED=1 (the last layer on the CUDA cores; SAGE with its
    aggregation in the same kernel): every step of an epoch within tolerance of the oracle."""
    monkeypatch.setenv("GS_LAST_FUSED", "1")
    w, inp, graph = inputs_for(name)
    g, m = make_gpu(w, inp)
    params = inp["params"].astype(np.float64)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    for step in range(w.n_batches):
        loss = m.train_minibatch(0, step)
        params = check_train_step(m, w, graph, params, 0, step, perm, loss)["params"]
    assert rel(m.get_params(), params) <= TOL_FP32
