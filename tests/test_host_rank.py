"""The host-core trainer rank (include/gnnhost.h, §3 lines
225-246) against the oracle, on the host (no GPU): the epoch permutation and every hop's source
ids bit-exact, the mini-batch gradient and loss within the fp32 tolerance, the update's
arithmetic, inactive ranks, argument errors; and a world-2 gloo run of two host ranks (the
Unified protocol's synchronous SGD with a host-side all-reduce) equal to the oracle's step with
two virtual ranks."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle import model as OM
from oracle import sampling as OS
from gnn_inputs import WORKLOADS, build_inputs
from paper_2403_17092_b200.hostrank import HostError, HostModel

TOL = 1e-4


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


_cache = {}


def setup(name):
    if name not in _cache:
        w = WORKLOADS[name]
        inp = build_inputs(w)
        graph = dict(row_ptr=inp["row_ptr"], col=inp["col"], X=inp["X"][:, :w.feat_dim], y=inp["y"],
                     train=inp["train"])
        _cache[name] = (w, inp, graph)
    return _cache[name]


def host_model(w, inp):
    hm = HostModel(inp["row_ptr"], inp["col"], inp["X"], inp["y"], w.num_classes, w.feat_dim, model=w.model,
                   num_layers=w.num_layers, hidden=w.hidden, fanouts=w.fanouts, lr=w.lr, seed=w.sampler_seed)
    hm.set_params(inp["params"])
    return hm


def oracle_grad(w, graph, params, seeds, b_total, epoch, g):
    s = OS.neighbor_sample(graph["row_ptr"], graph["col"], seeds, list(w.fanouts), w.sampler_seed, epoch, g)
    blocks, ids = OM.layer_blocks(s, w.sampler, w.num_layers)
    Ws = OM.unflatten(np.asarray(params, np.float64), w.dims, w.model)
    loss, grads, _ = OM.minibatch_grad(Ws, w.model, blocks, ids, graph["X"], graph["y"][seeds], len(seeds), b_total)
    return s, loss, OM.flatten(grads)


def test_host_epoch_permutation_bitexact():
    w, inp, graph = setup("tiny")
    hm = host_model(w, inp)
    for epoch in (0, 1, 7):
        assert np.array_equal(hm.epoch_permutation(graph["train"], epoch),
                              OS.epoch_perm(graph["train"], w.sampler_seed, epoch))


@pytest.mark.parametrize("name", ["tiny", "tiny_gcn"])
def test_host_grads_match_oracle(name):
    """Sampled source ids bit-exact per hop; loss and gradient (every layer) within 1e-4, on a
    full batch, a partial batch scaled by a larger b_total, and the ragged last batch."""
    w, inp, graph = setup(name)
    hm = host_model(w, inp)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    last = oracle.n_batches(len(graph["train"]), w.batch_size) - 1
    for g, b_total in ((0, w.batch_size), (3, 3 * w.batch_size), (last, None)):
        seeds = OS.batch_seeds(perm, w.batch_size, g)
        bt = len(seeds) if b_total is None else b_total
        grad, loss = hm.grads(seeds, bt, 0, g)
        s, oloss, ograd = oracle_grad(w, graph, inp["params"], seeds, bt, 0, g)
        for h, hop in enumerate(s):
            assert np.array_equal(hm.last_src_ids(h), hop["src_ids"]), (g, h)
        assert abs(loss - oloss) <= TOL * abs(oloss), (g, loss, oloss)
        assert rel(grad, ograd) <= TOL, (g, rel(grad, ograd))
        off = 0
        for r, c in OM.layer_shapes(w.dims, w.model):   # every layer's block on its own
            n = r * c
            assert rel(grad[off:off + n], ograd[off:off + n]) <= TOL, (g, off)
            off += n


def test_host_apply_is_fma_sgd_and_inactive_rank():
    w, inp, graph = setup("tiny")
    hm = host_model(w, inp)
    rng = np.random.default_rng(0)
    G = rng.standard_normal(hm.param_count).astype(np.float32)
    p0 = hm.get_params()
    hm.apply(G)
    want = (p0.astype(np.float64) - np.float64(np.float32(w.lr)) * G.astype(np.float64)).astype(np.float32)
    # one rounding of the exact p - lr*g (a fused multiply-add)
    assert np.array_equal(hm.get_params(), want)
    g0, l0 = hm.grads(np.zeros(0, np.int32), 5, 0, 0)
    assert l0 == 0.0 and not g0.any()


def test_host_argument_errors():
    w, inp, graph = setup("tiny")
    hm = host_model(w, inp)
    with pytest.raises(HostError) as e:
        hm.grads(np.array([0, w.num_nodes], np.int32), 2, 0, 0)
    assert e.value.code == -1
    with pytest.raises(HostError) as e:
        hm.grads(np.array([4, 4], np.int32), 2, 0, 0)
    assert e.value.code == -2
    with pytest.raises(HostError) as e:
        hm.grads(np.array([1, 2, 3], np.int32), 2, 0, 0)
    assert e.value.code == -2
    with pytest.raises(HostError):
        hm.set_params(np.zeros(3, np.float32))


def _two_host_ranks(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from paper_2403_17092_b200.unified import unified_step
    w, inp, graph = setup("tiny")
    hm = host_model(w, inp)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    losses = []
    for step in range(3):
        losses.append(unified_step(hm, perm, w.batch_size, 0, step, rank, world))
    q.put((rank, hm.get_params(), losses))
    dist.barrier()
    dist.destroy_process_group()


def test_two_host_ranks_gloo_equal_oracle_virtual_ranks():
    """World 2 over gloo: rank r trains batch g = 2s + r with the host trainer, the gradients are
    summed by all_reduce, both ranks apply the same update: after 3 steps the two replicas are
    bitwise equal and within 1e-4 of the oracle's steps with two virtual ranks."""
    w, inp, graph = setup("tiny")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 500
    procs = [ctx.Process(target=_two_host_ranks, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    res = {r: (p, l) for r, p, l in res}
    assert np.array_equal(res[0][0], res[1][0])
    params = inp["params"].astype(np.float64)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    for step in range(3):
        o = oracle.train_step(w, graph, params, 0, step, 2, perm=perm)
        assert abs(res[0][1][step] + res[1][1][step] - o["loss"]) <= TOL * abs(o["loss"])
        params = o["params"]
    assert rel(res[0][0], params) <= TOL
