"""The Unified CPU-GPU protocol on one B200 (§3):
rank 0 trains on the GPU (libgnnstep, GNN_EXCH_HOST: its step stops at the reduced gradient),
rank 1 on the host cores (libgnnhost); the gradients are summed by a gloo all-reduce and each rank
applies the update.  After 3 steps the GPU and host replicas are bitwise equal (same summed
gradient, the same fused-multiply-add update) and within 1e-4 of the oracle's synchronous steps
with two virtual ranks; also with unequal sub-batches (the workload ratio)."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle import model as OM
from oracle import sampling as OS
from tests.gpu_common import TOL_FP32, inputs_for, make_gpu, rel

pytestmark = pytest.mark.gpu
STEPS = 3


def _rank(rank, world, port, q, sizes):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2403_17092_b200.hostrank import HostModel
    from paper_2403_17092_b200.unified import GpuRank, unified_step
    w, inp, graph = inputs_for("tiny")
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    if rank == 0:
        g, m = make_gpu(w, inp)
        t = GpuRank(m, rank, world)
    else:
        t = HostModel(inp["row_ptr"], inp["col"], inp["X"], inp["y"], w.num_classes, w.feat_dim, model=w.model,
                      num_layers=w.num_layers, hidden=w.hidden, fanouts=w.fanouts, lr=w.lr, seed=w.sampler_seed)
        t.set_params(inp["params"])
    losses = [unified_step(t, perm, w.batch_size, 0, s, rank, world, sizes) for s in range(STEPS)]
    params = t.m.get_params() if rank == 0 else t.get_params()
    q.put((rank, params, losses))
    dist.barrier()
    dist.destroy_process_group()


def _run(sizes):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29100 + os.getpid() % 700 + (0 if sizes is None else 1)
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q, sizes)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, p, l = q.get(timeout=600)
        res[r] = (p, l)
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    return res


def _oracle_steps(sizes):
    """The oracle's synchronous steps with the unified sub-batch rule (gradients of each rank's
    slice summed, then SGD)."""
    from paper_2403_17092_b200.unified import step_slice
    w, inp, graph = inputs_for("tiny")
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    params = inp["params"].astype(np.float64)
    losses = []
    for s in range(STEPS):
        Ws = OM.unflatten(params, w.dims, w.model)
        G, tot = None, 0.0
        for r in range(2):
            g, seeds, bt = step_slice(perm, sizes, s, r)
            smp = OS.neighbor_sample(graph["row_ptr"], graph["col"], seeds, list(w.fanouts), w.sampler_seed, 0, g)
            blocks, ids = OM.layer_blocks(smp, w.sampler, w.num_layers)
            loss, grads, _ = OM.minibatch_grad(Ws, w.model, blocks, ids, graph["X"], graph["y"][seeds], len(seeds), bt)
            G = grads if G is None else [a + b for a, b in zip(G, grads)]
            tot += loss
        params = OM.flatten(OM.sgd(Ws, G, w.lr))
        losses.append(tot)
    return params, losses


@pytest.mark.parametrize("sizes", [None, [56, 8]])
def test_gpu_rank_plus_host_rank(sizes):
    w, inp, graph = inputs_for("tiny")
    res = _run(sizes)
    assert np.array_equal(res[0][0], res[1][0])   # the two replicas hold identical bits
    want_p, want_l = _oracle_steps(sizes or [w.batch_size, w.batch_size])
    for s in range(STEPS):
        got = res[0][1][s] + res[1][1][s]
        assert abs(got - want_l[s]) <= TOL_FP32 * abs(want_l[s]), (s, got, want_l[s])
    assert rel(res[0][0], want_p) <= TOL_FP32
    if sizes is None:   # equal sub-batches = the engine's rule = oracle.train_step with 2 virtual ranks
        params = inp["params"].astype(np.float64)
        perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
        for s in range(STEPS):
            params = oracle.train_step(w, graph, params, 0, s, 2, perm=perm)["params"]
        assert rel(res[0][0], params) <= TOL_FP32
