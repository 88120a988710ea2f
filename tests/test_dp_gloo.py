"""Data-parallel host logic at world size 2 on CPU (gloo): the engine's batch -> rank plan
(gnn_plan_step), the unique-id broadcast the NCCL communicator is built from, and the
synchronous-SGD gradient semantics (§2.2; R8/R9) with a
real all-reduce over the process group."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, queue):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        queue.put((rank, fn(rank, world)))
    except Exception as e:  # surface worker failures in the parent
        queue.put((rank, e))
    finally:
        dist.destroy_process_group()


def _run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return out


def _plan_and_uid(rank, world):
    from paper_2403_17092_b200 import comm_get_unique_id, plan_step, steps_per_epoch
    from gnn_inputs import WORKLOADS
    w = WORKLOADS["tiny"]
    obj = [comm_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    uid = obj[0]
    S = steps_per_epoch(w.n_train, w.batch_size, world)
    mine = [plan_step(w.n_train, w.batch_size, world, rank, s) for s in range(S)]
    allp = [None] * world
    dist.all_gather_object(allp, (uid, mine))
    return allp


def test_plan_and_unique_id_world2():
    out = _run(_plan_and_uid)
    from gnn_inputs import WORKLOADS
    import oracle
    w = WORKLOADS["tiny"]
    allp = out[0]
    assert allp == out[1]
    uids = {p[0] for p in allp}
    assert len(uids) == 1 and len(next(iter(uids))) == 128
    plans = [p[1] for p in allp]
    S = len(plans[0])
    assert S == (w.n_batches + 1) // 2
    seen = []
    for s in range(S):
        g0, n0, off0, bt0 = plans[0][s]
        g1, n1, off1, bt1 = plans[1][s]
        assert (g0, g1) == (2 * s, 2 * s + 1)
        assert bt0 == bt1 == n0 + n1                       # b_total = seeds of the step (R9)
        for g, n, off in ((g0, n0, off0), (g1, n1, off1)):
            if n:
                seen.append(g)
                assert off == g * w.batch_size
                assert n == min(w.batch_size, w.n_train - off)
    assert sorted(seen) == list(range(w.n_batches))         # every batch exactly once per epoch
    assert plans[1][S - 1][1] == 0                           # ragged last step: rank 1 idle
    # the oracle's virtual ranks agree on b_total
    g = None
    for s in (0, S - 1):
        import gnn_inputs
        inp = gnn_inputs.build_inputs(w)
        graph = dict(row_ptr=inp["row_ptr"], col=inp["col"], X=inp["X"], y=inp["y"], train=inp["train"])
        assert oracle.train_step(w, graph, inp["params"], 0, s, 2)["b_total"] == plans[0][s][3]


def _dp_grad(rank, world):
    """Each rank: the oracle gradient of ITS batch scaled by 1/b_total; SUM all-reduce."""
    import oracle
    from oracle import model as M
    from oracle import sampling as OS
    from paper_2403_17092_b200 import plan_step
    from gnn_inputs import WORKLOADS, build_inputs
    w = WORKLOADS["tiny"]
    inp = build_inputs(w)
    graph = dict(row_ptr=inp["row_ptr"], col=inp["col"], X=inp["X"], y=inp["y"], train=inp["train"])
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    Ws = M.unflatten(inp["params"], w.dims, w.model)
    res = []
    for step in (0, 5, 78):
        g, n, off, bt = plan_step(w.n_train, w.batch_size, world, rank, step)
        if n:
            seeds = perm[off:off + n]
            hops = OS.neighbor_sample(graph["row_ptr"], graph["col"], seeds, list(w.fanouts), w.sampler_seed, 0, g)
            blocks, ids = M.layer_blocks(hops, "neighbor", w.num_layers)
            _, grads, _ = M.minibatch_grad(Ws, w.model, blocks, ids, graph["X"], graph["y"][seeds], n, bt)
            flat = M.flatten(grads)
        else:
            flat = np.zeros(sum(W.size for W in Ws))
        t = torch.from_numpy(flat.copy())
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        res.append((step, t.numpy()))
    return res


def test_dp_gradient_allreduce_equals_union_batch():
    out = _run(_dp_grad)
    import oracle
    from gnn_inputs import WORKLOADS, build_inputs
    w = WORKLOADS["tiny"]
    inp = build_inputs(w)
    graph = dict(row_ptr=inp["row_ptr"], col=inp["col"], X=inp["X"], y=inp["y"], train=inp["train"])
    for (s0, g0), (s1, g1) in zip(out[0], out[1]):
        assert s0 == s1 and np.array_equal(g0, g1)            # identical on every rank
        want = oracle.train_step(w, graph, inp["params"], 0, s0, 2)["grad"]
        assert np.allclose(g0, want, rtol=1e-12, atol=1e-15)


def _balanced_plan(rank, world):
    """NEXT-3 host logic on every rank: the same workload vector (in training it comes from the
    sampler pass, identical on all ranks since keys use the global batch index) gives the same
    plan everywhere; each rank reads its batch of every step from it."""
    from paper_2403_17092_b200 import plan_balanced
    rng = np.random.default_rng(11)
    work = rng.pareto(1.2, size=157).astype(np.int64) * 100 + 1   # the tiny epoch's 157 batches, skewed
    order = [int(x) for x in plan_balanced(work, world)]
    S = (len(order) + world - 1) // world
    mine = [order[s * world + rank] if s * world + rank < len(order) else None for s in range(S)]
    allp = [None] * world
    dist.all_gather_object(allp, (order, mine))
    return allp


def test_balanced_schedule_world2():
    from oracle import balance
    out = _run(_balanced_plan)
    allp = out[0]
    assert allp == out[1]
    (order0, mine0), (order1, mine1) = allp
    assert order0 == order1                                      # every rank holds the same plan
    seen = [b for pair in zip(mine0, mine1) for b in pair if b is not None]
    assert sorted(seen) == list(range(157))                      # every batch exactly once
    rng = np.random.default_rng(11)
    work = rng.pareto(1.2, size=157).astype(np.int64) * 100 + 1
    assert order0 == balance.plan(work, 2)                       # the oracle's plan (R31)
    assert balance.makespan(order0, work, 2) <= balance.makespan(list(range(157)), work, 2)
