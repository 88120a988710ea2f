"""The world > 1 step for real: two trainer processes (ranks) on this GPU, each training its own
mini-batch (global batch g = step*2 + rank, §2.2 lines 173-175 synchronous SGD), with the
gradient exchanged by the library's one-shot peer-memory all-reduce (GNN_EXCH_PEER: CUDA-IPC
inboxes, summed in rank order inside the update).  Checks, every step: the parameters are
bit-identical on both ranks, and equal the oracle's 2-virtual-rank step within 1e-4 (loss of each
rank, the all-reduced gradient, the parameters); the ragged last step with an inactive rank."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, q, optimizer):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from oracle import model as OM
        from oracle import sampling as OS
        from tests.gpu_common import TOL_FP32, inputs_for, kink_override, make_gpu, rel
        w, inp, graph = inputs_for(name)
        g, m = make_gpu(w, inp, optimizer=optimizer)
        handles = [None] * world
        dist.all_gather_object(handles, m.exchange_export(rank, world))
        m.exchange_import(handles)
        m.set_exchange("peer")
        perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
        params = inp["params"].astype(np.float64)
        state = {}
        nsteps = (w.n_batches + world - 1) // world
        errs = []
        for step in list(range(6)) + [nsteps - 1]:
            if step == nsteps - 1:        # ragged last step (rank 1 inactive for tiny: 157 batches)
                m.set_params(params)
            loss = m.train_minibatch(0, step)
            out = oracle.train_step(w, graph, params, 0, step, world, perm=perm, keep_cache=True)
            # reading R27: ReLU decisions at kink-ambiguous units (validated per rank, exchanged)
            g_r = step * world + rank
            ovr = {}
            if g_r < w.n_batches:
                ovr, _ = kink_override(m, out["caches"][rank], w, len(OS.batch_seeds(perm, w.batch_size, g_r)))
            allo = [None] * world
            dist.all_gather_object(allo, ovr)
            if any(allo):
                out = oracle.train_step(w, graph, params, 0, step, world, perm=perm, mask_override=allo)
            if optimizer == "adam":
                Ws = OM.unflatten(params, w.dims, w.model)
                G = OM.unflatten(out["grad"], w.dims, w.model)
                new = OM.flatten(OM.adam(Ws, G, state, w.lr))
            else:
                new = out["params"]
            got = m.get_params()
            allp = [None] * world
            dist.all_gather_object(allp, got)
            assert all(np.array_equal(allp[0], p) for p in allp), "ranks disagree after the exchange"
            e = dict(loss=abs(loss - out["rank_losses"][rank]) / max(abs(out["rank_losses"][rank]), 1e-30)
                     if out["rank_losses"][rank] else abs(loss),
                     grad=rel(m.grads(), out["grad"]), params=rel(got, new))
            errs.append((step, e))
            for k, v in e.items():
                assert v <= TOL_FP32, (rank, step, k, v)
            params = new
        dist.barrier()
        m.close(); g.close()
        q.put((rank, errs))
    except Exception:
        import traceback
        q.put((rank, RuntimeError(traceback.format_exc())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,optimizer", [("tiny", "sgd"), ("tiny_gcn", "sgd"), ("tiny", "adam")])
def test_two_ranks_peer_exchange_matches_oracle(name, optimizer):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q, optimizer)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for r, v in res.items():
        if isinstance(v, Exception):
            raise v
        print("rank", r, v[-1])
