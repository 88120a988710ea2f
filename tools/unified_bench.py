"""The Unified CPU-GPU protocol measured on one B200 box (§3,
§4, §5.3): the host-core trainer's own speed (full batches, all host
cores), the workload ratio it implies, then synchronous steps of 1 GPU rank + 1 host rank over
gloo with that ratio, against the GPU rank alone.  Prints one JSON line.  Diagnostics, not the
bench contract.

  python tools/unified_bench.py [config] [steps]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _host_model(w, inp):
    from paper_2403_17092_b200.hostrank import HostModel
    hm = HostModel(inp["row_ptr"], inp["col"], inp["X"], inp["y"], w.num_classes, w.feat_dim, model=w.model,
                   num_layers=w.num_layers, hidden=w.hidden, fanouts=w.fanouts, lr=w.lr, seed=w.sampler_seed)
    hm.set_params(inp["params"])
    return hm


def _rank(rank, world, port, q, name, steps, sizes):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from gnn_inputs import WORKLOADS, build_inputs
    from paper_2403_17092_b200 import Graph, Model
    from paper_2403_17092_b200.unified import GpuRank, unified_step
    w = WORKLOADS[name]
    inp = build_inputs(w)
    if rank == 0:
        g = Graph(inp["row_ptr"], inp["col"], inp["X"], inp["y"], w.num_classes, feat_dim=w.feat_dim)
        m = Model(g, model=w.model, sampler=w.sampler, num_layers=w.num_layers, hidden=w.hidden,
                  batch_size=w.batch_size, fanouts=w.fanouts, lr=w.lr, seed=w.sampler_seed, init_seed=w.init_seed)
        m.set_train_nodes(inp["train"])
        m.set_params(inp["params"])
        t = GpuRank(m, rank, world)
        perm = m.epoch_permutation(0)
    else:
        t = _host_model(w, inp)
        perm = t.epoch_permutation(inp["train"], 0)
    for s in range(2):
        unified_step(t, perm, w.batch_size, 0, s, rank, world, sizes)
    dist.barrier()
    t0 = time.perf_counter()
    for s in range(2, 2 + steps):
        unified_step(t, perm, w.batch_size, 0, s, rank, world, sizes)
    dist.barrier()
    q.put((rank, time.perf_counter() - t0))
    dist.destroy_process_group()


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "products"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    from gnn_inputs import WORKLOADS, build_inputs
    from paper_2403_17092_b200.unified import ratio_sizes
    w = WORKLOADS[name]
    inp = build_inputs(w)
    # the host trainer's own speed on full batches (all host cores)
    hm = _host_model(w, inp)
    perm = hm.epoch_permutation(inp["train"], 0)
    hm.grads(perm[:w.batch_size], w.batch_size, 0, 0)
    t0 = time.perf_counter()
    nb = 3
    for g in range(1, 1 + nb):
        hm.grads(perm[g * w.batch_size:(g + 1) * w.batch_size], w.batch_size, 0, g)
    host_mbs = nb / (time.perf_counter() - t0)
    hm.close()
    # the GPU rank's speed: the bench's device-timed value (passed in, or a nominal default)
    gpu_mbs = float(os.environ.get("GPU_MBS", "4200"))
    sizes = ratio_sizes(w.batch_size, [gpu_mbs, host_mbs])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29900 + os.getpid() % 50
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q, name, steps, sizes)) for r in range(2)]
    for p in procs:
        p.start()
    secs = dict(q.get(timeout=3600) for _ in range(2))
    for p in procs:
        p.join()
    step_s = max(secs.values()) / steps
    print(json.dumps({"workload": name, "host_cores": os.cpu_count(), "omp_threads": torch.get_num_threads(),
                      "host_rank_full_batch_mini_batches_per_s": host_mbs, "gpu_rank_mini_batches_per_s": gpu_mbs,
                      "sub_batch_sizes": sizes, "unified_step_ms": step_s * 1e3,
                      "unified_global_batches_per_s": (sum(sizes) / w.batch_size) / step_s,
                      "gpu_only_step_ms": 1e3 / gpu_mbs,
                      "note": "1 GPU rank + 1 host rank, gloo all-reduce of the gradient every step"}))


if __name__ == "__main__":
    main()
