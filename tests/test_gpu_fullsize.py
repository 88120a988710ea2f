"""Full-size parity (BASELINE.json configs[1..3]) in the launch configuration bench.py times
(CUDA graph replay, batch 1024): sampling bit-exact on sampled batches (first, second,
middle, ragged last), training steps within 1e-4 of the oracle."""
import numpy as np
import pytest

import oracle
from oracle import sampling as OS
from tests.gpu_common import (TOL_FP32, assert_blocks_equal, check_train_step, inputs_for, make_gpu,
                              rel)

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CASES = {
    "products": dict(batches=(0, 1, 96, 192), steps=3),
    "reddit": dict(batches=(0, 1, 75, 149), steps=2),
    "products_shadow": dict(batches=(0, 192), steps=1),
    # SURVEY.md §8(f) NEXT-1 grid: same samplers as above (their sampling is covered there)
    "products_gcn": dict(batches=(), steps=1),
    "products_sage_shadow": dict(batches=(), steps=1),
    "products_shadow_l5": dict(batches=(), steps=1),
    "papers_small": dict(batches=(0, 1, 19), steps=2),
}


@pytest.mark.parametrize("name", [n for n in CASES if CASES[n]["batches"]])
def test_fullsize_sampling_bitexact(name):
    w, inp, graph = inputs_for(name)
    g, m = make_gpu(w, inp)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    for b in CASES[name]["batches"]:
        want, _ = oracle.sample_batch(w, graph, 0, b, perm)
        got = m.sample(0, b)
        if w.sampler == "shadow":
            assert_blocks_equal(got[0], want[0])
            assert_blocks_equal([got[1]], [want[1]])
        else:
            assert_blocks_equal(got, want)


@pytest.mark.parametrize("name", list(CASES))
def test_fullsize_training_parity(name):
    w, inp, graph = inputs_for(name)
    g, m = make_gpu(w, inp)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    params = inp["params"].astype(np.float64)
    for step in range(CASES[name]["steps"]):
        loss = m.train_minibatch(0, step)
        out = check_train_step(m, w, graph, params, 0, step, perm, loss)
        print(name, step, out["errors"], "elementwise", out["elem"], "kink flips", out["kink_flips"])
        params = out["params"]
        assert rel(m.get_params(), params) <= TOL_FP32
    # ragged last batch through the end-to-end host call, from the initial params
    last = w.n_batches - 1
    seeds = OS.batch_seeds(perm, w.batch_size, last)
    m.set_params(inp["params"])
    loss = m.train_batch_host(seeds, len(seeds), 0, last)
    out = check_train_step(m, w, graph, inp["params"], 0, last, perm, loss)
    print(name, "ragged", out["errors"], "kink flips", out["kink_flips"])


@pytest.mark.parametrize("name", ["products", "reddit"])
def test_fullsize_bf16_gemm_parity(name):
    """The bf16-GEMM variant at full size (BASELINE.json north_star: within 2e-2): steps 0-1 and
    the ragged last batch, loss / logits / every layer's dW."""
    w, inp, graph = inputs_for(name)
    g, m = make_gpu(w, inp, precision="bf16")
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    params = inp["params"].astype(np.float64)
    for step in range(2):
        loss = m.train_minibatch(0, step)
        out = check_train_step(m, w, graph, params, 0, step, perm, loss, precision="bf16")
        print(name, "bf16", step, out["errors"], "kink flips", out["kink_flips"])
        params = out["params"]
        assert rel(m.get_params(), params) <= 2e-2
    last = w.n_batches - 1
    seeds = OS.batch_seeds(perm, w.batch_size, last)
    m.set_params(inp["params"])
    loss = m.train_batch_host(seeds, len(seeds), 0, last)
    out = check_train_step(m, w, graph, inp["params"], 0, last, perm, loss, precision="bf16")
    print(name, "bf16 ragged", out["errors"], "kink flips", out["kink_flips"])


@pytest.mark.parametrize("name", ["products"])
def test_fullsize_exchange_nccl_equals_fused(name):
    """The multi-rank branch (reduce -> one-rank ncclAllReduce -> update) in the bench's launch
    configuration: bit-identical to the fused path over 3 steps."""
    w, inp, graph = inputs_for(name)
    runs = []
    for exch in ("auto", "nccl"):
        g, m = make_gpu(w, inp, exchange=exch)
        losses = [m.train_minibatch(0, s) for s in range(3)]
        runs.append((np.array(losses), m.grads(), m.get_params()))
        m.close(); g.close()
    for a, b in zip(*runs):
        assert np.array_equal(a, b)



@pytest.mark.parametrize("name", ["products", "reddit"])
def test_fullsize_l1_on_sampler_bitidentical(name, monkeypatch):
    """Layer 1's gather on the sampling stream (GS_L1_ON_SAMPLER=1: per-set operand planes, the
    gather of step s+1 overlapping step s) trains bit-identically to the in-graph gather: losses,
    gradients and parameters over 4 steps, then the end-to-end host call on the ragged last batch."""
    w, inp, graph = inputs_for(name)
    perm = OS.epoch_perm(graph["train"], w.sampler_seed, 0)
    last = w.n_batches - 1
    seeds = OS.batch_seeds(perm, w.batch_size, last)
    runs = []
    for mode in ("0", "1"):
        monkeypatch.setenv("GS_L1_ON_SAMPLER", mode)
        g, m = make_gpu(w, inp)
        losses = [m.train_minibatch(0, s) for s in range(4)]
        losses.append(m.train_batch_host(seeds, len(seeds), 0, last))
        runs.append((np.array(losses), m.grads(), m.get_params()))
        m.close(); g.close()
    for a, b in zip(*runs):
        assert np.array_equal(a, b)
