"""The C-ABI library builds for sm_100a, loads without a GPU, and exports every symbol
include/gnnstep.h declares (no compute calls here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gnnstep.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(gnn_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["gnn_graph_create", "gnn_model_create", "gnn_sample", "gnn_train_minibatch",
              "gnn_train_epoch", "gnn_get_params", "gnn_set_params", "gnn_comm_init",
              "gnn_train_batch_host"]:
        assert s in syms


def test_library_loads_and_exports_every_symbol():
    from paper_2403_17092_b200 import lib
    L = lib()
    for s in declared_symbols():
        assert hasattr(L, s), s
    assert L.gnn_abi_version() == 2   # 2: gnn_model_config gained optimizer, beta1, beta2, eps
    path = L._name
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    for s in declared_symbols():
        assert re.search(rf"\bT {s}\b", out), s


def test_library_is_sm100a():
    from paper_2403_17092_b200 import lib
    path = lib()._name
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_oracle_not_linked_into_product():
    """The product library and binding never reference the oracle."""
    from paper_2403_17092_b200 import lib
    path = lib()._name
    out = subprocess.run(["nm", "-D", path], capture_output=True, text=True).stdout
    assert "oracle_" not in out
    pkg = os.path.join(ROOT, "paper_2403_17092_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_cache_plan_by_degree_matches_definition():
    """gnn_cache_plan_by_degree (host only, NEXT-2) == its definition written with numpy: the
    `capacity` highest-degree rows outside this shard's block, ties by id, ascending."""
    import numpy as np
    from paper_2403_17092_b200 import cache_plan_by_degree
    rng = np.random.default_rng(8)
    for n, P, cap in ((50, 2, 10), (97, 4, 30), (10, 3, 100), (64, 8, 0)):
        deg = rng.integers(0, 6, size=n)
        rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
        for shard in range(P):
            rps = -(-n // P)
            b, e = min(n, shard * rps), min(n, shard * rps + rps)
            remote = [v for v in range(n) if not (b <= v < e)]
            want = sorted(sorted(remote, key=lambda v: (-deg[v], v))[:cap])
            assert list(cache_plan_by_degree(rp, P, shard, cap)) == want


def test_host_rank_library_exports_its_header_and_is_separate():
    """libgnnhost.so (the host-core trainer rank, include/gnnhost.h) exports every declared gnnh_
    symbol; the GPU library neither defines nor references any of them (no CPU fallback path)."""
    from paper_2403_17092_b200.hostrank import lib as hlib
    txt = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", "gnnhost.h")).read(), flags=re.S)
    syms = sorted(set(re.findall(r"\b(gnnh_[a-z_0-9]+)\s*\(", txt)))
    assert "gnnh_grads" in syms and "gnnh_apply" in syms
    out = subprocess.run(["nm", "-D", "--defined-only", hlib()._name], capture_output=True, text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}\b", out), s
    from paper_2403_17092_b200 import lib
    gpu = subprocess.run(["nm", "-D", lib()._name], capture_output=True, text=True).stdout
    assert "gnnh_" not in gpu
