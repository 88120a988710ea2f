"""Workload registry: BASELINE.json configs[0..4] (SURVEY.md §8(d) size table).

Fanouts are listed input-layer-first (reading R1): hop h (seeds = hop 0)
uses fanouts[L-1-h].  Batch size is per rank (reading R8).
"""
from __future__ import annotations

from dataclasses import dataclass, field, asdict


@dataclass(frozen=True)
class Workload:
    name: str
    num_nodes: int
    nnz: int            # target CSR entries (directed); the generator records the actual count
    feat_dim: int
    num_classes: int
    model: str          # "sage" | "gcn"
    sampler: str        # "neighbor" | "shadow"
    fanouts: tuple      # input-layer-first
    num_layers: int
    hidden: int
    batch_size: int
    n_train: int
    graph_seed: int = 17092
    sampler_seed: int = 1
    init_seed: int = 2
    lr: float = 0.01

    @property
    def feat_stride(self) -> int:
        return (self.feat_dim + 3) // 4 * 4

    @property
    def dims(self):
        return [self.feat_dim] + [self.hidden] * (self.num_layers - 1) + [self.num_classes]

    @property
    def n_batches(self) -> int:
        return (self.n_train + self.batch_size - 1) // self.batch_size

    def to_dict(self):
        return asdict(self)


WORKLOADS = {
    # configs[0]: the oracle finishes a whole epoch in seconds
    "tiny": Workload("tiny", 10_000, 100_000, 32, 8, "sage", "neighbor", (10, 5), 2, 32, 64, 10_000),
    # configs[1]: the bench workload (BASELINE.json metric)
    "products": Workload("products", 2_449_029, 61_859_140, 100, 47, "sage", "neighbor",
                         (15, 10, 5), 3, 256, 1024, 196_615),
    # configs[2]: ShaDow K-hop (L'=3 hops [15,10,5]) + 3-layer GCN
    "products_shadow": Workload("products_shadow", 2_449_029, 61_859_140, 100, 47, "gcn", "shadow",
                                (15, 10, 5), 3, 256, 1024, 196_615),
    # configs[3]: Reddit-shaped, high-degree stress
    "reddit": Workload("reddit", 232_965, 114_615_892, 602, 41, "sage", "neighbor",
                       (25, 10), 2, 256, 1024, 153_431),
    # the rest of the paper's model x sampler grid (Table 3,
    # lines 478-493) and its ShaDow depth setting (L' = 3 hops, L = 5 layers)
    "tiny_gcn": Workload("tiny_gcn", 10_000, 100_000, 32, 8, "gcn", "neighbor", (10, 5), 2, 32, 64, 10_000),
    "tiny_sage_shadow": Workload("tiny_sage_shadow", 10_000, 100_000, 32, 8, "sage", "shadow", (10, 5), 2, 32,
                                 64, 10_000),
    "tiny_shadow_l5": Workload("tiny_shadow_l5", 10_000, 100_000, 32, 8, "gcn", "shadow", (10, 5), 5, 32, 64,
                               10_000),
    "products_gcn": Workload("products_gcn", 2_449_029, 61_859_140, 100, 47, "gcn", "neighbor",
                             (15, 10, 5), 3, 256, 1024, 196_615),
    "products_sage_shadow": Workload("products_sage_shadow", 2_449_029, 61_859_140, 100, 47, "sage", "shadow",
                                     (15, 10, 5), 3, 256, 1024, 196_615),
    "products_shadow_l5": Workload("products_shadow_l5", 2_449_029, 61_859_140, 100, 47, "gcn", "shadow",
                                   (15, 10, 5), 5, 256, 1024, 196_615),
    # papers100M's layer shapes (F = 128, C = 172: logits wider than one GEMM tile, the separate
    # cross-entropy kernel) on a graph small enough for the oracle and one GPU; the sharded-table
    # test runs it too (configs[4]'s code path at a testable size)
    "papers_small": Workload("papers_small", 200_000, 3_000_000, 128, 172, "sage", "neighbor",
                             (15, 10, 5), 3, 256, 1024, 20_000),
    # configs[4]: papers100M-shaped (row-sharded features across ranks)
    "papers100m": Workload("papers100m", 111_059_956, 1_615_685_872, 128, 172, "sage", "neighbor",
                           (15, 10, 5), 3, 256, 1024, 1_207_179),
}
