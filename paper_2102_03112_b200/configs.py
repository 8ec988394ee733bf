"""The benchmark configurations (BASELINE.json `configs`).

Plain data, importable without CUDA: bench.py, the golden generator
(tools/make_config_goldens.py) and the config-size parity tests
(tests/test_gpu_configs.py) all read the workload from here.  Method ids are
FORMAT.md's (index: 1 bitmap, 2 rle, 4 bloom-p0, 6 bloom-p2; value: 0 raw f32,
1 fit-poly).
"""
from __future__ import annotations

CONFIGS = {
    "c4": dict(workload="ResNet-50-sized 25.6M-element gradient, top-r 1%, bloom-filter P2 (eps=1e-3) + "
                        "polynomial curve-fit (degree 5), encode+allgather+decode",
               d=25_557_032, ratio=0.01, index=6, value=1, fpr=0.001, degree=5, max_segments=0, sparse=False),
    "c4s": dict(workload="C4 stress point: bloom-filter P2 at eps=1e-2 + polynomial curve-fit",
                d=25_557_032, ratio=0.01, index=6, value=1, fpr=0.01, degree=5, max_segments=0, sparse=False),
    "c4ef": dict(workload="C4 with error feedback (memory compensation, harness.cpp:230/269-271): encode of "
                          "g + residual, residual <- input - decode(own container), then allgather + decode",
                 d=25_557_032, ratio=0.01, index=6, value=1, fpr=0.001, degree=5, max_segments=0, sparse=False,
                 ef=True),
    "c1": dict(workload="synthetic 1M-element gradient, top-r 1%, bloom-filter P0 (eps=1e-2) + polynomial "
                        "curve-fit, single-worker round trip",
               d=1_000_000, ratio=0.01, index=4, value=1, fpr=0.01, degree=5, max_segments=0, sparse=False),
    "c2": dict(workload="ResNet-20-sized 0.27M-element gradient, top-r 1%, bitmap indices + raw f32 values",
               d=269_722, ratio=0.01, index=1, value=0, fpr=0.01, degree=5, max_segments=0, sparse=False),
    "c3": dict(workload="NCF-style natural sparsity (40% zero 64-wide rows), 32M elements, bitmap indices + "
                        "raw f32 values (support = nonzeros)",
               d=31_832_577, ratio=None, index=1, value=0, fpr=0.01, degree=5, max_segments=0, sparse=True),
    "c3r": dict(workload="NCF-style natural sparsity (40% zero 64-wide rows), 32M elements, RLE indices + "
                         "raw f32 values (support = nonzeros)",
                d=31_832_577, ratio=None, index=2, value=0, fpr=0.01, degree=5, max_segments=0, sparse=True),
    "c2r": dict(workload="ResNet-20-sized 0.27M-element gradient, top-r 1%, RLE indices + raw f32 values",
                d=269_722, ratio=0.01, index=2, value=0, fpr=0.01, degree=5, max_segments=0, sparse=False),
    "c5": dict(workload="BERT-large-sized 340M-element gradient, top-r 0.1%, bloom-filter P2 (eps=1e-3) + "
                        "piecewise curve-fit (8 pieces), 16 independent 21.25M buckets, one codec context and stream each",
               d=340_000_000, ratio=0.001, index=6, value=1, fpr=0.001, degree=5, max_segments=8, sparse=False,
               buckets=16),
}
METHOD_NAMES = {0: "none", 1: "bitmap", 2: "rle", 4: "bloom-p0", 5: "bloom-p1", 6: "bloom-p2", 7: "bloom-pd",
                8: "bloom-naive"}
VALUE_NAMES = {0: "raw-f32", 1: "fit-poly", 5: "raw-f64"}


def case_input(cfg: dict, rank: int = 0, seed: int = 1, bucket: int | None = None):
    """(gradient f32 array, r, element offset) of one rank's container in `cfg`
    (one bucket of a bucketed config)."""
    from .inputs import gradient, natural_sparse_gradient
    from .seeds import bucket_bounds, ratio_r
    lo, hi = 0, cfg["d"]
    if cfg.get("buckets"):
        lo, hi = bucket_bounds(cfg["d"], cfg["buckets"])[bucket or 0]
    gen = natural_sparse_gradient if cfg["sparse"] else gradient
    g = gen(hi - lo, rank=rank, seed=seed, first=lo)
    import numpy as np
    r = int(np.count_nonzero(g)) if cfg["ratio"] is None else ratio_r(hi - lo, cfg["ratio"])
    return g, r, lo


def case_seed(cfg: dict, rank: int = 0, step: int = 0, seed: int = 1, bucket: int | None = None) -> int:
    """The pipeline seed of (rank, step) — per bucket for bucketed configs."""
    from .seeds import bucket_seed, pipeline_seed
    if cfg.get("buckets"):
        return bucket_seed(seed, rank, step, bucket or 0)
    return pipeline_seed(seed, rank, step)
