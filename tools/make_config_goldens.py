#!/usr/bin/env python
"""Generates tests/golden/configs.json: the reference's own containers at the
BASELINE configurations' full sizes (TEST INFRASTRUCTURE; run here, where
/root/reference exists and oracle/_ref was built from it by oracle/Makefile).

For each case the unmodified reference build (oracle/_ref/libgpref.so:
top_r sparsify.cpp:32-46 → compress_gradient pipeline.cpp:146-221 → pack
container.cpp:58-82, then unpack + decompress_gradient pipeline.cpp:223-306)
encodes the host-generated input (paper_2102_03112_b200/inputs.py, the same
bytes the bench uploads) with the step-0 pipeline seed of rank 0
(harness.cpp:201-203; per-bucket seeds for C5) and decodes its own container.
Stored: SHA-256 of the input, of the container, of every payload and of the
decoded support/values; the 49-byte header and the full fit payload (small),
so that a device-encoded fit container can be compared within the
coefficient tolerance and the reference container rebuilt from it.

  python tools/make_config_goldens.py [case ...]
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from golden_util import GOLDEN, sha, split  # noqa: E402
from oracle.bindings import GpConfig, reference  # noqa: E402
from paper_2102_03112_b200.configs import CONFIGS, case_input, case_seed  # noqa: E402

# (case name, config, bucket)
CASES = [
    ("c1", "c1", None), ("c2", "c2", None), ("c2r", "c2r", None), ("c3", "c3", None), ("c3r", "c3r", None),
    ("c4", "c4", None), ("c4s", "c4s", None), ("c5_b0", "c5", 0), ("c5_b15", "c5", 15),
]


def make(name, cfg_name, bucket, ref):
    cfg = CONFIGS[cfg_name]
    g, r, lo = case_input(cfg, bucket=bucket)
    seed = case_seed(cfg, bucket=bucket)
    cc = GpConfig.make(cfg["index"], cfg["value"], fpr=cfg["fpr"], degree=cfg["degree"],
                       max_segments=cfg["max_segments"], seed=seed)
    t0 = time.perf_counter()
    c = ref.encode_dense(g, r, cc)
    t1 = time.perf_counter()
    d, sup, val = ref.decode(c)
    t2 = time.perf_counter()
    p = split(c)
    assert d == g.size and p["r"] == r
    out = dict(config=cfg_name, bucket=bucket, first=lo, d=int(g.size), r=r, seed=seed,
               index_method=cfg["index"], value_method=cfg["value"], fpr=cfg["fpr"], degree=cfg["degree"],
               max_segments=cfg["max_segments"], input_sha256=sha(g.view(np.uint32)),
               container_len=len(c), container_sha256=sha(c), header_hex=p["header"].hex(),
               index_len=p["il"], index_sha256=sha(p["index"]), value_len=p["vl"], value_sha256=sha(p["value"]),
               reorder_len=p["rl"], reorder_sha256=sha(p["reorder"]), n_decoded=int(sup.size),
               decoded_support_sha256=sha(sup.astype("<u4")), decoded_values_sha256=sha(val.astype("<f8")),
               bits_per_nonzero=8.0 * len(c) / r, ref_encode_s=round(t1 - t0, 3), ref_decode_s=round(t2 - t1, 3))
    if cfg["value"] in (1, 2):
        out["value_hex"] = p["value"].hex()
    return out


# error feedback at C4 size in the reference's f64 loop (harness.cpp:230-271):
# three compensated steps of rank 0 on the same gradient, P2 (eps 1e-3) with
# raw f32 values, so every step's container and the final residual are
# bit-exact targets (with a fit value codec the coefficient tolerance feeds
# into the residual and the next step's selection; tests/test_gpu_ef64.py
# covers fit EF bit-exactly against the reference loop at 200k elements)
EF_CASES = [("c4ef_raw", "c4", 3)]


def make_ef(name, cfg_name, steps, ref):
    cfg = CONFIGS[cfg_name]
    g, r, lo = case_input(cfg)
    res = np.zeros(g.size, np.float64)
    out = dict(config=cfg_name, bucket=None, first=lo, d=int(g.size), r=r, index_method=cfg["index"],
               value_method=0, fpr=cfg["fpr"], degree=cfg["degree"], max_segments=cfg["max_segments"],
               input_sha256=sha(g.view(np.uint32)), ef_steps=[])
    for step in range(steps):
        seed = case_seed(cfg, step=step)
        cc = GpConfig.make(cfg["index"], 0, fpr=cfg["fpr"], seed=seed)
        t0 = time.perf_counter()
        c = ref.ef_step64(g, res, r, cc)
        out["ef_steps"].append(dict(seed=seed, container_len=len(c), container_sha256=sha(c),
                                    residual_sha256=sha(res.astype("<f8")), ref_step_s=round(time.perf_counter() - t0, 3)))
    return out


def main(argv):
    ref = reference()
    if ref is None:
        sys.exit("oracle/_ref/libgpref.so is missing: run `make -C oracle ref` where /root/reference exists")
    want = set(argv) or {c[0] for c in CASES}
    gold = {}
    if os.path.exists(GOLDEN):
        with open(GOLDEN) as f:
            gold = json.load(f)
    for name, cfg_name, bucket in CASES:
        if name not in want:
            continue
        gold[name] = make(name, cfg_name, bucket, ref)
        print(name, {k: gold[name][k] for k in ("d", "r", "container_len", "ref_encode_s", "ref_decode_s")},
              flush=True)
    if not argv:
        want |= {c[0] for c in EF_CASES}
    for name, cfg_name, steps in EF_CASES:
        if name not in want:
            continue
        gold[name] = make_ef(name, cfg_name, steps, ref)
        print(name, gold[name]["ef_steps"], flush=True)
    gold["_meta"] = {"generator": "tools/make_config_goldens.py",
                     "reference": "oracle/_ref/libgpref.so (unmodified /root/reference/proj/src, oracle/Makefile)",
                     "inputs": "paper_2102_03112_b200/inputs.py (rank 0, master seed 1, step 0)"}
    with open(GOLDEN, "w") as f:
        json.dump(dict(sorted(gold.items())), f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main(sys.argv[1:])
