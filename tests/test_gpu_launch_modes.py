"""Launch-mode independence: the step with programmatic dependent launch and
fill kernels (the default) must produce the same bytes as plain stream
ordering with cudaMemsetAsync (GP_PDL=0, GP_FILL_KERNEL=0, read once per
process, hence a subprocess) — containers and dense means of eager and graph
steps, for the dense fast path, RLE, P2 + fit and P1 + quantizer."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import hashlib, json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
from oracle.bindings import synthetic_gradient
from paper_2102_03112_b200 import Codec, PipelineConfig
from paper_2102_03112_b200.dp import SparseAllgather
out = {}
cases = {"bitmap_dense": (dict(index_method=1, value_method=0), None),
         "rle": (dict(index_method=2, value_method=0), 3000),
         "p2_fit": (dict(index_method=6, value_method=1, fpr=0.001), 3000),
         "p1_quant": (dict(index_method=5, value_method=3, fpr=0.01), 3000)}
d = 300_001
for name, (kw, r) in cases.items():
    g = synthetic_gradient(d, rank=3)
    if r is None:  # natural sparsity: the dense fast path (r = nnz)
        g[::3] = 0.0
        r = int(np.count_nonzero(g))
    for graph in (False, True):
        c = Codec(max_d=d)
        ex = SparseAllgather(c, d, r, PipelineConfig(**kw), graph=graph)
        gd = torch.from_numpy(g).cuda()
        h = hashlib.sha256()
        for step in (1, 2):
            dense = ex.step(gd, step=step).clone()
            torch.cuda.synchronize()
            c.status()
            n = int(ex.length.item())
            h.update(ex.out[:n].cpu().numpy().tobytes())
            h.update(dense.cpu().numpy().tobytes())
        out[f"{name}/graph={graph}"] = h.hexdigest()
print(json.dumps(out))
"""


def _run(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    res = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], capture_output=True, text=True, env=env, cwd=ROOT,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    return json.loads(res.stdout.strip().splitlines()[-1])


def test_pdl_and_fill_kernels_do_not_change_results():
    on = _run({"GP_PDL": "1", "GP_FILL_KERNEL": "1"})
    off = _run({"GP_PDL": "0", "GP_FILL_KERNEL": "0"})
    assert on.keys() == off.keys() and len(on) == 8
    for k in on:
        assert on[k] == off[k], k
