"""The host input generator (paper_2102_03112_b200/inputs.py) reproduces the
inputs the config goldens were made from, and equals the C restatement's
CounterRng normal stream (gradpack_main.cpp:279-281 generator)."""
from __future__ import annotations

import sys

import numpy as np
import pytest

from golden_util import load, sha


def test_inputs_do_not_load_the_cuda_library():
    import subprocess
    code = ("import sys; from paper_2102_03112_b200 import inputs, seeds, configs; "
            "inputs.gradient(1000); import paper_2102_03112_b200 as p; "
            "assert 'paper_2102_03112_b200.api' not in sys.modules and 'torch' not in sys.modules")
    subprocess.run([sys.executable, "-c", code], check=True, cwd=__file__.rsplit("/tests/", 1)[0])


def test_generator_equals_oracle_stream():
    from oracle.bindings import synthetic_gradient
    from paper_2102_03112_b200 import inputs
    g = inputs.gradient(300_000, rank=3)
    assert np.array_equal(g.view(np.uint32), synthetic_gradient(300_000, rank=3).view(np.uint32))
    assert np.array_equal(inputs.gradient(1000, rank=3, first=123_457), g[123_457:124_457])


@pytest.mark.parametrize("name", sorted(k for k in load() if not k.startswith("_")))
def test_golden_inputs(name):
    from paper_2102_03112_b200.configs import CONFIGS, case_input
    gd = load()[name]
    g, r, lo = case_input(CONFIGS[gd["config"]], bucket=gd["bucket"])
    assert (g.size, r, lo) == (gd["d"], gd["r"], gd["first"])
    assert sha(g.view(np.uint32)) == gd["input_sha256"]


def test_reference_arm_does_not_load_the_cuda_library():
    """bench.py --impl reference runs the reference build only (the
    arm must not map libgradpack_b200.so)."""
    import subprocess
    root = __file__.rsplit("/tests/", 1)[0]
    code = ("import runpy, sys\n"
            "sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c2', '--steps', '1', '--warmup', '0']\n"
            "try:\n    runpy.run_path('bench.py', run_name='__main__')\nexcept SystemExit:\n    pass\n"
            "maps = open('/proc/self/maps').read()\n"
            "assert 'libgradpack_b200' not in maps and 'paper_2102_03112_b200.api' not in sys.modules\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert '"impl": "reference"' in r.stdout
