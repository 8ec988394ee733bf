"""Error feedback on the CPU: the oracle's restatement (oracle/ef.py over the C
oracle) against the same loop over the reference's own sources (oracle/_ref),
bit-exact, over several compensated steps (harness.cpp:230, :269-271)."""
import numpy as np
import pytest

from oracle.bindings import GpConfig, reference, synthetic_gradient
from oracle.ef import ef_step

CASES = [(1, 0), (2, 0), (0, 5), (4, 0), (5, 0), (6, 0), (7, 0), (8, 0)]


@pytest.mark.parametrize("im,vm", CASES)
def test_ef_oracle_matches_reference(oracle, im, vm):
    ref = reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    d, r = 20_000, 200
    cfg = GpConfig.make(im, vm, fpr=0.01, seed=11)
    e_o = np.zeros(d, np.float32)
    e_r = np.zeros(d, np.float32)
    for step in range(3):
        g = synthetic_gradient(d, rank=step)
        c_o, e_o = ef_step(oracle, g, e_o, r, cfg)
        c_r, e_r = ef_step(ref, g, e_r, r, cfg)
        assert c_o == c_r, f"step {step}: containers differ"
        assert np.array_equal(e_o, e_r), f"step {step}: residuals differ"


def test_ef_residual_identity(oracle):
    """residual + decoded == input exactly where the decoded value is exact
    (raw f32 values: the kept coordinates' residual is 0)."""
    d, r = 10_000, 100
    g = synthetic_gradient(d, rank=3)
    e = synthetic_gradient(d, rank=4) * np.float32(0.1)
    c, res = ef_step(oracle, g, e, r, GpConfig.make(1, 0, seed=5))
    _, sup, _ = oracle.decode(c)
    inp = (g + e).astype(np.float32)
    assert np.all(res[sup] == 0)
    mask = np.ones(d, bool)
    mask[sup] = False
    assert np.array_equal(res[mask], inp[mask])
