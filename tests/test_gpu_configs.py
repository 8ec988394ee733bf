"""Parity at the BASELINE configurations' full sizes (C1, C2, C3, C4, C4 stress,
C5 buckets) against containers the unmodified reference build wrote
(tests/golden/configs.json, tools/make_config_goldens.py).

Per case, on the same host-generated input and step-0 pipeline seed:
  * the device container's header, index payload (bitmap / RLE bytes, Bloom
    filter) and reorder payload are bit-exact; raw-value containers are
    byte-identical as a whole;
  * fit payloads: identical structure (kind, segment count and bounds, degree,
    sign split) and f32 coefficients within |Δc| <= 1e-5·|c| + 1e-6·max|c_seg|
    (SURVEY §8(a) exactness contract; Eigen's QR is unpinned);
  * substituting the reference's fit payload into the device container gives
    the reference container byte for byte (its SHA-256), and the device decode
    of THAT container reproduces the reference decode bit for bit (support
    and f64 values, including the Bloom positive scan and P2 replay);
  * the device decode of its own container selects the same support, with
    values within 1e-5·max|v| of the reference's.
"""
from __future__ import annotations

import numpy as np
import pytest

from golden_util import coeff_close, load, parse_fit, repack, sha, split

GOLD = load()
CASES = sorted(k for k in GOLD if not k.startswith("_") and "ef_steps" not in GOLD[k])
EF_CASES = sorted(k for k in GOLD if not k.startswith("_") and "ef_steps" in GOLD[k])


def _run(name, oracle):
    import torch

    from paper_2102_03112_b200 import Codec, PipelineConfig
    from paper_2102_03112_b200.configs import CONFIGS, case_input

    gd = GOLD[name]
    cfg = CONFIGS[gd["config"]]
    g, r, lo = case_input(cfg, bucket=gd["bucket"])
    assert lo == gd["first"] and r == gd["r"] and g.size == gd["d"]
    assert sha(g.view(np.uint32)) == gd["input_sha256"], "host input generator drifted from the golden"
    codec = Codec(max_d=gd["d"])
    try:
        pc = PipelineConfig(index_method=gd["index_method"], value_method=gd["value_method"], fpr=gd["fpr"],
                            degree=gd["degree"], max_segments=gd["max_segments"], seed=gd["seed"])
        c = codec.compress(torch.from_numpy(g).cuda(), r, pc).cpu().numpy().tobytes()
        p = split(c)
        assert p["header"].hex() == gd["header_hex"], "header (ids, d, r, payload lengths) differs"
        assert sha(p["index"]) == gd["index_sha256"], "index payload differs"
        assert sha(p["reorder"]) == gd["reorder_sha256"], "reorder payload differs"
        fit = gd["value_method"] in (1, 2)
        if fit:
            ref_v = bytes.fromhex(gd["value_hex"])
            a, b = parse_fit(p["value"]), parse_fit(ref_v)
            for k in ("kind", "S", "bounds", "degree", "l"):
                assert a[k] == b[k], f"fit structure differs: {k}"
            assert coeff_close(a["coeffs"], b["coeffs"]), "fit coefficients outside tolerance"
            ref_c = repack(p, ref_v, oracle.crc32c)
        else:
            assert sha(p["value"]) == gd["value_sha256"], "value payload differs"
            ref_c = c
        assert sha(ref_c) == gd["container_sha256"], "rebuilt reference container differs"

        # the device decode of the reference's own container: bit-exact
        dev_ref = torch.from_numpy(np.frombuffer(ref_c, np.uint8).copy()).cuda()
        d, sup, val = codec.decompress(dev_ref)
        sup_h, val_h = sup.cpu().numpy().astype("<u4"), val.cpu().numpy()
        assert d == gd["d"] and sup_h.size == gd["n_decoded"]
        assert sha(sup_h) == gd["decoded_support_sha256"], "decoded support differs"
        assert sha(val_h.astype("<f8")) == gd["decoded_values_sha256"], "decoded values differ"

        # ... and through the dense accumulate (f32 scatter of the same values)
        dense = torch.zeros(gd["d"], dtype=torch.float32, device="cuda")
        codec.decode_accumulate(dev_ref, dense)
        codec.status()
        want = np.zeros(gd["d"], np.float32)
        want[sup_h] = val_h.astype(np.float32)
        assert np.array_equal(dense.cpu().numpy(), want)

        if fit:  # the device's own container: same support, values within tolerance
            dev_c = torch.from_numpy(np.frombuffer(c, np.uint8).copy()).cuda()
            _, sup2, val2 = codec.decompress(dev_c)
            assert sha(sup2.cpu().numpy().astype("<u4")) == gd["decoded_support_sha256"]
            v2 = val2.cpu().numpy()
            assert np.max(np.abs(v2 - val_h)) <= 1e-5 * np.max(np.abs(val_h))
    finally:
        codec.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_config_parity(name, oracle):
    _run(name, oracle)


@pytest.mark.gpu
@pytest.mark.parametrize("name", EF_CASES)
def test_config_ef_parity(name):
    """Error feedback at the C4 size in the reference's own f64 loop
    (harness.cpp:230-271): every step's container and the residual after it
    are bit-identical to the reference build's (tools/make_config_goldens.py)."""
    import torch

    from paper_2102_03112_b200 import Codec, PipelineConfig
    from paper_2102_03112_b200.configs import CONFIGS, case_input

    gd = GOLD[name]
    cfg = CONFIGS[gd["config"]]
    g, r, _ = case_input(cfg)
    assert sha(g.view(np.uint32)) == gd["input_sha256"]
    codec = Codec(max_d=gd["d"])
    try:
        gdev = torch.from_numpy(g).cuda()
        e = torch.zeros(gd["d"], dtype=torch.float64, device="cuda")
        for k, st in enumerate(gd["ef_steps"]):
            pc = PipelineConfig(index_method=gd["index_method"], value_method=gd["value_method"], fpr=gd["fpr"],
                                seed=st["seed"])
            c = codec.compress_ef64(gdev, e, r, pc).cpu().numpy().tobytes()
            assert sha(c) == st["container_sha256"], f"step {k}: container differs"
            assert sha(e.cpu().numpy().astype("<f8")) == st["residual_sha256"], f"step {k}: residual differs"
    finally:
        codec.close()
