"""The C-ABI library loads on the CPU build box and exports every symbol that
include/gradpack_b200.h declares (no compute calls: there is no GPU here)."""
import ctypes

import pytest

from paper_2102_03112_b200 import PipelineConfig, bloom_params
from paper_2102_03112_b200._lib import LIB_PATH, GpConfig, header_symbols, lib


def test_every_header_symbol_is_exported():
    syms = header_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(lib, name), name


def test_config_defaults_match_pipeline_config():
    c = GpConfig()
    lib.gp_pipeline_config_default(ctypes.byref(c))
    py = PipelineConfig().to_c()
    for f, _ in GpConfig._fields_:
        assert getattr(c, f) == getattr(py, f), f


@pytest.mark.parametrize("eps,r,m,k", [(1e-3, 1000, 14378, 10), (1e-2, 10000, 95851, 7),
                                       (1e-9, 100, 4314, 30), (0.5, 1, 2, 1)])
def test_host_bloom_params(eps, r, m, k):
    assert bloom_params(eps, r) == (m, k)


def test_max_container_bytes_bounds_the_oracle(oracle):
    from oracle.bindings import GpConfig as OC, synthetic_gradient
    g = synthetic_gradient(5000, rank=3)
    for im, vm in [(0, 0), (1, 0), (1, 5), (0, 5)]:
        cfg = PipelineConfig(index_method=im, value_method=vm)
        got = len(oracle.encode_dense(g, 50, OC.make(im, vm)))
        assert got <= lib.gp_max_container_bytes(5000, 50, ctypes.byref(cfg.to_c()))


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("im,vm,kw", [(0, 0, {}), (1, 0, {}), (2, 0, {}), (4, 1, {}), (5, 5, {}), (6, 1, {}),
                                      (7, 0, {}), (8, 1, {}), (1, 1, {}), (1, 3, {}), (6, 3, dict(quant_bits=3)),
                                      (2, 3, dict(quant_bits=16, quant_bucket=7)), (6, 4, dict(slot_codec=0)),
                                      (3, 0, {}), (3, 1, {})])
def test_volume_matches_reference(oracle, reference, im, vm, kw):
    # gp_volume is host code: it runs here, against the reference's own volume()
    from oracle.bindings import GpConfig as OC, synthetic_gradient
    from paper_2102_03112_b200 import volume
    g = synthetic_gradient(20_000, rank=im)
    c = oracle.encode_dense(g, 200, OC.make(im, vm, fpr=0.01, seed=5, **kw))
    got, want = volume(c), reference.volume(c)
    for k in want:
        assert got[k] == pytest.approx(want[k], rel=0, abs=0), k
